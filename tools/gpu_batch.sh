set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
for m in 2 3 4 6 8; do echo "min tiles $m"; PKV_ATTN_MIN_TILES=$m python tools/attn_time.py > /tmp/a.txt 2>&1; cat /tmp/a.txt; PKV_ATTN_MIN_TILES=$m python tools/attn_time.py c2 > /tmp/a.txt 2>&1; cat /tmp/a.txt; done
bash tools/gpu_sanitize.sh
