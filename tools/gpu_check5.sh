set -x
timeout 1500 python -m pytest tests -m gpu -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -6 gpurun_out/pytest_gpu.log
for dt in bf16 f32; do python tools/time_codec.py --iters 30 --dtype $dt > /tmp/t.txt 2>&1; head -1 /tmp/t.txt; done
python tools/attn_time.py > /tmp/a.txt 2>&1; cat /tmp/a.txt
python tools/attn_time.py c2 > /tmp/a.txt 2>&1; cat /tmp/a.txt
