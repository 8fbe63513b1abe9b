set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
for dt in bf16 f32; do
python tools/time_codec.py --iters 30 --dtype $dt > /tmp/t.txt 2>&1; head -1 /tmp/t.txt
echo "dbg1 (no math)"; PKV_DBG_ENC=1 python tools/time_codec.py --iters 30 --dtype $dt > /tmp/t.txt 2>&1; head -1 /tmp/t.txt
done
