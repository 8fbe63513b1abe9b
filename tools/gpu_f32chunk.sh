set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -4 gpurun_out/pytest_gpu.log
for f in 0.36 0.40 0.45 0.50; do echo "f32 frac $f"; PKV_KEY_SM_FRACTION=$f python tools/time_codec.py --iters 40 --dtype f32 > /tmp/t.txt 2>&1; head -1 /tmp/t.txt | cut -c1-170; done
python tools/time_codec.py --iters 40 --dtype f32 --config c2 > /tmp/t.txt 2>&1; head -1 /tmp/t.txt | cut -c1-170
