set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -15 gpurun_out/pytest_gpu.log
for dt in f32 bf16; do for lag in 2 4 6; do echo "co $dt lag $lag"; PKV_KEY_LAG=$lag timeout 300 python tools/time_codec.py --iters 40 --dtype $dt > /tmp/t.txt 2>&1; head -1 /tmp/t.txt | cut -c1-170; done; done
echo "split f32"; PKV_ENC_ROLES=split timeout 300 python tools/time_codec.py --iters 40 --dtype f32 > /tmp/t.txt 2>&1; head -1 /tmp/t.txt | cut -c1-170
echo "co c2 f32"; timeout 300 python tools/time_codec.py --iters 40 --dtype f32 --config c2 > /tmp/t.txt 2>&1; head -1 /tmp/t.txt | cut -c1-170
echo "co c2 bf16"; timeout 300 python tools/time_codec.py --iters 40 --dtype bf16 --config c2 > /tmp/t.txt 2>&1; head -1 /tmp/t.txt | cut -c1-170
