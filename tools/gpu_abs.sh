set -x
for f in 0.22 0.26 0.3 0.34; do echo "values-absmax frac $f"; PKV_ABSMAX_ROLE=values PKV_KEY_SM_FRACTION=$f python tools/time_codec.py --iters 30 --dtype bf16 > /tmp/t.txt 2>&1; head -1 /tmp/t.txt | cut -c1-160; done
for f in 0.3 0.36 0.42; do echo "f32 values-absmax frac $f"; PKV_ABSMAX_ROLE=values PKV_KEY_SM_FRACTION=$f python tools/time_codec.py --iters 30 --dtype f32 > /tmp/t.txt 2>&1; head -1 /tmp/t.txt | cut -c1-160; done
for f in 0.34 0.38 0.42; do echo "f32 baseline frac $f"; PKV_KEY_SM_FRACTION=$f python tools/time_codec.py --iters 30 --dtype f32 > /tmp/t.txt 2>&1; head -1 /tmp/t.txt | cut -c1-160; done
PKV_ABSMAX_ROLE=values timeout 900 python -m pytest tests/test_gpu_parity.py tests/test_gpu_full_configs.py -q -p no:cacheprovider -x -k "bit_exact or role or random" > gpurun_out/pytest_abs.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_abs.log
