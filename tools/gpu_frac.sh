set -x
for f in 0.42 0.45 0.47 0.49 0.52; do echo "f32 frac $f"; PKV_KEY_SM_FRACTION=$f python tools/time_codec.py --iters 40 --dtype f32 > /tmp/t.txt 2>&1; head -1 /tmp/t.txt | cut -c90-140; done
for f in 0.34 0.36 0.38 0.40 0.42; do echo "bf16 frac $f"; PKV_KEY_SM_FRACTION=$f python tools/time_codec.py --iters 40 --dtype bf16 > /tmp/t.txt 2>&1; head -1 /tmp/t.txt | cut -c90-140; done
