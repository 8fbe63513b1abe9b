# encode balance: K-only / V-only on the whole GPU, and the fused kernel vs key-SM share
python tools/time_codec.py --iters 20
for f in 0.3 0.35 0.4 0.45 0.5; do echo "frac $f"; PKV_KEY_SM_FRACTION=$f python tools/time_codec.py --iters 20 2>&1 | head -1; done
python tools/time_codec.py --iters 20 --dtype f32 2>&1 | head -1
python tools/time_codec.py --iters 20 --config c2 2>&1 | head -1
