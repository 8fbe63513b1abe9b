# fused encode vs key-SM share
for rep in 1 2; do for f in "$@"; do echo "frac $f"; PKV_KEY_SM_FRACTION=$f python tools/time_codec.py --iters 50 2>&1 | head -1 | cut -c100-150; done; done
