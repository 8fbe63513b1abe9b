# encode experiments: layer wait off (dbg 4), 8K-element items (variant c8k)
echo base; python tools/time_codec.py --iters 20 2>&1 | head -1 | cut -c1-140
for f in 0.3 0.35 0.4; do echo "frac $f"; PKV_KEY_SM_FRACTION=$f python tools/time_codec.py --iters 20 2>&1 | head -1 | cut -c1-140; done
