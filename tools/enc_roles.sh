# which role bounds the fused encode at the default split: 1 no math, 2 no value math, 3 no key math
for d in 0 1 2 3; do echo "dbg $d"; PKV_DBG_ENC=$d python tools/time_codec.py --iters 50 2>&1 | head -1 | cut -c100-150; done
