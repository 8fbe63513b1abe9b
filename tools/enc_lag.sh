# key-role absmax lag (layers): key-only on all SMs and fused at 0.4
for lag in 2 4 6 8 12; do echo "lag $lag"; PKV_KEY_LAG=$lag python tools/time_codec.py --iters 20 2>&1 | head -1 | cut -c1-140; done
