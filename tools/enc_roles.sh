# which role bounds the fused encode: skip value math (2) / key math (3)
for f in 0.3 0.4 0.5; do for d in 0 2 3; do echo "frac $f dbg $d"; PKV_DBG_ENC=$d PKV_KEY_SM_FRACTION=$f python tools/time_codec.py --iters 20 2>&1 | head -1 | cut -c1-120; done; done
ncu --set full --import-source on --clock-control none -k regex:enc_kernel -c 1 -o gpurun_out/enc_k_only -f python tools/prof_codec.py --iters 1 --only k > gpurun_out/ncu_konly.log 2>&1
