# fused encode time vs the share of SMs given to the key role (C3 bf16)
timeout 200 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 60 python tools/prof_codec.py --iters 1 --only kv > gpurun_out/plain_f.log 2>&1
for f in 0.3 0.4 0.5; do PKV_KEY_SM_FRACTION=$f ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"enc_kernel" -c 1 --csv python tools/prof_codec.py --iters 1 --only kv > gpurun_out/ncu_frac_$f.csv 2>&1; done
for o in k v; do ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum --clock-control none -k regex:"enc_kernel" -c 1 --csv python tools/prof_codec.py --iters 1 --only $o > gpurun_out/ncu_only_$o.csv 2>&1; done
ncu --metrics gpu__time_duration.sum --clock-control none -k regex:"dec_kernel" -c 1 --csv python tools/prof_codec.py --iters 1 > gpurun_out/ncu_dec7.csv 2>&1
