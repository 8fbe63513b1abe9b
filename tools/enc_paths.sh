# encode-kernel time for K only, V only, K+V (C3 bf16), one ncu timing pass each
for o in k v kv; do timeout 60 python tools/prof_codec.py --iters 1 --only $o > gpurun_out/plain_$o.log 2>&1; done
for o in k v kv; do ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,smsp__inst_executed.sum --clock-control none -k regex:"enc_kernel|absmax_kernel" -c 3 --csv python tools/prof_codec.py --iters 1 --only $o > gpurun_out/ncu_path_$o.csv 2>&1; done
