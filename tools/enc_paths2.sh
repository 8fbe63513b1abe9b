timeout 200 python -m pytest tests -m gpu -x -q 2>&1 | tail -1
timeout 60 python tools/prof_codec.py --iters 1 > gpurun_out/plain_p2.log 2>&1
ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none -k regex:"enc_kernel|key_kernel|dec_kernel" -c 3 --csv python tools/prof_codec.py --iters 1 > gpurun_out/ncu_p2.csv 2>&1
