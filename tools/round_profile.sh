# bench line + launch list + full captures of the codec kernels (one GPU)
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --skip-e2e --skip-decode-e2e > gpurun_out/ncu_launch.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"enc_kernel|dec_kernel" -c 2 -o gpurun_out/codec_full -f python tools/prof_codec.py --iters 1 > gpurun_out/ncu_codec.log 2>&1
ncu --set full --import-source on --clock-control none -k regex:"prefix_kernel2|combine_kernel" -c 2 -o gpurun_out/attn_full -f python tools/prof_codec.py --iters 1 --attn > gpurun_out/ncu_attn.log 2>&1
tail -c 300 gpurun_out/bench.json
