# bench lines + launch list + full captures of the codec / attention kernels (one GPU);
# summaries are written on the box (reports are large); keeps codec_full.ncu-rep only
set -x
python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
python bench.py --config c2 --skip-decode-e2e > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --skip-e2e --skip-decode-e2e > gpurun_out/ncu_launch.log 2>&1
python tools/show_ncu_csv.py gpurun_out/launches.csv | grep -vE "at::|elementwise|distribution" > gpurun_out/launches_bench_c3.txt
rm -f gpurun_out/launches.csv
ncu --set full --import-source on --clock-control none -k regex:"enc_kernel|dec_kernel" -c 2 -o gpurun_out/codec_full -f python tools/prof_codec.py --iters 1 > gpurun_out/ncu_codec.log 2>&1
python tools/ncu_summary.py gpurun_out/codec_full.ncu-rep > gpurun_out/encode_decode_full.txt 2>&1
ncu --set full --clock-control none -k regex:"enc_kernel|dec_kernel" -c 2 -o /tmp/codec_full_c2 -f python tools/prof_codec.py --iters 1 --config c2 > gpurun_out/ncu_codec_c2.log 2>&1
python tools/ncu_summary.py /tmp/codec_full_c2.ncu-rep > gpurun_out/encode_decode_full_c2.txt 2>&1
ncu --set full --clock-control none -k regex:"prefix_kernel2|combine_kernel" -c 2 -o /tmp/attn_full -f python tools/prof_codec.py --iters 1 --attn > gpurun_out/ncu_attn.log 2>&1
python tools/ncu_summary.py /tmp/attn_full.ncu-rep > gpurun_out/attention_full.txt 2>&1
du -sh gpurun_out
tail -c 300 gpurun_out/bench.json
