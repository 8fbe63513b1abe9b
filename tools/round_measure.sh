# round-2 measurements: bench (headline f32 + bf16 variant + e2e + attention + model decode + CPU ref),
# reference arm, C5 sweep, ncu launch list + full captures
set -x
nvidia-smi --query-gpu=name,clocks.sm,clocks.max.sm,power.draw --format=csv
python bench.py > gpurun_out/bench_c3.json 2> gpurun_out/bench_c3.err; echo "bench rc=$?"; tail -c 600 gpurun_out/bench_c3.json
python bench.py --config c2 --skip-cpu > gpurun_out/bench_c2.json 2> gpurun_out/bench_c2.err; echo "bench c2 rc=$?"
python bench.py --config c4 --skip-cpu --skip-decode-e2e > gpurun_out/bench_c4.json 2> gpurun_out/bench_c4.err; echo "bench c4 rc=$?"
python bench.py --impl reference --steps 3 --warmup 3 > gpurun_out/reference_arm.json 2> gpurun_out/reference_arm.err; echo "ref rc=$?"; cat gpurun_out/reference_arm.json
python tools/sweep.py > gpurun_out/sweep_c5.jsonl 2> gpurun_out/sweep.err; echo "sweep rc=$?"
ncu --metrics gpu__time_duration.sum --clock-control none -c 400 --csv --log-file gpurun_out/launches.csv python bench.py --steps 3 --warmup 3 --skip-e2e --skip-decode-e2e --skip-cpu --skip-variant > gpurun_out/ncu_launch.log 2>&1
python tools/show_ncu_csv.py gpurun_out/launches.csv | grep -vE "at::|elementwise|distribution" > gpurun_out/launches_bench_c3.txt; rm -f gpurun_out/launches.csv
ncu --set full --import-source on --clock-control none -k regex:"enc_kernel|dec_kernel" -c 2 -o /tmp/codec_f32 -f python tools/prof_codec.py --iters 1 --dtype f32 > gpurun_out/ncu_codec_f32.log 2>&1
python tools/ncu_summary.py /tmp/codec_f32.ncu-rep > gpurun_out/encode_decode_full_f32.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:"enc_kernel|dec_kernel" -c 2 -o /tmp/codec_bf16 -f python tools/prof_codec.py --iters 1 --dtype bf16 > gpurun_out/ncu_codec_bf16.log 2>&1
python tools/ncu_summary.py /tmp/codec_bf16.ncu-rep > gpurun_out/encode_decode_full_bf16.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:"prefix_mma|combine" -c 2 -o /tmp/attn -f python tools/prof_codec.py --iters 1 --attn > gpurun_out/ncu_attn.log 2>&1
python tools/ncu_summary.py /tmp/attn.ncu-rep > gpurun_out/attention_full.txt 2>&1
ls -la gpurun_out
