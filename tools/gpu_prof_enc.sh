# instruction-throughput microbenchmark + full ncu captures of the encode
# kernel (value-only, key-only, fused launches) with source attribution
set -x
tools/ubench_pipes > gpurun_out/ubench_pipes.txt 2>&1; cat gpurun_out/ubench_pipes.txt
for only in v k kv; do
  ncu --set full --import-source on --clock-control none -k regex:"enc_kernel" -c 1 -o gpurun_out/enc_$only -f \
    python tools/prof_codec.py --iters 1 --only $only > gpurun_out/ncu_enc_$only.log 2>&1
  python tools/ncu_summary.py gpurun_out/enc_$only.ncu-rep --ops 30 --top 20 > gpurun_out/enc_${only}_full.txt 2>&1
done
rm -f gpurun_out/enc_k.ncu-rep gpurun_out/enc_kv.ncu-rep
ls -la gpurun_out
