set -x
ncu --set full --import-source on --clock-control none -k regex:"enc_kernel" -c 1 -o gpurun_out/enc_k -f \
    python tools/prof_codec.py --iters 1 --only k > gpurun_out/ncu_enc_k.log 2>&1
python tools/ncu_summary.py gpurun_out/enc_k.ncu-rep --ops 30 --top 30 > gpurun_out/enc_k_full.txt 2>&1
ncu --set full --import-source on --clock-control none -k regex:"enc_kernel" -c 1 -o gpurun_out/enc_k32 -f \
    python tools/prof_codec.py --iters 1 --only k --dtype f32 > gpurun_out/ncu_enc_k32.log 2>&1
python tools/ncu_summary.py gpurun_out/enc_k32.ncu-rep --ops 30 --top 30 > gpurun_out/enc_k32_full.txt 2>&1
rm -f gpurun_out/enc_k32.ncu-rep
ls -la gpurun_out
