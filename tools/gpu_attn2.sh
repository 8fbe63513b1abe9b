set -x
for c in 1 2 3 4 6; do echo "ctas/sm $c"; PKV_ATTN_CTAS_PER_SM=$c python tools/attn_time.py > /tmp/a.txt 2>&1; cat /tmp/a.txt; PKV_ATTN_CTAS_PER_SM=$c python tools/attn_time.py c2 > /tmp/a.txt 2>&1; cat /tmp/a.txt; done
ncu --set full --import-source on --clock-control none -k regex:"prefix_mma|combine" -c 2 -o gpurun_out/attn_mma -f python tools/prof_codec.py --iters 1 --attn --only kv > gpurun_out/ncu_attn.log 2>&1
python tools/ncu_summary.py gpurun_out/attn_mma.ncu-rep --ops 30 --top 25 > gpurun_out/attn_mma_full.txt 2>&1
cat gpurun_out/attn_mma_full.txt | head -60
