# the N>1 bench path (layer-sharded encode + pool gather + per-shard decode,
# agents partitioned) on a 1-GPU box: ranks share cuda:0 over gloo; checks the
# code path end to end (the timing is meaningless)
set -x
timeout 900 python bench.py --gpus 2 --dist-backend gloo --steps 3 --warmup 3 --skip-cpu --skip-decode-e2e > gpurun_out/multi2.json 2> gpurun_out/multi2.err; echo "rc=$?"
tail -c 2500 gpurun_out/multi2.json; tail -5 gpurun_out/multi2.err
timeout 900 python bench.py --gpus 3 --dist-backend gloo --config c2 --steps 3 --warmup 3 --skip-cpu --skip-decode-e2e > gpurun_out/multi3.json 2> gpurun_out/multi3.err; echo "rc=$?"
tail -c 800 gpurun_out/multi3.json; tail -5 gpurun_out/multi3.err
