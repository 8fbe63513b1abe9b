set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_gpu.log
bash tools/ab_env.sh "" "" -- --dtype f32 --iters 40
bash tools/ab_env.sh "" "" -- --dtype bf16 --iters 40
