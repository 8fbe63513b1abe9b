set -x
tools/ubench_pipes > gpurun_out/ubench_pipes2.txt 2>&1; cat gpurun_out/ubench_pipes2.txt
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -5 gpurun_out/pytest_gpu.log
