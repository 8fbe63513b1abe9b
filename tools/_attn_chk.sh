set -x
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "attention or hf or sharding" > gpurun_out/pytest_attn.log 2>&1; echo "pytest rc=$?"; tail -3 gpurun_out/pytest_attn.log
python tools/attn_time.py > /tmp/a.txt 2>&1; cat /tmp/a.txt; python tools/attn_time.py c2 > /tmp/a.txt 2>&1; cat /tmp/a.txt
