set -x
timeout 900 python -m pytest tests -m gpu -x -q -p no:cacheprovider -k "attention or smoke or hf or decode" > gpurun_out/pytest_attn.log 2>&1; echo "pytest rc=$?"
tail -30 gpurun_out/pytest_attn.log
python tools/attn_time.py > gpurun_out/attn_time.txt 2>&1; cat gpurun_out/attn_time.txt
PKV_ATTN_PATH=simt python tools/attn_time.py > gpurun_out/attn_time_simt.txt 2>&1; cat gpurun_out/attn_time_simt.txt
python tools/attn_time.py c2 > /tmp/a.txt 2>&1; cat /tmp/a.txt
PKV_ATTN_PATH=simt python tools/attn_time.py c2 > /tmp/a.txt 2>&1; cat /tmp/a.txt
