# parity tests + a short bench (kernel timings only)
set -x
timeout 1500 python -m pytest tests -m gpu -x -q -p no:cacheprovider > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?"
tail -3 gpurun_out/pytest_gpu.log
timeout 600 python bench.py --steps 30 --warmup 5 --skip-e2e --skip-attention --skip-decode-e2e --skip-cpu > gpurun_out/bench_quick.json 2> gpurun_out/bench_quick.err; echo "bench rc=$?"
python - <<'PY'
import json
d=json.loads(open("gpurun_out/bench_quick.json").read().strip().splitlines()[-1])
for k in ("kernels","variant"):
    v=d[k]; print(k, {x: (round(y,4) if isinstance(y,float) else y) for x,y in v.items()})
print("value", d["value"], "frac", d["roofline"]["frac"])
PY
