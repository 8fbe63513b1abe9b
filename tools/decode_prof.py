"""Kernel-time breakdown of model-level pooled decode (torch.profiler / CUPTI):
which kernels a greedy decode step spends its time in. Usage: python tools/decode_prof.py [c3|c2]"""
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
sys.path.insert(0, str(Path(__file__).resolve().parent))
import decode_bench  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c3"
decode_bench.run(cfg, steps=2, modes=("pooled_graph",))  # warm (allocator, libraries)
with torch.profiler.profile(activities=[torch.profiler.ProfilerActivity.CUDA]) as prof:
    decode_bench.run(cfg, steps=8, modes=("pooled_graph",))
print(prof.key_averages().table(sort_by="cuda_time_total", row_limit=25, max_name_column_width=70))
