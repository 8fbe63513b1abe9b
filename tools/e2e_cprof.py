"""cProfile of the host side of a pinned-host build_pool (pipeline chunk 4)."""
import cProfile, pstats, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2604_24971_b200 as pk

L, H, D, T = 32, 8, 128, 4096
g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
dev = torch.device("cuda")
dump = pk.synth_gaussian_dump(g, seed=0, device=dev, dtype=torch.bfloat16, generator="torch")
host = [(k.values.cpu().pin_memory(), v.values.cpu().pin_memory()) for k, v in dump.layers]
hd = pk.KvDump(g, tuple((pk.KvTensor(g, k), pk.KvTensor(g, v)) for k, v in host))
for _ in range(2):
    pk.build_pool(hd, build_stats=False, device=dev, check=False)
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(3):
    pk.build_pool(hd, build_stats=False, device=dev, check=False)
pr.disable()
torch.cuda.synchronize()
pstats.Stats(pr).sort_stats("tottime").print_stats(12)
