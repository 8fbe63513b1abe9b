"""Run encode + decode (+ attention) once or a few times for ncu captures."""
import argparse, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2604_24971_b200 as pk
from paper_2604_24971_b200 import _codec
from paper_2604_24971_b200.pool import _Arena, _encode_layers
from paper_2604_24971_b200.attention import decode_attention

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--iters", type=int, default=2)
ap.add_argument("--attn", action="store_true")
ap.add_argument("--only", default="kv")
ap.add_argument("--kmode", default="tensor")
ap.add_argument("--dec", default="kv", help="decode keys (k), values (v) or both")
a = ap.parse_args()
L, H, D, T = {"c3": (32, 8, 128, 4096), "c2": (24, 32, 64, 1851)}[a.config]
dt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
dev = torch.device("cuda")
dump = pk.synth_gaussian_dump(g, seed=0, device=dev, dtype=dt, generator="torch")
ks = [k for k, _ in dump.layers]; vs = [v for _, v in dump.layers]
arena = _Arena(g, L, a.kmode, dev)
for _ in range(a.iters):
    kb, vb, _ = _encode_layers(ks if "k" in a.only else [None]*L, vs if "v" in a.only else [None]*L, g, pk.GAUSSIAN_3BIT, None, a.kmode, device=dev, arena=arena, check=False)
if a.only == "kv":
    pool = pk.SharedPool(g, list(zip(kb, vb))).seal()
    for _ in range(a.iters):
        pool.decode_layers(None, torch.bfloat16, keys="k" in a.dec, values="v" in a.dec)
if a.attn:
    q = torch.randn(15, H, 4, D, device=dev, dtype=torch.bfloat16)
    for _ in range(a.iters):
        decode_attention(pool, 0, q)
torch.cuda.synchronize()
print("replays", int(arena.replay.item()))
