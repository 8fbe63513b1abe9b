"""CUDA-event timings of encode (K only / V only / both) and decode for one config."""
import argparse, json, sys
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2604_24971_b200 as pk
from paper_2604_24971_b200.pool import _Arena, _encode_layers

ap = argparse.ArgumentParser()
ap.add_argument("--config", default="c3")
ap.add_argument("--dtype", default="bf16")
ap.add_argument("--iters", type=int, default=10)
ap.add_argument("--kmode", default="tensor")
ap.add_argument("--eager", action="store_true", help="no CUDA graph (includes host launch overhead)")
ap.add_argument("--path", default="stream", choices=["stream", "warp"])
ap.add_argument("--keys-detail", action="store_true", help="also time absmax alone, encode with external maxima, block32")
a = ap.parse_args()
import os
if a.path == 'warp':
    os.environ['PKV_CODEC_PATH'] = 'warp'
L, H, D, T = {"c3": (32, 8, 128, 4096), "c2": (24, 32, 64, 1851), "c1": (24, 32, 64, 600)}[a.config]
dt = torch.bfloat16 if a.dtype == "bf16" else torch.float32
g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
dev = torch.device("cuda")
dump = pk.synth_gaussian_dump(g, seed=0, device=dev, dtype=dt, generator="torch")
ks = [k for k, _ in dump.layers]; vs = [v for _, v in dump.layers]
arena = _Arena(g, L, a.kmode, dev)
none = [None] * L

def graph(fn):
    st = torch.cuda.Stream()
    st.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(st):
        fn()
    torch.cuda.current_stream().wait_stream(st)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr):
        fn()
    return gr.replay


def timeit(fn):
    if not a.eager:
        fn = graph(fn)
    for _ in range(3): fn()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record()
    for _ in range(a.iters): fn()
    e.record(); torch.cuda.synchronize()
    return s.elapsed_time(e) / a.iters

res = {}
res["enc_k"] = timeit(lambda: _encode_layers(ks, none, g, pk.GAUSSIAN_3BIT, None, a.kmode, device=dev, arena=arena, check=False))
res["enc_v"] = timeit(lambda: _encode_layers(none, vs, g, pk.GAUSSIAN_3BIT, None, a.kmode, device=dev, arena=arena, check=False))
kb, vb, _ = _encode_layers(ks, vs, g, pk.GAUSSIAN_3BIT, None, a.kmode, device=dev, arena=arena, check=False)
res["enc_kv"] = timeit(lambda: _encode_layers(ks, vs, g, pk.GAUSSIAN_3BIT, None, a.kmode, device=dev, arena=arena, check=False))
pool = pk.SharedPool(g, list(zip(kb, vb))).seal()
res["dec_k"] = timeit(lambda: pool.decode_layers(None, torch.bfloat16, values=False))
res["dec_v"] = timeit(lambda: pool.decode_layers(None, torch.bfloat16, keys=False))
res["dec_kv"] = timeit(lambda: pool.decode_layers(None, torch.bfloat16))
if a.keys_detail:
    # where the key role's time goes: the standalone absmax kernel, the key
    # encode with external maxima (one pass, no absmax items) and block32
    from paper_2604_24971_b200 import _codec as C
    mx = torch.empty(L, dtype=torch.int32, device=dev)
    kin = [k.values for k in ks]
    res["absmax_kernel"] = timeit(lambda: C.k_absmax(kin, mx, kin[0].device))
    res["enc_k_extmax"] = timeit(lambda: _encode_layers(ks, none, g, pk.GAUSSIAN_3BIT, None, a.kmode, device=dev,
                                                        arena=arena, check=False, k_layer_max=mx))
    arena32 = _Arena(g, L, "block32", dev)
    res["enc_k_block32"] = timeit(lambda: _encode_layers(ks, none, g, pk.GAUSSIAN_3BIT, None, "block32", device=dev,
                                                         arena=arena32, check=False))
n = g.elements_per_tensor * L
inb = 2 if a.dtype == "bf16" else 4
bytes_ = {"enc_k": n * (inb + 1), "enc_v": n * (inb + 3 / 8) + 4 * n / D, "dec_k": 3 * n, "dec_v": n * (2 + 3 / 8) + 4 * n / D}
bytes_["enc_kv"] = bytes_["enc_k"] + bytes_["enc_v"]; bytes_["dec_kv"] = bytes_["dec_k"] + bytes_["dec_v"]
bytes_["absmax_kernel"] = n * inb; bytes_["enc_k_extmax"] = bytes_["enc_k"]; bytes_["enc_k_block32"] = n * (inb + 1 + 2 / 32)
print(a.config, a.dtype, a.path, json.dumps({k: {"ms": round(v, 4), "GBs": round(bytes_[k] / v / 1e6, 1)} for k, v in res.items()}))
print("replays", int(arena.replay.item()), flush=True)
