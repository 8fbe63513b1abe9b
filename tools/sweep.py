"""BASELINE configs[4]: compression-kernel bandwidth sweep, 1K-128K tokens x
head_dim 64/128, one B200.

Each point: `build_pool` (pkv_encode, all layers) and a full materialise to
bf16 (pkv_decode), CUDA-graph captured, inputs (f32 or bf16) generated on the
device (torch generator). Prints one JSON line per point; GB/s use the §8(d)
algorithmic bytes. Layers are reduced at long contexts to bound memory.
Bit-exactness along the sweep: tests/test_gpu_sweep_parity.py.
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

import paper_2604_24971_b200 as pk  # noqa: E402
from paper_2604_24971_b200 import _codec  # noqa: E402
from paper_2604_24971_b200.keyquant import K_MODES  # noqa: E402
from paper_2604_24971_b200.pool import _Arena, _encode_layers  # noqa: E402

SHAPES = {64: (24, 32), 128: (32, 8)}  # head_dim -> (layers, kv_heads): SmolLM2 / Llama-3-8B


def algorithmic_bytes(L, H, D, T, in_b=2, out_b=2):
    n, vecs = H * T * D, H * T
    comp = L * (n * in_b + n + 4 + n * in_b + 3 * n / 8 + 4 * vecs)
    deq = L * (n + 4 + n * out_b + 3 * n / 8 + 4 * vecs + n * out_b)
    return comp, deq


def point(D, T, dtype="bf16", max_bytes=24e9, reps=10):
    L, H = SHAPES[D]
    in_b = 2 if dtype == "bf16" else 4
    per_layer = 2 * H * T * D * (in_b + 2)  # inputs + outputs
    L = max(1, min(L, int(max_bytes // per_layer)))
    g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
    dev = torch.device("cuda")
    dump = pk.synth_gaussian_dump(g, seed=0, device=dev, dtype=torch.bfloat16 if in_b == 2 else torch.float32,
                                  generator="torch")
    ks, vs = [k for k, _ in dump.layers], [v for _, v in dump.layers]
    arena = _Arena(g, L, "tensor", dev)
    kb, vb, _ = _encode_layers(ks, vs, g, pk.GAUSSIAN_3BIT, None, "tensor", device=dev, arena=arena)
    pool = pk.SharedPool(g, list(zip(kb, vb))).seal()
    ko = [torch.empty(g.tensor_shape, dtype=torch.bfloat16, device=dev) for _ in range(L)]
    vo = [torch.empty(g.tensor_shape, dtype=torch.bfloat16, device=dev) for _ in range(L)]

    def enc():
        _encode_layers(ks, vs, g, pk.GAUSSIAN_3BIT, None, "tensor", device=dev, arena=arena, check=False)

    def dec():
        _codec.decode(num_vectors=g.vectors_per_tensor, head_dim=D, out_dtype=torch.bfloat16,
                      k_mode=K_MODES["tensor"], k_codes=pool.k_codes, k_scale=pool.k_scale, k_bscale=None,
                      v_packed=pool.v_packed, v_scales=pool.v_scales, centroids=pk.GAUSSIAN_3BIT.centroids,
                      sign_seed=None, k_out=ko, v_out=vo, device=dev)

    def graph(fn):
        s = torch.cuda.Stream()
        s.wait_stream(torch.cuda.current_stream())
        with torch.cuda.stream(s):
            fn()
        torch.cuda.current_stream().wait_stream(s)
        gr = torch.cuda.CUDAGraph()
        with torch.cuda.graph(gr):
            fn()
        return gr.replay

    def timeit(fn):
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record()
        for _ in range(reps):
            fn()
        b.record()
        torch.cuda.synchronize()
        return a.elapsed_time(b) / reps

    te, td = timeit(graph(enc)), timeit(graph(dec))
    cb, dbb = algorithmic_bytes(L, H, D, T, in_b=in_b)
    peak = json.loads((Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").read_text()).get("hbm_gbs", 6561.0) \
        if (Path(__file__).resolve().parents[1] / "MEASURED_PEAKS.json").exists() else 6561.0
    res = {"head_dim": D, "seq_len": T, "layers": L, "kv_heads": H, "dtype_in": dtype, "encode_ms": te,
           "decode_ms": td, "encode_frac_of_hbm_peak": cb / te / 1e6 / peak,
           "encode_gbs": cb / te / 1e6, "decode_gbs": dbb / td / 1e6,
           "step_gbs": (cb + dbb) / (te + td) / 1e6, "frac_of_hbm_peak": (cb + dbb) / (te + td) / 1e6 / peak}
    del dump, ks, vs, arena, pool, ko, vo
    torch.cuda.empty_cache()
    return res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--tokens", default="1024,2048,4096,8192,16384,32768,65536,131072")
    ap.add_argument("--dims", default="64,128")
    ap.add_argument("--dtypes", default="f32,bf16")
    a = ap.parse_args()
    for dt in a.dtypes.split(","):
        for D in (int(x) for x in a.dims.split(",")):
            for T in (int(x) for x in a.tokens.split(",")):
                print(json.dumps(point(D, T, dt)), flush=True)
