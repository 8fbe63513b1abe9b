"""Bit-exact parity along the C5 sweep (BASELINE configs[4]: 1K-128K tokens x
head_dim 64/128, f32 and bf16 inputs): one build per point, the per-tensor
key scale over the WHOLE layer, key / value codes and scales and the 16-bit
decode checked on sampled head vectors (first, middle and last 2048 of the
layer; vectors are independent given the layer's key scale, valuequant.py:
200-211, keyquant.py:55-65). tools/sweep.py measures the same points."""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2604_24971_b200 as pk
from oracle import kvpool_oracle as O

pytestmark = pytest.mark.gpu

SHAPES = {64: 32, 128: 8}  # head_dim -> kv_heads (SmolLM2 / Llama-3-8B)
POINTS = [(128, 1024, "bf16"), (128, 16384, "f32"), (128, 131072, "bf16"),
          (64, 2048, "f32"), (64, 65536, "bf16"), (64, 131072, "f32")]


def u32(t):
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().astype(np.uint16).astype(np.uint32) << 16
    return t.float().numpy().view(np.uint32)


@pytest.mark.parametrize("D,T,dt", POINTS, ids=lambda p: str(p))
def test_sweep_point_bit_exact_on_sampled_vectors(D, T, dt):
    H = SHAPES[D]
    L = 2
    g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
    dtype = torch.bfloat16 if dt == "bf16" else torch.float32
    dump = pk.synth_gaussian_dump(g, seed=T + D, device="cuda", dtype=dtype, generator="torch")
    pool = pk.build_pool(dump, build_stats=False)
    li = L - 1
    k = dump.layers[li][0].values.reshape(-1, D)
    v = dump.layers[li][1].values.reshape(-1, D)
    nvec = k.shape[0]
    peak = float(k.float().abs().max())
    scale = float(np.float32(peak / 127))
    kq, vq = pool.layer_blocks(li)
    assert kq.scale == scale
    kc_all = kq.codes.reshape(-1, D)
    packed = vq.packed
    sc_all = vq.scales.reshape(-1)
    (kd16, vd16), = pool.decode_layers([li], torch.bfloat16)
    kd16, vd16 = kd16.reshape(-1, D), vd16.reshape(-1, D)
    for v0 in (0, nvec // 2 - 1024, nvec - 2048):
        sl = slice(v0, v0 + 2048)
        kh = k[sl].float().cpu().numpy()
        vh = v[sl].float().cpu().numpy()
        # keys with the WHOLE layer's scale (keyquant.py:60-64)
        q = kh.astype(np.float64) / scale
        want_k = np.clip(np.floor(np.abs(q) + 0.5) * np.sign(q), -128, 127).astype(np.int8)
        assert np.array_equal(kc_all[sl].cpu().numpy(), want_k)
        vc, vs = O.quantize_v(vh)
        got_packed = packed[v0 * 3 * D // 8:(v0 + 2048) * 3 * D // 8].cpu().numpy()
        assert np.array_equal(got_packed, np.frombuffer(O.pack3(vc), dtype=np.uint8))
        assert np.array_equal(u32(sc_all[sl]), vs.view(np.uint32))
        kd, vd = O.decode_layer(want_k, scale, vc, vs, 16)
        assert np.array_equal(u32(kd16[sl]), kd.view(np.uint32))
        assert np.array_equal(u32(vd16[sl]), vd.view(np.uint32))
