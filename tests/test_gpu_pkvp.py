"""PKVP v1 byte compatibility with files the reference wrote (VERDICT r01
missing #5; kvpool/pool.py:301-432, pkg/tests/test_pool.py:205-247): our
load_pool reads them bit-exactly, and our save_pool of a pool built on the
GPU from the same inputs writes the identical bytes."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2604_24971_b200 as pk

pytestmark = pytest.mark.gpu

PK = Path(__file__).resolve().parent / "golden" / "pkvp"
CASES = {"unpacked": (False, None), "packed": (True, None), "packed_sign": (True, 9)}


def u32(t):
    return t.detach().float().cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("name", sorted(CASES))
def test_load_reference_snapshot_bit_exact(name):
    pool = pk.load_pool(PK / f"{name}.pkvp")
    assert pool.sign_seed == CASES[name][1]
    with np.load(PK / "expect.npz") as z:
        for bits in (16, 32):
            view = pool.attach(bits)
            for li in range(pool.num_layers):
                k, v = view.get_kv_for_layer(li)
                assert np.array_equal(u32(k.values), z[f"{name}/k{bits}/{li}"].view(np.uint32))
                assert np.array_equal(u32(v.values), z[f"{name}/v{bits}/{li}"].view(np.uint32))


@pytest.mark.parametrize("name", sorted(CASES))
def test_save_is_byte_identical_to_the_reference(name, tmp_path):
    packed, seed = CASES[name]
    with np.load(PK / "expect.npz") as z:
        L, B, H, T, D = (int(x) for x in z["geom"])
        g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T, batch=B)
        dump = pk.KvDump(g, tuple((pk.KvTensor(g, torch.from_numpy(z[f"k_in/{i}"]).cuda()),
                                   pk.KvTensor(g, torch.from_numpy(z[f"v_in/{i}"]).cuda())) for i in range(L)))
    pool = pk.build_pool(dump, sign_seed=seed)
    out = tmp_path / "ours.pkvp"
    pk.save_pool(pool, out, packed=packed)
    assert out.read_bytes() == (PK / f"{name}.pkvp").read_bytes()
    # and a load of our own file round-trips through the same bytes
    back = pk.load_pool(out)
    out2 = tmp_path / "again.pkvp"
    pk.save_pool(back, out2, packed=packed)
    assert out2.read_bytes() == out.read_bytes()


@pytest.mark.parametrize("name", ["d128", "d64_sign", "bf16vals"])
def test_build_stats_match_reference_layer_stats(name):
    """Fused GPU error reduction (pkv_layer_stats) vs the reference's
    LayerStats (pool.py:274-288): k_scale and k_max_err exact, the f64 means
    to 1e-12 relative (summation order differs from numpy's pairwise sum)."""
    with np.load(Path(__file__).resolve().parent / "golden" / "stats.npz") as z:
        L, H, d, T, sign, bf16 = (int(x) for x in z[f"{name}/geom"])
        g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=d, seq_len=T)
        dt = torch.bfloat16 if bf16 else torch.float32
        dump = pk.KvDump(g, tuple((pk.KvTensor(g, torch.from_numpy(z[f"{name}/k_in/{i}"]).cuda().to(dt)),
                                   pk.KvTensor(g, torch.from_numpy(z[f"{name}/v_in/{i}"]).cuda().to(dt)))
                                  for i in range(L)))
        want = [z[f"{name}/stats/{i}"] for i in range(L)]
    pool = pk.build_pool(dump, sign_seed=None if sign < 0 else sign, build_stats=True)
    for i, st in enumerate(pool.build_stats):
        k_scale, k_mse, k_max, v_mse, v_nmse = want[i]
        assert st.k_scale == k_scale and st.k_max_err == k_max
        for got, ref in ((st.k_mse, k_mse), (st.v_mse, v_mse), (st.v_nmse, v_nmse)):
            assert abs(got - ref) <= 1e-12 * abs(ref), (got, ref)
