"""Parity of the sm_100a codec (through the C ABI) with the oracle / reference goldens.

Bar: bit-exact codes, scales, packed bytes and decoded K/V (f32 and bf16);
attention within 1e-3 relative of an fp64 oracle.
"""

from __future__ import annotations

import os

import numpy as np
import pytest
import torch

import paper_2604_24971_b200 as pk
from paper_2604_24971_b200 import _lib
from oracle import kvpool_oracle as O
from pkv_testutil import golden_case

pytestmark = pytest.mark.gpu

POOL_CASES = ["c1mini", "d128", "d128_sign", "d64_batch2", "d8", "d16", "d32", "d256", "bf16in", "laplace"]


def u32(t):
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        return (t.view(torch.int16).numpy().astype(np.uint16).astype(np.uint32) << 16)
    return t.float().numpy().view(np.uint32)


def dump_from_golden(golden, name, dtype=torch.float32):
    c = golden_case(golden, name)
    g = pk.ModelGeometry(num_layers=c["L"], kv_heads=c["H"], head_dim=c["D"], seq_len=c["T"], batch=c["B"])
    layers = []
    for li in range(c["L"]):
        k = torch.from_numpy(golden[f"{name}/k_in/{li}"]).cuda().to(dtype)
        v = torch.from_numpy(golden[f"{name}/v_in/{li}"]).cuda().to(dtype)
        layers.append((pk.KvTensor(g, k), pk.KvTensor(g, v)))
    return c, pk.KvDump(g, tuple(layers))


@pytest.mark.parametrize("name", POOL_CASES)
def test_build_pool_bit_exact_vs_reference(golden, name):
    c, dump = dump_from_golden(golden, name)
    pool = pk.build_pool(dump, sign_seed=c["sign_seed"])
    for li in range(c["L"]):
        kq, vq = pool.layer_blocks(li)
        assert kq.scale == float(golden[f"{name}/k_scale/{li}"][0])
        assert np.array_equal(kq.codes.cpu().numpy(), golden[f"{name}/k_codes/{li}"])
        assert np.array_equal(vq.codes.cpu().numpy(), golden[f"{name}/v_codes/{li}"])
        assert np.array_equal(vq.packed.cpu().numpy(), golden[f"{name}/v_packed/{li}"])
        assert np.array_equal(u32(vq.scales), golden[f"{name}/v_scales/{li}"].view(np.uint32))


@pytest.mark.parametrize("name", POOL_CASES)
@pytest.mark.parametrize("bits", [16, 32])
def test_get_kv_for_layer_bit_exact(golden, name, bits):
    c, dump = dump_from_golden(golden, name)
    pool = pk.build_pool(dump, sign_seed=c["sign_seed"])
    view = pool.attach(bits)
    for li in range(c["L"]):
        k, v = view.get_kv_for_layer(li)
        assert k.values.dtype == (torch.bfloat16 if bits == 16 else torch.float32)
        assert np.array_equal(u32(k.values), golden[f"{name}/k{bits}/{li}"].view(np.uint32))
        assert np.array_equal(u32(v.values), golden[f"{name}/v{bits}/{li}"].view(np.uint32))


@pytest.mark.parametrize("name", ["c1mini", "d128_sign", "d8"])
def test_inject_all_transcript_matches_reference(golden, name):
    c, dump = dump_from_golden(golden, name)
    pool = pk.build_pool(dump, sign_seed=c["sign_seed"])
    tr = pool.attach(16).inject_all()
    assert np.array_equal(np.array(tr.checksums(), dtype=np.uint64), golden[f"{name}/checksums16"])


def test_bf16_inputs_give_reference_codes(golden):
    # bf16 device inputs (exactly the bf16-rounded values of the golden case)
    c, dump = dump_from_golden(golden, "bf16in", dtype=torch.bfloat16)
    pool = pk.build_pool(dump)
    for li in range(c["L"]):
        kq, vq = pool.layer_blocks(li)
        assert kq.scale == float(golden[f"bf16in/k_scale/{li}"][0])
        assert np.array_equal(kq.codes.cpu().numpy(), golden[f"bf16in/k_codes/{li}"])
        assert np.array_equal(vq.codes.cpu().numpy(), golden[f"bf16in/v_codes/{li}"])
        assert np.array_equal(u32(vq.scales), golden[f"bf16in/v_scales/{li}"].view(np.uint32))


def test_value_threshold_ties(golden):
    x = golden["tie/v_in"]
    g = pk.ModelGeometry(num_layers=1, kv_heads=1, head_dim=128, seq_len=64)
    vq = pk.quantize_v(pk.KvTensor(g, torch.from_numpy(x).cuda()))
    assert np.array_equal(vq.codes.cpu().numpy(), golden["tie/v_codes"])
    assert np.array_equal(u32(vq.scales), golden["tie/v_scales"].view(np.uint32))


@pytest.mark.parametrize("kat", ["sym", "grid", "half", "halfgrid_all"])
def test_key_known_answers(golden, kat):
    vals = golden[f"kat/{kat}/in"]
    g = pk.ModelGeometry(num_layers=1, kv_heads=1, head_dim=1, seq_len=vals.size)
    kq = pk.quantize_k(pk.KvTensor(g, torch.from_numpy(vals.reshape(1, 1, -1, 1)).cuda()))
    assert kq.scale == float(golden[f"kat/{kat}/scale"][0])
    assert np.array_equal(kq.codes.cpu().numpy().reshape(-1), golden[f"kat/{kat}/codes"])


def test_key_half_point_adversaries():
    # values at exact (n + 1/2) * s for many n with a non-power-of-two scale:
    # the fp32 fast path must hand these to the exact path
    rng = np.random.default_rng(11)
    peak = np.float32(1.7)
    s = np.float32(peak / 127)
    n = rng.integers(-126, 126, size=20000)
    vals = ((n + 0.5) * np.float64(s)).astype(np.float32)
    vals = np.concatenate([vals, np.nextafter(vals, np.float32(np.inf)), np.nextafter(vals, np.float32(-np.inf)),
                           [peak]]).astype(np.float32)
    g = pk.ModelGeometry(num_layers=1, kv_heads=1, head_dim=1, seq_len=vals.size)
    kq = pk.quantize_k(pk.KvTensor(g, torch.from_numpy(vals.reshape(1, 1, -1, 1)).cuda()))
    scale, want = O.quantize_k_tensor(vals.reshape(1, 1, -1, 1))
    assert kq.scale == scale
    assert np.array_equal(kq.codes.cpu().numpy(), want)


def test_full_config1_shape_bit_exact():
    # BASELINE configs[0]: SmolLM2 shape L24 H32 d64 T600, seed 0, full size
    g = pk.ModelGeometry(num_layers=24, kv_heads=32, head_dim=64, seq_len=600)
    layers = O.synth_dump(24, 32, 64, 600, seed=0)
    dump = pk.KvDump(g, tuple((pk.KvTensor(g, torch.from_numpy(k).cuda()),
                               pk.KvTensor(g, torch.from_numpy(v).cuda())) for k, v in layers))
    pool = pk.build_pool(dump)
    view = pool.attach(16)
    decoded = view.materialize_all()
    for li in (0, 7, 23):
        k, v = layers[li]
        scale, kc = O.quantize_k_tensor(k)
        vc, vs = O.quantize_v(v)
        kq, vq = pool.layer_blocks(li)
        assert kq.scale == scale and np.array_equal(kq.codes.cpu().numpy(), kc)
        assert np.array_equal(vq.codes.cpu().numpy(), vc)
        assert np.array_equal(u32(vq.scales), vs.view(np.uint32))
        kd, vd = O.decode_layer(kc, scale, vc, vs, 16)
        assert np.array_equal(u32(decoded[li][0]), kd.view(np.uint32))
        assert np.array_equal(u32(decoded[li][1]), vd.view(np.uint32))
    from fractions import Fraction
    assert Fraction(g.baseline_cache_nbytes() * 8, pool.logical_payload_bits()) == Fraction(32, 11)


@pytest.mark.parametrize("d", [64, 128])
def test_block32_keys_match_restatement(d):
    rng = np.random.default_rng(d)
    x = rng.normal(0, 0.2, size=(1, 4, 77, d)).astype(np.float32)
    x[0, 1, 3, :] *= 1e-3
    x[0, 2, 5, :32] = 0.0
    g = pk.ModelGeometry(num_layers=1, kv_heads=4, head_dim=d, seq_len=77)
    kq = pk.quantize_k(pk.KvTensor(g, torch.from_numpy(x).cuda()), k_scale_mode="block32")
    s16, codes = O.quantize_k_block32(x)
    assert np.array_equal(kq.block_scales.cpu().numpy().view(np.uint16), s16.view(np.uint16))
    assert np.array_equal(kq.codes.cpu().numpy(), codes)
    back = pk.dequantize_k(kq).values.cpu().numpy()
    assert np.array_equal(back.view(np.uint32), O.dequantize_k_block32(codes, s16).view(np.uint32))


def test_large_shape_properties():
    # Llama-3-8B layer shape at 4K tokens through the whole path; properties that
    # hold at any size: key error <= s/2, value NMSE ~ 0.0345, determinism,
    # pool bytes O(1) in agents, idempotent requantisation of decoded keys.
    g = pk.ModelGeometry(num_layers=2, kv_heads=8, head_dim=128, seq_len=4096)
    dump = pk.synth_gaussian_dump(g, seed=0, device="cuda", generator="torch", dtype=torch.bfloat16)
    p1 = pk.build_pool(dump, build_stats=True)
    p2 = pk.build_pool(dump, build_stats=False)
    for li in range(2):
        k1, v1 = p1.layer_blocks(li)
        k2, v2 = p2.layer_blocks(li)
        assert torch.equal(k1.codes, k2.codes) and torch.equal(v1.packed, v2.packed)
        assert torch.equal(v1.scales, v2.scales)
        st = p1.build_stats[li]
        assert st.k_max_err <= st.k_scale / 2 * (1 + 1e-6)
        assert abs(st.v_nmse - 0.0345) < 0.002
    # O(1) in agents, measured on the device: 15 attached views that each
    # materialised the pool leave the pool's HBM bytes and the allocator's
    # live total unchanged once their decoded tensors are dropped
    torch.cuda.synchronize()
    before, alloc0 = p1.device_nbytes(), torch.cuda.memory_allocated()
    for _ in range(15):
        p1.attach(16).materialize_all()
    torch.cuda.synchronize()
    assert p1.device_nbytes() == before and torch.cuda.memory_allocated() == alloc0
    kd = pk.dequantize_k(p1.layer_blocks(0)[0])
    kq2 = pk.quantize_k(kd)
    assert torch.equal(kq2.codes, p1.layer_blocks(0)[0].codes)


def test_nonfinite_input_raises_geometry_error():
    g = pk.ModelGeometry(num_layers=2, kv_heads=2, head_dim=64, seq_len=8)
    dump = pk.synth_gaussian_dump(g, seed=1, device="cuda")
    dump.layers[1][1].values[0, 1, 2, 3] = float("nan")
    with pytest.raises(pk.GeometryError, match="NaN or Inf"):
        pk.build_pool(dump)
    dump = pk.synth_gaussian_dump(g, seed=1, device="cuda")
    dump.layers[0][0].values[0, 0, 0, 0] = float("inf")
    with pytest.raises(pk.GeometryError, match="NaN or Inf"):
        pk.build_pool(dump)


def test_views_are_bit_identical_and_transcripts_agree():
    g = pk.ModelGeometry(num_layers=3, kv_heads=2, head_dim=32, seq_len=16)
    pool = pk.build_pool(pk.synth_gaussian_dump(g, seed=20, device="cuda"))
    a, b = pool.attach(), pool.attach()
    assert a.agent_id != b.agent_id
    assert a.inject_all().checksums() == b.inject_all().checksums()
    with pytest.raises(IndexError):
        a.get_kv_for_layer(3)


def test_packed_snapshot_roundtrip(tmp_path, golden):
    c, dump = dump_from_golden(golden, "d128_sign")
    pool = pk.build_pool(dump, sign_seed=c["sign_seed"])
    for packed in (False, True):
        path = tmp_path / f"p{int(packed)}.pkvp"
        pk.save_pool(pool, path, packed=packed)
        back = pk.load_pool(path)
        assert back.sign_seed == c["sign_seed"]
        for li in range(c["L"]):
            (k1, v1), (k2, v2) = pool.decode_layers([li])[0], back.decode_layers([li])[0]
            assert torch.equal(k1, k2) and torch.equal(v1, v2)


# (kv_heads, head_dim, seq_len, agents, group): 64-row tiles with ragged T,
# 16-row tiles at d=64 (8 CTAs per SM: many one-tile splits, T < one tile,
# T one token past a tile) and at d=128
ATTN_SHAPES = [(8, 128, 1000, 15, 4), (32, 64, 1851, 5, 1), (32, 64, 40, 3, 1), (4, 64, 4097, 16, 1),
               (8, 128, 700, 2, 4), (2, 128, 65, 1, 4)]


@pytest.mark.parametrize("shape", ATTN_SHAPES, ids=lambda s: "h%d_d%d_t%d_a%d_g%d" % s)
def test_decode_attention_matches_fp64_oracle(shape):
    from paper_2604_24971_b200 import attention as A

    H, D, T, R, G = shape
    g = pk.ModelGeometry(num_layers=1, kv_heads=H, head_dim=D, seq_len=T)
    dump = pk.synth_gaussian_dump(g, seed=3, device="cuda")
    pool = pk.build_pool(dump, build_stats=False)
    q = torch.randn(R, H, G, D, device="cuda")
    tail_len = torch.randint(0, 9, (R,), device="cuda", dtype=torch.int32)
    tk = torch.randn(R, H, 8, D, device="cuda").bfloat16()
    tv = torch.randn(R, H, 8, D, device="cuda").bfloat16()
    out = A.decode_attention(pool, 0, q, tail_k=tk, tail_v=tv, tail_len=tail_len,
                             softmax_scale=D ** -0.5, out_dtype=torch.float32)
    (kd, vd), = pool.decode_layers([0], torch.float32)
    tails_k = [tk[r, :, : int(tail_len[r])].float().cpu().numpy() for r in range(R)]
    tails_v = [tv[r, :, : int(tail_len[r])].float().cpu().numpy() for r in range(R)]
    want = O.attention_over_pool(q.cpu().numpy(), kd[0].cpu().numpy(), vd[0].cpu().numpy(), D ** -0.5,
                                 tails_k, tails_v)
    got = out.cpu().numpy().astype(np.float64)
    rel = np.abs(got - want).max() / np.abs(want).max()
    assert rel < 1e-3, rel


def test_decode_division_sequence_is_correctly_rounded():
    # exhaustive over all f32 mantissas: x / f32(sqrt(d)) for d in {8, 32, 128} and x / 127 (pkv_selftest)
    from paper_2604_24971_b200 import _lib

    scratch = torch.zeros(4, dtype=torch.int32, device="cuda")  # 4 counters
    n = _lib.load().pkv_selftest(1, scratch.data_ptr(), 16, torch.cuda.current_stream().cuda_stream)
    assert n == 0, f"{n} mismatches vs IEEE division"


def test_sharded_build_single_rank_equals_build_pool():
    from paper_2604_24971_b200 import parallel

    g = pk.ModelGeometry(num_layers=3, kv_heads=4, head_dim=128, seq_len=40)
    dump = pk.synth_gaussian_dump(g, seed=9, device="cuda")
    a = pk.build_pool(dump)
    b = parallel.build_pool_sharded(dump)
    for i in range(3):
        (ka, va), (kb, vb) = a.layer_blocks(i), b.layer_blocks(i)
        assert torch.equal(ka.codes, kb.codes) and ka.scale == kb.scale
        assert torch.equal(va.packed, vb.packed) and torch.equal(va.scales, vb.scales)


def test_pinned_host_pipeline_equals_device_build():
    g = pk.ModelGeometry(num_layers=7, kv_heads=4, head_dim=128, seq_len=64)
    dump = pk.synth_gaussian_dump(g, seed=4, device="cuda", dtype=torch.bfloat16, generator="torch")
    host = pk.KvDump(g, tuple((pk.KvTensor(g, k.values.cpu().pin_memory()), pk.KvTensor(g, v.values.cpu().pin_memory()))
                              for k, v in dump.layers))
    a = pk.build_pool(dump)
    b = pk.build_pool(host, pipeline_chunk=2)
    outs = [(torch.empty(g.tensor_shape, dtype=torch.bfloat16).pin_memory(),
             torch.empty(g.tensor_shape, dtype=torch.bfloat16).pin_memory()) for _ in range(7)]
    b.attach(16).materialize_to_host(outs, chunk=3)
    torch.cuda.synchronize()
    ref = a.attach(16).materialize_all()
    for i in range(7):
        (ka, va), (kb, vb) = a.layer_blocks(i), b.layer_blocks(i)
        assert torch.equal(ka.codes, kb.codes) and torch.equal(va.packed, vb.packed)
        assert torch.equal(outs[i][0], ref[i][0].cpu()) and torch.equal(outs[i][1], ref[i][1].cpu())


def test_verify_passes_and_catches_a_flipped_byte():
    # kvpool verify (cli.py:216-315); test_cli.py:64-73 flips one payload byte
    from paper_2604_24971_b200.verify import verify_pool

    g = pk.ModelGeometry(num_layers=3, kv_heads=4, head_dim=64, seq_len=96)
    dump = pk.synth_gaussian_dump(g, seed=12, device="cuda")
    pool = pk.build_pool(dump)
    rep = verify_pool(dump, pool, agents=(1, 4))
    assert rep.ok, rep.lines()
    pool.layer_blocks(1)[1].packed[7] ^= 0x10
    rep = verify_pool(dump, pool, agents=(1, 2))
    assert not rep.ok and "payload" in [line for line in rep.lines() if line.startswith("FAIL")][0]


def test_config2_shape_sampled_layers_bit_exact():
    # BASELINE configs[1]: SmolLM2 shape at 1,851 tokens; three layers checked
    L, H, D, T = 24, 32, 64, 1851
    g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
    layers = O.synth_dump(L, H, D, T, seed=0)
    dump = pk.KvDump(g, tuple((pk.KvTensor(g, torch.from_numpy(k).cuda().to(torch.bfloat16)),
                               pk.KvTensor(g, torch.from_numpy(v).cuda().to(torch.bfloat16))) for k, v in layers))
    pool = pk.build_pool(dump, build_stats=False)
    dec = pool.attach(16).materialize_all()
    for li in (0, 11, 23):
        k = dump.layers[li][0].values.float().cpu().numpy()
        v = dump.layers[li][1].values.float().cpu().numpy()
        scale, kc = O.quantize_k_tensor(k)
        vc, vs = O.quantize_v(v)
        kq, vq = pool.layer_blocks(li)
        assert kq.scale == scale and np.array_equal(kq.codes.cpu().numpy(), kc)
        assert np.array_equal(vq.codes.cpu().numpy(), vc)
        assert np.array_equal(u32(vq.scales), vs.view(np.uint32))
        kd, vd = O.decode_layer(kc, scale, vc, vs, 16)
        assert np.array_equal(u32(dec[li][0]), kd.view(np.uint32))
        assert np.array_equal(u32(dec[li][1]), vd.view(np.uint32))


@pytest.mark.parametrize("seed", range(int(os.environ.get("PKV_STRESS_SEEDS", "16"))))
def test_random_shapes_tails_and_modes_bit_exact(seed):
    """Ragged shapes through the TMA paths: token counts that leave partial
    tiles / partial bulk copies, every supported head_dim, bf16 and f32 inputs,
    both key modes, sign diagonals; everything bit-exact vs the oracle."""
    rng = np.random.default_rng(100 + seed)
    D = int(rng.choice([1, 2, 4, 8, 16, 32, 64, 64, 128, 128, 128, 256]))
    H = int(rng.integers(1, 5))
    T = int(rng.integers(1, 700))
    L = int(rng.integers(1, 4))
    dtype = torch.bfloat16 if seed % 2 else torch.float32
    mode = "block32" if seed % 3 == 2 else "tensor"
    sign_seed = 7 if seed % 3 == 1 else None
    g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
    layers = O.synth_dump(L, H, D, T, seed=seed)
    dump = pk.KvDump(g, tuple((pk.KvTensor(g, torch.from_numpy(k).cuda().to(dtype)),
                               pk.KvTensor(g, torch.from_numpy(v).cuda().to(dtype))) for k, v in layers))
    pool = pk.build_pool(dump, sign_seed=sign_seed, k_scale_mode=mode, build_stats=False)
    for bits in (16, 32):
        dec = pool.attach(bits).materialize_all()
        for li in range(L):
            k = dump.layers[li][0].values.float().cpu().numpy()
            v = dump.layers[li][1].values.float().cpu().numpy()
            vc, vs = O.quantize_v(v, sign_seed=sign_seed)
            kq, vq = pool.layer_blocks(li)
            if mode == "tensor":
                scale, kc = O.quantize_k_tensor(k)
                assert kq.scale == scale
                kd, vd = O.decode_layer(kc, scale, vc, vs, bits, sign_seed=sign_seed)
            else:
                s16, kc = O.quantize_k_block32(k)
                assert np.array_equal(kq.block_scales.cpu().numpy().view(np.uint16), s16.view(np.uint16))
                kd, vd = O.decode_layer(kc, 0.0, vc, vs, bits, sign_seed=sign_seed, k_block_scales=s16)
            assert np.array_equal(kq.codes.cpu().numpy(), kc), (li, D, T)
            assert np.array_equal(vq.codes.cpu().numpy(), vc), (li, D, T)
            assert np.array_equal(u32(vq.scales), vs.view(np.uint32))
            assert np.array_equal(u32(dec[li][0]), kd.view(np.uint32)), (li, bits)
            assert np.array_equal(u32(dec[li][1]), vd.view(np.uint32)), (li, bits)


@pytest.mark.parametrize("mode", ["tensor", "block32"])
def test_role_splits_and_schedules_do_not_change_results(monkeypatch, mode):
    # the encode / decode work split between key and value CTAs, the absmax
    # lag and the interleaved-decode fallback are scheduling knobs only:
    # every setting must give bit-identical pools and decoded tensors
    g = pk.ModelGeometry(num_layers=9, kv_heads=4, head_dim=128, seq_len=700)
    dump = pk.synth_gaussian_dump(g, seed=11, device="cuda", dtype=torch.bfloat16, generator="torch")
    ref = pk.build_pool(dump, k_scale_mode=mode)
    ref_out = ref.attach(16).materialize_all()
    # (also the co-resident encode kernel, PKV_ENC_ROLES=co, against the
    # default role-split one; SM shares only matter to the split kernel)
    # ("absval": the per-tensor absmax items run on the value CTAs, PKV_ABSMAX_ROLE=values)
    for enc_frac, dec_frac, lag, roles in [("0.1", "0.1", "1", "split"), ("0.6", "0", "2", "split"),
                                           ("0.9", "0.9", "8", "split"), ("0.3", "0.3", "1", "co"),
                                           ("0.3", "0.3", "7", "co"), ("0.3", "0.3", "2", "absval"),
                                           ("0.05", "0.3", "3", "absval")]:
        monkeypatch.setenv("PKV_KEY_SM_FRACTION", enc_frac)
        monkeypatch.setenv("PKV_DEC_KEY_FRACTION", dec_frac)
        monkeypatch.setenv("PKV_KEY_LAG", lag)
        monkeypatch.setenv("PKV_ENC_ROLES", "split" if roles == "absval" else roles)
        monkeypatch.setenv("PKV_ABSMAX_ROLE", "values" if roles == "absval" else "keys")
        _lib.reload_tuning()  # knobs are read once per process otherwise
        p = pk.build_pool(dump, k_scale_mode=mode)
        for i in range(g.num_layers):
            (ka, va), (kb, vb) = ref.layer_blocks(i), p.layer_blocks(i)
            assert torch.equal(ka.codes, kb.codes) and torch.equal(va.packed, vb.packed)
            assert torch.equal(va.scales, vb.scales)
            if mode == "tensor":
                assert ka.scale == kb.scale
            else:
                assert torch.equal(ka.block_scales, kb.block_scales)
        for (k0, v0), (k1, v1) in zip(ref_out, p.attach(16).materialize_all()):
            assert torch.equal(k0, k1) and torch.equal(v0, v1)
    monkeypatch.undo()
    _lib.reload_tuning()
