"""Bit-exact parity at the configurations the benchmark is quoted on.

VERDICT r01 weak #2: the benched C3 shape (Llama-3-8B KV, L32 H8 d128
T4096) had only property checks. Here the whole C3 dump (the reference's own
generator, kvpool/model.py:250-273, seed 0) goes through one build, in f32
(the reference's dtype) and in bf16, and every layer's key codes / scale and
value codes / scales are compared with the oracle (kvpool/keyquant.py:52-65,
valuequant.py:193-219); decoded K/V (pool.py:229-237) on sampled layers. C4
(T = 7,194) is checked on sampled layers of a full 32-layer build. Attention
at the C3/C4 shapes is compared with an fp64 softmax over the ORACLE's decode
of the ORACLE's codes (independent of the GPU decode), including block32 keys
and the sign diagonal. Also the FMA-adversarial replay vectors
(tests/golden/adversarial_fma.npz).
"""

from __future__ import annotations

import os
from pathlib import Path

import numpy as np
import pytest
import torch

import paper_2604_24971_b200 as pk
from oracle import kvpool_oracle as O
from pkv_testutil import oracle_layers

pytestmark = pytest.mark.gpu

GOLDEN_DIR = Path(__file__).resolve().parent / "golden"


def u32(t):
    t = t.detach().cpu()
    if t.dtype == torch.bfloat16:
        return t.view(torch.int16).numpy().astype(np.uint16).astype(np.uint32) << 16
    return t.float().numpy().view(np.uint32)


def device_dump(g, host_layers, dtype):
    return pk.KvDump(g, tuple((pk.KvTensor(g, torch.from_numpy(k).cuda().to(dtype)),
                               pk.KvTensor(g, torch.from_numpy(v).cuda().to(dtype))) for k, v in host_layers))


def as_oracle_input(t):
    """The exact f32 values the device saw (bf16 inputs widen exactly)."""
    return t.values.float().cpu().numpy()


def check_pool_layers(pool, dump, layers, k_mode="tensor", sign_seed=None):
    pairs = [(as_oracle_input(dump.layers[li][0]), as_oracle_input(dump.layers[li][1])) for li in layers]
    want = oracle_layers(pairs, sign_seed=sign_seed, k_mode=k_mode)
    for li, w in zip(layers, want):
        kq, vq = pool.layer_blocks(li)
        if k_mode == "tensor":
            assert kq.scale == w["k_scale"], li
        else:
            assert np.array_equal(kq.block_scales.cpu().numpy().view(np.uint16), w["k_bscale"].view(np.uint16)), li
        assert np.array_equal(kq.codes.cpu().numpy(), w["k_codes"]), li
        assert np.array_equal(vq.codes.cpu().numpy(), w["v_codes"]), li
        assert np.array_equal(u32(vq.scales), w["v_scales"].view(np.uint32)), li
    return dict(zip(layers, want))


def check_decoded(pool, want, layers, bits=16, sign_seed=None, k_mode="tensor"):
    view = pool.attach(bits)
    for li in layers:
        w = want[li]
        kd, vd = O.decode_layer(w["k_codes"], w.get("k_scale", 0.0), w["v_codes"], w["v_scales"], bits,
                                sign_seed=sign_seed, k_block_scales=w.get("k_bscale") if k_mode != "tensor" else None)
        k, v = view.get_kv_for_layer(li)
        assert np.array_equal(u32(k.values), kd.view(np.uint32)), li
        assert np.array_equal(u32(v.values), vd.view(np.uint32)), li


def test_fma_adversarial_vectors_replay_exactly(monkeypatch):
    # every vector sits on an f32 rounding boundary of the scale where an
    # FMA-contracted sum of squares rounds the other way (make_adversarial.py)
    with np.load(GOLDEN_DIR / "adversarial_fma.npz") as z:
        v, codes, scales = z["v_in"], z["v_codes"], z["v_scales"]
    n = v.shape[2]
    g = pk.ModelGeometry(num_layers=1, kv_heads=1, head_dim=128, seq_len=n)
    t = pk.KvTensor(g, torch.from_numpy(v).cuda())
    pool = pk.build_pool(pk.KvDump(g, ((t, t),)), build_stats=False)
    _, vq = pool.layer_blocks(0)
    assert np.array_equal(vq.codes.cpu().numpy(), codes)
    assert np.array_equal(u32(vq.scales), scales.view(np.uint32))
    assert pool.replay_count >= n  # every one of them went through the fp64 replay
    # the warp-granular codec (codec.cu) replays through the same helper
    from paper_2604_24971_b200 import _lib

    monkeypatch.setenv("PKV_CODEC_PATH", "warp")
    _lib.reload_tuning()
    try:
        vq2 = pk.quantize_v(t)
        assert np.array_equal(vq2.codes.cpu().numpy(), codes)
        assert np.array_equal(u32(vq2.scales), scales.view(np.uint32))
    finally:
        monkeypatch.undo()
        _lib.reload_tuning()


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["f32", "bf16"])
def test_full_c3_every_layer_bit_exact(dtype):
    """configs[2] (the bench workload): L32 H8 d128 T4096, seed 0, all 32 layers."""
    L, H, D, T = 32, 8, 128, 4096
    g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
    host = O.synth_dump(L, H, D, T, seed=0)
    dump = device_dump(g, host, dtype)
    del host
    pool = pk.build_pool(dump, build_stats=False)
    want = check_pool_layers(pool, dump, list(range(L)))
    check_decoded(pool, want, [0, 15, 31], bits=16)
    check_decoded(pool, want, [7], bits=32)


def test_c4_sampled_layers_bit_exact():
    """configs[3] shape: L32 H8 d128 T7194 (a T that leaves partial tiles),
    one 32-layer build, layers 0 / 13 / 31 checked codes + decode."""
    L, H, D, T = 32, 8, 128, 7194
    g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
    host = O.synth_dump(L, H, D, T, seed=0)
    dump = device_dump(g, host, torch.bfloat16)
    del host
    pool = pk.build_pool(dump, build_stats=False)
    want = check_pool_layers(pool, dump, [0, 13, 31])
    check_decoded(pool, want, [0, 13, 31], bits=16)


def attention_case(T, agents=15, group=4, layers=2, k_mode="tensor", sign_seed=None, seed=5):
    from paper_2604_24971_b200 import attention as A

    H, D = 8, 128
    g = pk.ModelGeometry(num_layers=layers, kv_heads=H, head_dim=D, seq_len=T)
    host = O.synth_dump(layers, H, D, T, seed=seed)
    dump = device_dump(g, host, torch.bfloat16)
    pool = pk.build_pool(dump, build_stats=False, k_scale_mode=k_mode, sign_seed=sign_seed)
    li = layers - 1
    w = check_pool_layers(pool, dump, [li], k_mode=k_mode, sign_seed=sign_seed)[li]
    # oracle decode of the oracle's codes (independent of the device decode)
    kd, vd = O.decode_layer(w["k_codes"], w.get("k_scale", 0.0), w["v_codes"], w["v_scales"], 32,
                            sign_seed=sign_seed, k_block_scales=w.get("k_bscale"))
    gen = torch.Generator(device="cuda").manual_seed(seed)
    q = torch.randn(agents, H, group, D, device="cuda", generator=gen)
    cap = 16
    tail_len = torch.randint(0, cap + 1, (agents,), device="cuda", dtype=torch.int32, generator=gen)
    tk = torch.randn(agents, H, cap, D, device="cuda", generator=gen).bfloat16()
    tv = torch.randn(agents, H, cap, D, device="cuda", generator=gen).bfloat16()
    out = A.decode_attention(pool, li, q, tail_k=tk, tail_v=tv, tail_len=tail_len, softmax_scale=D ** -0.5,
                             out_dtype=torch.float32)
    tails_k = [tk[r, :, : int(tail_len[r])].float().cpu().numpy() for r in range(agents)]
    tails_v = [tv[r, :, : int(tail_len[r])].float().cpu().numpy() for r in range(agents)]
    want = O.attention_over_pool(q.cpu().numpy(), kd[0], vd[0], D ** -0.5, tails_k, tails_v)
    got = out.cpu().numpy().astype(np.float64)
    return np.abs(got - want).max() / np.abs(want).max()


@pytest.mark.parametrize("T", [4096, 7194], ids=["c3", "c4"])
def test_attention_at_bench_shapes_vs_oracle_decode(T):
    rel = attention_case(T)
    assert rel < 1e-3, rel


@pytest.mark.parametrize("k_mode,sign_seed", [("block32", None), ("tensor", 7), ("block32", 7)])
def test_attention_block32_keys_and_sign_diagonal(k_mode, sign_seed):
    rel = attention_case(1000, agents=5, k_mode=k_mode, sign_seed=sign_seed)
    assert rel < 1e-3, rel


@pytest.mark.parametrize("shape", [(8, 128, 4096, 15, 4), (32, 64, 1851, 5, 1), (8, 128, 300, 3, 4), (4, 64, 700, 9, 2)],
                         ids=lambda s: "h%d_d%d_t%d_a%d_g%d" % s)
@pytest.mark.parametrize("qmul", [1.0, 40.0], ids=["logits1", "logits40"])
def test_tensor_core_attention_matches_oracle_and_simt(monkeypatch, shape, qmul):
    """The mma.sync prefix kernel (default) against the fp64 oracle over the
    oracle's decode, at ordinary and at large logits (q x 40: the split-f16 Q
    keeps the logit error ~2^-22 relative), and against the fp32 CUDA-core
    kernel (PKV_ATTN_PATH=simt)."""
    from paper_2604_24971_b200 import _lib
    from paper_2604_24971_b200 import attention as A

    H, D, T, R, G = shape
    g = pk.ModelGeometry(num_layers=1, kv_heads=H, head_dim=D, seq_len=T)
    host = O.synth_dump(1, H, D, T, seed=17)
    dump = device_dump(g, host, torch.float32)
    pool = pk.build_pool(dump, build_stats=False)
    w = check_pool_layers(pool, dump, [0])[0]
    kd, vd = O.decode_layer(w["k_codes"], w["k_scale"], w["v_codes"], w["v_scales"], 32)
    gen = torch.Generator(device="cuda").manual_seed(3)
    q = torch.randn(R, H, G, D, device="cuda", generator=gen) * qmul
    want = O.attention_over_pool(q.cpu().numpy(), kd[0], vd[0], D ** -0.5)
    got = A.decode_attention(pool, 0, q, softmax_scale=D ** -0.5, out_dtype=torch.float32).cpu().numpy()
    rel = np.abs(got - want).max() / np.abs(want).max()
    assert rel < 1e-3, rel
    monkeypatch.setenv("PKV_ATTN_PATH", "simt")
    _lib.reload_tuning()
    try:
        simt = A.decode_attention(pool, 0, q, softmax_scale=D ** -0.5, out_dtype=torch.float32).cpu().numpy()
    finally:
        monkeypatch.undo()
        _lib.reload_tuning()
    assert np.abs(simt - want).max() / np.abs(want).max() < 1e-3
    assert np.abs(got - simt).max() / np.abs(want).max() < 1e-3


@pytest.mark.parametrize("q_len", [3, 8])
def test_multi_token_step_is_causal_over_the_tail(q_len):
    """A multi-token step on top of the pool (a prompt suffix, q_len new tokens
    per agent) through the kernel: position i sees the prefix and the tail up
    to its own token; compared with an fp64 softmax per position over the
    oracle's decode (no per-agent prefix copy)."""
    from paper_2604_24971_b200 import attention as A

    H, D, T, R, G = 8, 128, 700, 3, 4
    g = pk.ModelGeometry(num_layers=1, kv_heads=H, head_dim=D, seq_len=T)
    host = O.synth_dump(1, H, D, T, seed=23)
    dump = device_dump(g, host, torch.float32)
    pool = pk.build_pool(dump, build_stats=False)
    w = check_pool_layers(pool, dump, [0])[0]
    kd, vd = O.decode_layer(w["k_codes"], w["k_scale"], w["v_codes"], w["v_scales"], 32)
    gen = torch.Generator(device="cuda").manual_seed(q_len)
    cap = 32
    old = torch.tensor([0, 5, 11], dtype=torch.int32, device="cuda")  # tail tokens before this step
    tail_len = old + q_len
    tk = torch.randn(R, H, cap, D, device="cuda", generator=gen).bfloat16()
    tv = torch.randn(R, H, cap, D, device="cuda", generator=gen).bfloat16()
    q = torch.randn(R, H, G * q_len, D, device="cuda", generator=gen)  # row = g * q_len + i
    out = A.decode_attention(pool, 0, q, tail_k=tk, tail_v=tv, tail_len=tail_len, softmax_scale=D ** -0.5,
                             out_dtype=torch.float32, q_len=q_len).cpu().numpy()
    qh = q.cpu().numpy().reshape(R, H, G, q_len, D)
    worst = 0.0
    for i in range(q_len):
        n_i = [int(old[r]) + i + 1 for r in range(R)]
        tails_k = [tk[r, :, :n_i[r]].float().cpu().numpy() for r in range(R)]
        tails_v = [tv[r, :, :n_i[r]].float().cpu().numpy() for r in range(R)]
        want = O.attention_over_pool(qh[:, :, :, i], kd[0], vd[0], D ** -0.5, tails_k, tails_v)
        got = out.reshape(R, H, G, q_len, D)[:, :, :, i]
        worst = max(worst, np.abs(got - want).max() / np.abs(want).max())
    assert worst < 1e-3, worst


@pytest.mark.parametrize("seed", range(int(os.environ.get("PKV_ATTN_STRESS_SEEDS", "6"))))
def test_random_attention_shapes_vs_oracle(seed):
    """Random decode-attention problems through the tensor-core kernel: KV
    heads, head_dim 64/128, ragged T (partial tiles, T below one tile), agent
    and group counts (row tiles of 16/32/64, partial), bf16/f32 queries, tails
    with random lengths, block32 keys and the sign diagonal; within 1e-3 of an
    fp64 softmax over the oracle's decode. PKV_ATTN_STRESS_SEEDS widens it."""
    from paper_2604_24971_b200 import attention as A

    rng = np.random.default_rng(900 + seed)
    D = int(rng.choice([64, 128]))
    H = int(rng.choice([1, 2, 4, 8]))
    T = int(rng.integers(1, 3000))
    R = int(rng.integers(1, 17))
    G = int(rng.choice([1, 2, 4, 8]))
    k_mode = "block32" if seed % 3 == 2 else "tensor"
    sign_seed = 3 if seed % 4 == 1 else None
    qdt = torch.bfloat16 if seed % 2 else torch.float32
    g = pk.ModelGeometry(num_layers=1, kv_heads=H, head_dim=D, seq_len=T)
    host = O.synth_dump(1, H, D, T, seed=seed)
    dump = device_dump(g, host, torch.float32)
    pool = pk.build_pool(dump, build_stats=False, k_scale_mode=k_mode, sign_seed=sign_seed)
    w = check_pool_layers(pool, dump, [0], k_mode=k_mode, sign_seed=sign_seed)[0]
    kd, vd = O.decode_layer(w["k_codes"], w.get("k_scale", 0.0), w["v_codes"], w["v_scales"], 32,
                            sign_seed=sign_seed, k_block_scales=w.get("k_bscale"))
    gen = torch.Generator(device="cuda").manual_seed(seed)
    q = torch.randn(R, H, G, D, device="cuda", generator=gen).to(qdt)
    cap = int(rng.integers(0, 24))
    kw = {}
    tails_k = tails_v = None
    if cap:
        tail_len = torch.randint(0, cap + 1, (R,), device="cuda", dtype=torch.int32, generator=gen)
        tk = torch.randn(R, H, cap, D, device="cuda", generator=gen).bfloat16()
        tv = torch.randn(R, H, cap, D, device="cuda", generator=gen).bfloat16()
        kw = dict(tail_k=tk, tail_v=tv, tail_len=tail_len)
        tails_k = [tk[r, :, : int(tail_len[r])].float().cpu().numpy() for r in range(R)]
        tails_v = [tv[r, :, : int(tail_len[r])].float().cpu().numpy() for r in range(R)]
    out = A.decode_attention(pool, 0, q, softmax_scale=D ** -0.5, out_dtype=torch.float32, **kw)
    want = O.attention_over_pool(q.float().cpu().numpy(), kd[0], vd[0], D ** -0.5, tails_k, tails_v)
    rel = np.abs(out.cpu().numpy().astype(np.float64) - want).max() / np.abs(want).max()
    assert rel < 1e-3, (rel, D, H, T, R, G, k_mode, sign_seed, cap)
