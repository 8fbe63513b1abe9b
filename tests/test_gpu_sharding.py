"""Head-sharded and layer-sharded pools on one GPU, through the real kernels.

SURVEY §8(e): a layer's KV heads can live on different GPUs; the only
cross-head dependency of the codec is the per-tensor key scale
f32(max|K| / 127) over the whole layer (kvpool/keyquant.py:55-60). Here the
shards are built one after the other in one process with the MAX of their
pkv_k_absmax results standing in for the all-reduce (the multi-rank plumbing
itself is covered by tests/test_parallel_cpu.py over gloo): every shard's
codes must equal the single-GPU build's codes for its heads, bit for bit.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2604_24971_b200 as pk
from oracle import kvpool_oracle as O
from paper_2604_24971_b200 import parallel

pytestmark = pytest.mark.gpu


def u32(t):
    return t.detach().float().cpu().numpy().view(np.uint32)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16], ids=["f32", "bf16"])
@pytest.mark.parametrize("count", [4096 * 128, 1000 * 64 + 8, 77])  # vector path, ragged, scalar path
def test_k_absmax_matches_torch(dtype, count):
    gen = torch.Generator(device="cuda").manual_seed(count)
    xs = [(torch.randn(count, device="cuda", generator=gen) * (li + 1)).to(dtype) for li in range(3)]
    xs[1][count // 2] = -1e4  # a negative peak
    out = parallel.local_key_max([pk.KvTensor(pk.ModelGeometry(1, 1, 1, count), x.view(1, 1, count, 1))
                                  for x in xs], torch.device("cuda"))
    want = [float(x.float().abs().max()) for x in xs]
    assert out.view(torch.float32).cpu().tolist() == want


def test_k_absmax_flags_nan():
    x = torch.randn(1, 1, 64, 64, device="cuda")
    x[0, 0, 3, 5] = float("nan")
    out = parallel.local_key_max([pk.KvTensor(pk.ModelGeometry(1, 1, 64, 64), x)], torch.device("cuda"))
    assert int(out[0]) > 0x7F800000  # above +inf: the encode reports a non-finite layer


@pytest.mark.parametrize("mode", ["tensor", "block32"])
def test_head_sharded_world1_is_build_pool(mode):
    g = pk.ModelGeometry(num_layers=3, kv_heads=8, head_dim=128, seq_len=300)
    dump = pk.synth_gaussian_dump(g, seed=21, device="cuda", dtype=torch.bfloat16, generator="torch")
    a = pk.build_pool(dump, k_scale_mode=mode, build_stats=False)
    b = parallel.build_pool_head_sharded(dump, k_scale_mode=mode)
    assert b.head_range == range(0, 8)
    for i in range(3):
        (ka, va), (kb, vb) = a.layer_blocks(i), b.layer_blocks(i)
        assert torch.equal(ka.codes, kb.codes) and torch.equal(va.packed, vb.packed)
        assert torch.equal(va.scales, vb.scales)
        if mode == "tensor":
            assert ka.scale == kb.scale
        else:
            assert torch.equal(ka.block_scales, kb.block_scales)


@pytest.mark.parametrize("split", [(0, 3, 8), (0, 4, 8), (0, 1, 2, 5, 8)])
def test_head_shards_with_reduced_max_equal_the_whole_pool(split):
    L, H, D, T = 4, 8, 128, 515
    g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
    host = O.synth_dump(L, H, D, T, seed=7)
    # make the layer max sit in different heads per layer
    for li, (k, _) in enumerate(host):
        k[0, (3 * li) % H, 11, 5] = 0.9 + 0.1 * li
    dump = pk.KvDump(g, tuple((pk.KvTensor(g, torch.from_numpy(k).cuda()), pk.KvTensor(g, torch.from_numpy(v).cuda()))
                              for k, v in host))
    whole = pk.build_pool(dump, build_stats=False)
    shards = [range(a, b) for a, b in zip(split[:-1], split[1:])]
    gls = [parallel.head_geometry(g, hs) for hs in shards]
    local = [parallel.local_key_max([parallel.head_slice(k, hs, gl) for k, _ in dump.layers], torch.device("cuda"))
             for hs, gl in zip(shards, gls)]
    gmax = torch.stack(local).max(dim=0).values  # what all_reduce_layer_max returns on every rank
    n_head = T * D
    for hs, lm in zip(shards, local):
        p = parallel.build_pool_head_sharded(dump, heads=hs, reduce_max=lambda m: gmax)
        for li in range(L):
            (kw, vw), (ks, vs) = whole.layer_blocks(li), p.layer_blocks(li)
            assert ks.scale == kw.scale
            assert torch.equal(ks.codes, kw.codes[:, hs.start:hs.stop])
            assert torch.equal(vs.scales, vw.scales[:, hs.start:hs.stop])
            pb = 3 * n_head // 8
            assert torch.equal(vs.packed[: len(hs) * pb], vw.packed[hs.start * pb: hs.stop * pb])
        # without the reduction a shard that lacks the layer max gets another scale
        if not torch.equal(lm, gmax):
            p2 = parallel.build_pool_head_sharded(dump, heads=hs, reduce_max=lambda m: m)
            assert any(p2.layer_blocks(li)[0].scale != whole.layer_blocks(li)[0].scale for li in range(L))


def test_head_sharded_attention_gathers_to_the_whole_pool_result():
    from paper_2604_24971_b200.attention import decode_attention

    L, H, D, T, R, G = 2, 8, 128, 1000, 5, 4
    g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
    dump = pk.synth_gaussian_dump(g, seed=5, device="cuda", dtype=torch.bfloat16, generator="torch")
    whole = pk.build_pool(dump, build_stats=False)
    q = torch.randn(R, H, G, D, device="cuda")
    want = decode_attention(whole, 1, q, softmax_scale=D ** -0.5, out_dtype=torch.float32)
    shards = [range(0, 3), range(3, 8)]
    local = [parallel.local_key_max([parallel.head_slice(k, hs, parallel.head_geometry(g, hs))
                                     for k, _ in dump.layers], torch.device("cuda")) for hs in shards]
    gmax = torch.stack(local).max(dim=0).values
    outs = []
    for hs in shards:
        p = parallel.build_pool_head_sharded(dump, heads=hs, reduce_max=lambda m: gmax)
        outs.append(decode_attention(p, 1, q[:, hs.start:hs.stop].contiguous(), softmax_scale=D ** -0.5,
                                     out_dtype=torch.float32))
    got = torch.cat(outs, dim=1)
    rel = float((got - want).abs().max() / want.abs().max())
    assert rel < 1e-5, rel
