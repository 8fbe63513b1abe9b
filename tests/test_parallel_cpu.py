"""Multi-rank host logic of parallel.py on CPU (gloo, world_size 2).

The sm_100a encoder needs a GPU, so these tests inject a deterministic CPU
stand-in for it: what is under test is the sharding plan, the all-gather of
the packed pool fields and their reassembly into one pool, the MAX reduction
of per-layer key maxima and the head-sharded output gather.
"""

from __future__ import annotations

import os
import socket

import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import paper_2604_24971_b200 as pk
from paper_2604_24971_b200 import parallel
from paper_2604_24971_b200.pool import _Arena


def test_layer_and_agent_partitions():
    assert [list(parallel.layer_shard(32, 8, r)) for r in (0, 7)] == [[0, 1, 2, 3], [28, 29, 30, 31]]
    shards = [parallel.layer_shard(5, 2, r) for r in range(2)]
    assert [list(s) for s in shards] == [[0, 1, 2], [3, 4]]
    sizes = [len(parallel.partition_agents(15, 8, r)) for r in range(8)]
    assert sizes == [2, 2, 2, 2, 2, 2, 2, 1] and sum(sizes) == 15
    assert sorted(a for r in range(8) for a in parallel.partition_agents(15, 8, r)) == list(range(15))
    assert [len(parallel.layer_shard(3, 4, r)) for r in range(4)] == [1, 1, 1, 0]
    with pytest.raises(ValueError):
        parallel.layer_shard(4, 2, 2)


def fake_encode(ks, vs, g, codebook, sign_seed, k_scale_mode, device=None, check=False, k_layer_max=None):
    """Deterministic CPU stand-in for the sm_100a encoder (same arena layout;
    the key scale honours external per-layer maxima like pkv_encode)."""
    L = len(ks)
    a = _Arena(g, L, k_scale_mode, torch.device("cpu"))
    n, vecs = g.elements_per_tensor, g.vectors_per_tensor
    a.k_codes.zero_()
    a.v_packed.zero_()
    a.v_scales.zero_()
    for i, (k, v) in enumerate(zip(ks, vs)):
        kv = k.values.reshape(-1).float()
        a.k_codes[i, :n] = (kv * 50).round().clamp(-127, 127).to(torch.int8)
        peak = kv.abs().max() if k_layer_max is None else k_layer_max[i:i + 1].view(torch.float32)[0]
        a.k_scale[i] = (peak.to(torch.float64) / 127).to(torch.float32)
        vv = v.values.reshape(-1).float()
        a.v_packed[i, :3 * n // 8] = (vv[: 3 * n // 8] * 1000).abs().round().remainder(256).to(torch.uint8)
        a.v_scales[i, :vecs] = v.values.reshape(vecs, -1).float().pow(2).mean(-1).sqrt()
        if not bool(torch.isfinite(kv).all()):
            a.status[i] |= 1  # PKV_FLAG_K_NONFINITE, as the device encoder reports it
    return None, None, a


def _cpu_absmax(ks, device):
    """Test stand-in for pkv_k_absmax: max|K| bit pattern per layer (int32)."""
    return torch.stack([k.values.abs().max().reshape(1).view(torch.int32)[0] for k in ks])


def _geometry():
    return pk.ModelGeometry(num_layers=5, kv_heads=2, head_dim=16, seq_len=8)


def _dump(g):
    gen = torch.Generator().manual_seed(3)
    layers = tuple((pk.KvTensor(g, torch.randn(g.tensor_shape, generator=gen)),
                    pk.KvTensor(g, torch.randn(g.tensor_shape, generator=gen))) for _ in range(g.num_layers))
    return pk.KvDump(g, layers)


def _worker(rank, world, port, q):
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        g = _geometry()
        dump = _dump(g)
        pool = parallel.build_pool_sharded(dump, encode_fn=fake_encode)
        _, _, ref = fake_encode([k for k, _ in dump.layers], [v for _, v in dump.layers], g, None, None, "tensor")
        ok = all(torch.equal(getattr(pool._arena, f), getattr(ref, f)) for f in ("k_codes", "k_scale", "v_packed",
                                                                                  "v_scales"))
        ok = ok and pool.num_layers == 5 and pool.sealed
        ok = ok and all(torch.equal(pool.layer_blocks(i)[0].codes.reshape(-1), ref.k_codes[i, :g.elements_per_tensor])
                        for i in range(5))
        # per-layer key maxima split across ranks: MAX of the f32 bit patterns
        local = torch.tensor([[1.5, 0.25, 3.0], [0.75, 2.5, 1.0]][rank]).view(torch.int32)
        red = parallel.all_reduce_layer_max(local).view(torch.float32)
        ok = ok and torch.equal(red, torch.tensor([1.5, 2.5, 3.0]))
        # head-sharded attention: each rank "attends" over its KV heads only
        qs = torch.arange(2 * 3 * 2 * 4, dtype=torch.float32).view(2, 3, 2, 4)
        out = parallel.decode_attention_head_sharded(lambda ql: ql * 2, qs, kv_heads=3)
        ok = ok and torch.equal(out, qs * 2)
        # a data fault in a layer only rank 1 encodes: EVERY rank raises the
        # reference's GeometryError after the collective (none hangs in it)
        bad = _dump(g)
        bad.layers[4][0].values[0, 1, 2, 3] = float("nan")
        try:
            parallel.build_pool_sharded(bad, encode_fn=fake_encode)
            ok = False
        except pk.GeometryError as exc:
            ok = ok and "NaN or Inf" in str(exc) and "layer 4" in str(exc)
        # head-sharded pool with the real head slicing: rank r keeps heads
        # head_shard(3, 2, r); the per-layer key max is MAX-reduced over the
        # ranks, so both ranks' scales are the WHOLE layer's f32(max|K|/127)
        g3 = pk.ModelGeometry(num_layers=2, kv_heads=3, head_dim=16, seq_len=8)
        d3 = _dump(g3)
        hp = parallel.build_pool_head_sharded(d3, encode_fn=fake_encode, absmax_fn=_cpu_absmax)
        hs = parallel.head_shard(3, 2, rank)
        ok = ok and hp.head_range == hs and hp.geometry.kv_heads == len(hs)
        for li in range(2):
            whole = d3.layers[li][0].values.abs().max().to(torch.float64) / 127
            ok = ok and hp.layer_blocks(li)[0].scale == float(whole.to(torch.float32))
            mine = d3.layers[li][0].values[:, hs.start:hs.stop].reshape(-1)
            ok = ok and torch.equal(hp.layer_blocks(li)[0].codes.reshape(-1), (mine * 50).round().clamp(-127, 127)
                                    .to(torch.int8))
        q_ok = ok
    except Exception as exc:  # noqa: BLE001
        q_ok = repr(exc)
    finally:
        dist.destroy_process_group()
    q.put((rank, q_ok))


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_sharded_build_gathers_the_whole_pool_on_every_rank():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    results = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
    assert results == {0: True, 1: True}, results


def test_single_process_is_a_plain_build():
    g = _geometry()
    dump = _dump(g)
    pool = parallel.build_pool_sharded(dump, encode_fn=fake_encode)
    _, _, ref = fake_encode([k for k, _ in dump.layers], [v for _, v in dump.layers], g, None, None, "tensor")
    assert torch.equal(pool._arena.k_codes, ref.k_codes)
    assert pool.packed_payload_nbytes() == sum(kq.payload_nbytes + vq.packed_payload_nbytes
                                               for kq, vq in (pool.layer_blocks(i) for i in range(5)))
