"""Multi-GPU SharedKVPool: shard the write side, replicate the packed pool.

SURVEY §8(e): every layer (and every KV head) of the pool is independent
except for the per-tensor key scale, one max per layer (keyquant.py:55).

* `build_pool_sharded` — each rank compresses a contiguous slice of layers
  (no collective inside the compress), then ONE `all_gather_into_tensor` per
  pool field over NCCL assembles the whole packed pool on every rank. The
  gathered bytes are O(1) in agents (C4: 331.5 MB total).
* `partition_agents` — agents are split over ranks; each rank decodes its
  agents against its local replica, so decode needs no per-step collective.
* `decode_attention_head_sharded` — the alternative the north star asks for
  "where a shard boundary requires it": the pool stays sharded by KV head,
  each rank attends over its heads and the outputs are all-gathered.

Host logic here is backend-agnostic (NCCL on GPUs, gloo in the CPU tests).
"""

from __future__ import annotations

from typing import Callable

import torch
import torch.distributed as dist

from . import _codec
from .model import KvDump, KvTensor, ModelGeometry
from .pool import SharedPool, _Arena, _device_inputs, _encode_layers, pool_from_arena, raise_for_status
from .valuequant import GAUSSIAN_3BIT, Codebook



def _world(group) -> tuple[int, int]:
    if not dist.is_available() or not dist.is_initialized():
        return 1, 0
    return dist.get_world_size(group), dist.get_rank(group)


def layer_shard(num_layers: int, world: int, rank: int) -> range:
    """Contiguous, balanced slice of layers owned by `rank` (first ranks take the remainder)."""
    if world < 1 or not 0 <= rank < world:
        raise ValueError(f"bad rank {rank} of world {world}")
    base, extra = divmod(num_layers, world)
    start = rank * base + min(rank, extra)
    return range(start, start + base + (1 if rank < extra else 0))


def partition_agents(num_agents: int, world: int, rank: int) -> list[int]:
    """Agent ids served by `rank` (C4: 15 agents over 8 GPUs -> 2,2,2,2,2,2,2,1)."""
    return list(layer_shard(num_agents, world, rank))


def _all_gather_rows(local: torch.Tensor, rows_max: int, group) -> torch.Tensor:
    """Gather [rows_r, ...] from every rank as [world, rows_max, ...] (padded)."""
    world, _ = _world(group)
    padded = local
    if local.shape[0] != rows_max:
        padded = torch.zeros((rows_max,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        padded[:local.shape[0]] = local
    padded = padded.contiguous()
    if world == 1:
        return padded.unsqueeze(0)
    if dist.get_backend(group) == "nccl":
        out = torch.empty((world * rows_max,) + tuple(local.shape[1:]), dtype=local.dtype, device=local.device)
        dist.all_gather_into_tensor(out, padded, group=group)
        return out.view((world, rows_max) + tuple(local.shape[1:]))
    parts = [torch.empty_like(padded) for _ in range(world)]
    dist.all_gather(parts, padded, group=group)
    return torch.stack(parts)


def gather_arena(local: _Arena, num_layers: int, group=None) -> _Arena:
    """Assemble the full [L, layer_bytes] pool from every rank's layer slice
    with ONE all-gather of the layer-major arena (pool._Arena): rank r's rows
    are its layers' codes, packed values, scales and status words, already
    back to back, so the collective moves exactly the packed pool bytes."""
    world, _ = _world(group)
    local.status_row.copy_(local.status)  # status words travel inside the rows
    rows_max = len(layer_shard(num_layers, world, 0))
    g = _all_gather_rows(local.flat, rows_max, group)  # [world, rows_max, layer_bytes]
    sizes = [len(layer_shard(num_layers, world, r)) for r in range(world)]
    if all(sz == rows_max for sz in sizes):
        flat = g.view(world * rows_max, local.layer_bytes)  # no compaction needed
    else:
        flat = torch.cat([g[r, :sizes[r]] for r in range(world)], dim=0).contiguous()
    full = _Arena.like(local, flat)
    full.replay = local.replay  # this rank's fp64-replay count
    return full


def build_pool_sharded(dump: KvDump, codebook: Codebook = GAUSSIAN_3BIT, sign_seed: int | None = None, *,
                       k_scale_mode: str = "tensor", group=None, device=None,
                       encode_fn: Callable | None = None, check: bool = True) -> SharedPool:
    """build_pool (pool.py:258-293) with the layers spread over the ranks of `group`.

    Each rank reads only its own layers of `dump`; the returned pool is the
    complete, bit-identical pool on every rank. `encode_fn` (default: the
    sm_100a encoder) is injectable so the collective plumbing can be tested
    on CPU ranks.
    """
    g: ModelGeometry = dump.geometry
    world, rank = _world(group)
    mine = layer_shard(g.num_layers, world, rank)
    enc = encode_fn or _encode_layers
    ks = [dump.layers[i][0] for i in mine]
    vs = [dump.layers[i][1] for i in mine]
    if device is None and torch.cuda.is_available():
        device = torch.device("cuda", torch.cuda.current_device())
    if ks:
        _, _, arena = enc(ks, vs, g, codebook, sign_seed, k_scale_mode, device=device, check=False)
    else:  # more ranks than layers: contribute an empty slice (on the device NCCL gathers from)
        arena = _Arena(g, 0, k_scale_mode, device)
    full = gather_arena(arena, g.num_layers, group)
    # Data faults (non-finite input, fp16 scale overflow) are checked on the
    # GATHERED status words, so every rank sees every rank's faults and raises
    # the same exception after the collective; raising before it would leave
    # the healthy ranks blocked in all_gather.
    if check:
        raise_for_status(full.status)
    return pool_from_arena(full, g, codebook, sign_seed, k_scale_mode)


def all_reduce_layer_max(local_max_bits: torch.Tensor, group=None) -> torch.Tensor:
    """Per-layer max|K| across ranks when a layer's keys are split by head or
    token: |K| bit patterns order like the floats, so a MAX
    reduction of the int32 bit patterns is exact."""
    world, _ = _world(group)
    t = local_max_bits.to(torch.int32).clone()
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX, group=group)
    return t


def head_shard(kv_heads: int, world: int, rank: int) -> range:
    return layer_shard(kv_heads, world, rank)


def head_geometry(g: ModelGeometry, heads: range) -> ModelGeometry:
    return ModelGeometry(num_layers=g.num_layers, kv_heads=len(heads), head_dim=g.head_dim, seq_len=g.seq_len,
                         batch=g.batch, baseline_bits=g.baseline_bits)


def head_slice(t: KvTensor, heads: range, g_local: ModelGeometry) -> KvTensor:
    """[B, H, T, D] -> [B, len(heads), T, D]: the KV heads this rank owns
    (a view for batch 1, where a head range is contiguous)."""
    v = t.values[:, heads.start:heads.stop]
    return KvTensor(g_local, v if v.is_contiguous() else v.contiguous())


def local_key_max(ks, device) -> torch.Tensor:
    """int32 [L]: max|K| bit pattern of each layer's local key slice (pkv_k_absmax)."""
    dev = _codec.require_device(device if device is not None else ks[0].values.device)
    vals = _device_inputs(ks, dev)
    out = torch.empty(len(vals), dtype=torch.int32, device=dev)
    return _codec.k_absmax(vals, out, dev)


def _or_status_over_ranks(status: torch.Tensor, group) -> torch.Tensor:
    world, _ = _world(group)
    if world == 1:
        return status
    parts = _all_gather_rows(status.view(1, -1), 1, group)  # [world, 1, L]
    acc = parts[0, 0].clone()
    for r in range(1, world):
        acc |= parts[r, 0]
    return acc


def build_pool_head_sharded(dump: KvDump, codebook: Codebook = GAUSSIAN_3BIT, sign_seed: int | None = None, *,
                            k_scale_mode: str = "tensor", group=None, device=None, heads: range | None = None,
                            reduce_max: Callable | None = None, absmax_fn: Callable | None = None,
                            encode_fn: Callable | None = None, check: bool = True) -> SharedPool:
    """build_pool (pool.py:258-293) for the KV heads `heads` (default: this
    rank's head_shard) of every layer -- the head-sharded alternative of
    SURVEY §8(e): the pool stays split by KV head across the ranks.

    The only cross-rank dependency of the codec is the per-tensor key scale,
    f32(max|K| / 127) over the WHOLE layer (keyquant.py:55-60): each rank
    takes the max of its heads (pkv_k_absmax), the ranks MAX-reduce the bit
    patterns (all_reduce_layer_max; `reduce_max` overrides, e.g. a
    precomputed global max), and pkv_encode uses the reduced maxima
    (k_layer_max), so every rank's codes equal the single-GPU build's codes
    for its heads, bit for bit. Block32 keys and values need no collective.
    Data faults are OR-ed over the ranks before raising, so all ranks agree.
    Returns a pool over the local heads (geometry kv_heads = len(heads));
    `pool.head_range` / `pool.full_geometry` describe the slice.
    """
    g: ModelGeometry = dump.geometry
    world, rank = _world(group)
    hs = heads if heads is not None else head_shard(g.kv_heads, world, rank)
    if len(hs) == 0:
        raise ValueError(f"rank {rank} owns no KV heads ({g.kv_heads} heads over {world} ranks)")
    if g.batch != 1 and (hs.start, hs.stop) != (0, g.kv_heads):
        raise ValueError("head sharding needs batch 1 (a head range is then contiguous)")
    gl = head_geometry(g, hs)
    ks = [head_slice(k, hs, gl) for k, _ in dump.layers]
    vs = [head_slice(v, hs, gl) for _, v in dump.layers]
    if device is None and torch.cuda.is_available():
        device = torch.device("cuda", torch.cuda.current_device())
    kmax = None
    if k_scale_mode == "tensor":
        local = (absmax_fn or local_key_max)(ks, device)
        kmax = reduce_max(local) if reduce_max is not None else all_reduce_layer_max(local, group)
    _, _, arena = (encode_fn or _encode_layers)(ks, vs, gl, codebook, sign_seed, k_scale_mode, device=device,
                                                check=False, k_layer_max=kmax)
    status = _or_status_over_ranks(arena.status, group)
    if check:
        raise_for_status(status)
    pool = pool_from_arena(arena, gl, codebook, sign_seed, k_scale_mode)
    pool.head_range = hs
    pool.full_geometry = g
    return pool


def decode_attention_head_sharded(attend: Callable[[torch.Tensor], torch.Tensor], q: torch.Tensor,
                                  kv_heads: int, group=None) -> torch.Tensor:
    """Head-sharded decode attention: rank r owns KV heads head_shard(r);
    `attend(q_local)` runs the pool attention for those heads and returns
    [rows, heads_r, group, d]; the result is all-gathered along the head dim.
    q: [rows, kv_heads, group, d] (every rank holds all queries)."""
    world, rank = _world(group)
    hs = head_shard(kv_heads, world, rank)
    local = attend(q[:, hs.start:hs.stop].contiguous())
    if world == 1:
        return local
    hmax = len(head_shard(kv_heads, world, 0))
    moved = local.transpose(0, 1).contiguous()  # [heads_r, rows, group, d]
    g = _all_gather_rows(moved, hmax, group)
    parts = [g[r, :len(head_shard(kv_heads, world, r))] for r in range(world)]
    return torch.cat(parts, dim=0).transpose(0, 1).contiguous()


__all__ = [
    "all_reduce_layer_max", "build_pool_head_sharded", "build_pool_sharded", "decode_attention_head_sharded",
    "head_geometry", "head_slice", "local_key_max",
    "gather_arena", "head_shard", "layer_shard", "partition_agents",
]
