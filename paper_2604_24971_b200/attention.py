"""Shared-pool GQA decode attention (pkv_decode_attention in libpolykv.so).

All agents' query rows that share a KV head attend to the packed pool in one
launch; no per-agent K/V copy is ever written to HBM. Each agent may carry a
private bf16 tail (tokens generated after the shared prefix).
"""

from __future__ import annotations

import torch

from . import _codec
from ._lib import PKV_BF16, PKV_F32, check, load
from .keyquant import K_MODES
from .pool import SharedPool

_DT = {torch.float32: PKV_F32, torch.bfloat16: PKV_BF16}


def decode_attention(pool: SharedPool, layer: int, q: torch.Tensor, *, tail_k: torch.Tensor | None = None,
                     tail_v: torch.Tensor | None = None, tail_len: torch.Tensor | None = None,
                     softmax_scale: float | None = None, out: torch.Tensor | None = None,
                     out_dtype: torch.dtype | None = None, workspace: torch.Tensor | None = None,
                     q_len: int = 1) -> torch.Tensor:
    """softmax(q k^T * scale) v over [pool prefix ; agent tail] for one layer.

    q: [agents, kv_heads, group, head_dim] f32/bf16. One decode token per
    agent (q_len = 1), or q_len new tokens per agent: then group = G * q_len,
    row g is position g % q_len, and position i sees the prefix plus the tail
    up to its own token (tail_len counts all q_len new tokens) -- a causal
    multi-token step with no per-agent copy of the prefix.
    tail_k/tail_v: [agents, kv_heads, tail_cap, head_dim] bf16; tail_len: int32 [agents].
    Returns [agents, kv_heads, group, head_dim].
    """
    g = pool.geometry
    if g.batch != 1:
        raise ValueError("decode attention reads a batch-1 shared prefix pool")
    R, H, G, D = q.shape
    if H != g.kv_heads or D != g.head_dim:
        raise ValueError(f"q shape {tuple(q.shape)} does not match pool geometry {g}")
    if q_len < 1 or G % q_len:
        raise ValueError(f"q_len {q_len} must divide the {G} rows per KV head")
    kq, vq = pool.layer_blocks(layer)
    dev = pool.device
    q = q.contiguous()
    if q.dtype not in _DT:
        q = q.float()
    od = out_dtype or q.dtype
    if out is None:
        out = torch.empty((R, H, G, D), dtype=od, device=dev)
    lib = load()
    need = lib.pkv_attention_workspace_bytes(R, H, G, D, g.seq_len)
    if workspace is None or workspace.numel() * workspace.element_size() < need:
        workspace = torch.empty((need + 3) // 4, dtype=torch.float32, device=dev)
    if tail_len is not None:
        if tail_k is None or tail_v is None:
            raise ValueError("tail_len needs tail_k and tail_v")
        if tail_k.dim() != 4 or tuple(tail_k.shape[:2]) != (R, H) or tail_k.shape[3] != D:
            raise ValueError(f"tail_k shape {tuple(tail_k.shape)} is not [{R}, {H}, cap, {D}]")
        if tail_v.shape != tail_k.shape:
            raise ValueError(f"tail_v shape {tuple(tail_v.shape)} != tail_k shape {tuple(tail_k.shape)}")
        if tail_len.numel() != R:
            raise ValueError(f"tail_len has {tail_len.numel()} entries for {R} agents")
        for t in (tail_k, tail_v, tail_len):
            if t.device != dev:
                raise ValueError(f"tail tensors must be on {dev}, got {t.device}")
        tail_k = tail_k.to(torch.bfloat16).contiguous()
        tail_v = tail_v.to(torch.bfloat16).contiguous()
        tail_len = tail_len.to(dtype=torch.int32).contiguous()
        cap = tail_k.shape[2]  # the kernel clamps tail_len[r] to cap
    else:
        cap = 0
    scale = float(softmax_scale if softmax_scale is not None else D ** -0.5)
    with torch.cuda.device(dev):  # the library launches on the current device
        rc = lib.pkv_decode_attention(
            R, H, G, D, g.seq_len, _DT[q.dtype], q.data_ptr(), K_MODES[kq.mode], kq.codes.data_ptr(),
            kq.scale_t.data_ptr() if kq.mode == "tensor" else None,
            kq.block_scales.data_ptr() if kq.mode == "block32" else None,
            vq.packed.data_ptr(), vq.scales.data_ptr(), _codec.centroid_array(pool.codebook.centroids),
            _codec.sign_word_array(pool.sign_seed, D),
            tail_k.data_ptr() if tail_len is not None else None,
            tail_v.data_ptr() if tail_len is not None else None,
            tail_len.data_ptr() if tail_len is not None else None, cap, q_len, scale, _DT[out.dtype],
            out.data_ptr(), workspace.data_ptr(), workspace.numel() * workspace.element_size(),
            _codec.stream_ptr(dev))
    check(rc, "pkv_decode_attention")
    return out

