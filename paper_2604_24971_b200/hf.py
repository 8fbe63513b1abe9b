"""Inject a SharedKVPool into a transformers model (kvbridge/hfcache.py on B200).

The reference rebuilds a per-agent `DynamicCache` from decompressed f32
tensors (`kvbridge/hfcache.py:58-67`, called from `evaluator.py:112-132`), so
every agent owns a full copy of the prefix K/V and every decode step
re-concatenates it (`transformers/cache_utils.py` `DynamicLayer.update`).

Two injection modes:

* ``build_cache(view, mode="materialize")`` — the reference semantics: a
  real `DynamicCache` whose layers are filled by ONE `pkv_decode` launch for
  all layers (bit-identical to `AgentCacheView.get_kv_for_layer`), cast to
  the model dtype.
* ``build_cache(view, mode="stream")`` — a `PooledCache`: every layer keeps
  a reference to the shared packed pool plus a small per-agent bf16 tail for
  the tokens generated after the prefix. Attention for those layers runs the
  `"polykv"` attention function (registered in transformers'
  `AttentionInterface`), which calls `pkv_decode_attention` over the packed
  pool directly: no per-agent K/V copy ever exists in HBM.

Agents of one batch share the prefix and advance in lockstep (the PolyKV
setting, `evaluator.py:191-212`), so there is no padding inside a batch.
"""

from __future__ import annotations

from typing import Sequence

import torch
from transformers import DynamicCache
from transformers.cache_utils import Cache, CacheLayerMixin
from transformers.modeling_utils import AttentionInterface

from .attention import decode_attention
from .pool import AgentCacheView, SharedPool

ATTN_IMPLEMENTATION = "polykv"


class CacheLayoutError(TypeError):
    """The model returned a past_key_values layout this bridge cannot read (hfcache.py:17-18)."""


def cache_layers(past_key_values) -> list[tuple[torch.Tensor, torch.Tensor]]:
    """Per-layer (K, V) tensors of a prefill cache, left on their device.

    Same layouts as the reference (`hfcache.py:32-55`: transformers 5
    `layers`, 4.x `key_cache`/`value_cache`, legacy tuples) but without the
    f32 CPU copy — the pool is built straight from the device tensors.
    """
    if past_key_values is None:
        raise CacheLayoutError("model returned no past_key_values; call with use_cache=True")
    if hasattr(past_key_values, "layers"):
        pairs = [(layer.keys, layer.values) for layer in past_key_values.layers]
    elif hasattr(past_key_values, "key_cache") and hasattr(past_key_values, "value_cache"):
        pairs = list(zip(past_key_values.key_cache, past_key_values.value_cache))
    elif isinstance(past_key_values, (tuple, list)):
        pairs = []
        for entry in past_key_values:
            if not (isinstance(entry, (tuple, list)) and len(entry) == 2):
                raise CacheLayoutError(f"unsupported legacy cache entry {type(entry).__name__}")
            pairs.append((entry[0], entry[1]))
    else:
        raise CacheLayoutError(f"unsupported cache layout {type(past_key_values).__name__}")
    out = []
    for k, v in pairs:
        if k.dim() != 4 or v.dim() != 4:
            raise CacheLayoutError(f"expected 4-D [batch, heads, seq, dim] cache tensors, got {tuple(k.shape)}")
        out.append((k.detach().contiguous(), v.detach().contiguous()))
    return out


def model_kv_geometry(model) -> dict:
    """KV-cache shape the model will produce, read off its config (hfcache.py:70-80)."""
    cfg = model.config
    attn_heads = cfg.num_attention_heads
    kv_heads = getattr(cfg, "num_key_value_heads", None) or attn_heads
    head_dim = getattr(cfg, "head_dim", None) or cfg.hidden_size // attn_heads
    return {"num_layers": cfg.num_hidden_layers, "kv_heads": int(kv_heads), "head_dim": int(head_dim)}


# ---------------------------------------------------------------------------
# materialising injection (reference semantics)
# ---------------------------------------------------------------------------

def build_dynamic_cache(layers: Sequence[tuple[torch.Tensor, torch.Tensor]]) -> DynamicCache:
    """A fresh DynamicCache from per-layer tensors (hfcache.py:58-67); tensors are cloned."""
    cache = DynamicCache()
    for idx, (k, v) in enumerate(layers):
        cache.update(k.clone(), v.clone(), idx)
    return cache


def _as_view(src) -> AgentCacheView:
    if isinstance(src, AgentCacheView):
        return src
    if isinstance(src, SharedPool):
        return src.attach(16)
    raise TypeError(f"expected an AgentCacheView or SharedPool, got {type(src).__name__}")


def build_cache(src, mode: str = "materialize", *, batch: int = 1, dtype: torch.dtype | None = None,
                tail_capacity: int = 256):
    """Cache for `batch` agents sharing the pool's prefix.

    mode="materialize": DynamicCache filled by one decode launch (the view's
    decode_bits decides bf16 vs f32 values, exactly get_kv_for_layer's),
    expanded to `batch` rows and cast to `dtype` (default: decoded dtype).
    mode="stream": PooledCache reading the packed pool in attention.
    """
    view = _as_view(src)
    if mode == "materialize":
        cache = DynamicCache()
        for idx, (k, v) in enumerate(view.materialize_all()):
            if dtype is not None:
                k, v = k.to(dtype), v.to(dtype)
            if batch != 1:
                k = k.expand(batch, -1, -1, -1).contiguous()
                v = v.expand(batch, -1, -1, -1).contiguous()
            cache.update(k, v, idx)
        return cache
    if mode == "stream":
        return PooledCache(view.pool, batch=batch, tail_capacity=tail_capacity, decode_bits=view.decode_bits)
    raise ValueError(f"mode must be 'materialize' or 'stream', got {mode!r}")


# ---------------------------------------------------------------------------
# streaming injection
# ---------------------------------------------------------------------------

class PooledLayer(CacheLayerMixin):
    """One model layer over the shared pool: prefix = packed pool layer
    (never copied), suffix = per-agent bf16 tail of generated tokens."""

    is_sliding = False

    def __init__(self, pool: SharedPool, layer_idx: int, batch: int, tail_capacity: int, decode_bits: int):
        super().__init__()
        self.pool = pool
        self.layer_idx = layer_idx
        self.batch = batch
        self.capacity = max(1, tail_capacity)
        self.decode_bits = decode_bits
        self.tail_len = 0
        self._len_t: torch.Tensor | None = None  # device tail length (read by the attention kernel)
        self._pos_t: torch.Tensor | None = None  # device write position of the next token

    @property
    def prefix_len(self) -> int:
        return self.pool.geometry.seq_len

    def lazy_initialization(self, key_states: torch.Tensor, value_states: torch.Tensor) -> None:
        self.dtype, self.device = key_states.dtype, key_states.device
        B, H, _, D = key_states.shape
        self.keys = torch.zeros((B, H, self.capacity, D), dtype=torch.bfloat16, device=self.device)
        self.values = torch.zeros_like(self.keys)
        self._len_t = torch.zeros(B, dtype=torch.int32, device=self.device)
        self._pos_t = torch.zeros(1, dtype=torch.int64, device=self.device)
        self.is_initialized = True

    def _grow(self, need: int) -> None:
        cap = self.capacity
        while cap < need:
            cap *= 2
        if cap != self.capacity:
            B, H, _, D = self.keys.shape
            k = torch.zeros((B, H, cap, D), dtype=self.keys.dtype, device=self.device)
            v = torch.zeros_like(k)
            k[:, :, :self.tail_len] = self.keys[:, :, :self.tail_len]
            v[:, :, :self.tail_len] = self.values[:, :, :self.tail_len]
            self.keys, self.values, self.capacity = k, v, cap

    def update(self, key_states: torch.Tensor, value_states: torch.Tensor, *args, **kwargs):
        if not self.is_initialized:
            self.lazy_initialization(key_states, value_states)
        n = key_states.shape[-2]
        if n == 1:
            # decode step: device-side position, so the step can be CUDA-graph
            # captured and replayed (no Python int baked into the launches)
            if self.tail_len + 1 > self.capacity:
                self._grow(self.tail_len + 1)
            self.keys.index_copy_(2, self._pos_t, key_states.to(torch.bfloat16))
            self.values.index_copy_(2, self._pos_t, value_states.to(torch.bfloat16))
            self._len_t.add_(1)
            self._pos_t.add_(1)
            self.tail_len += 1
            k, v = self.keys, self.values  # full buffers: the kernel reads _len_t
        else:
            self._grow(self.tail_len + n)
            self.keys[:, :, self.tail_len:self.tail_len + n] = key_states.to(torch.bfloat16)
            self.values[:, :, self.tail_len:self.tail_len + n] = value_states.to(torch.bfloat16)
            self.tail_len += n
            self._len_t.fill_(self.tail_len)
            self._pos_t.fill_(self.tail_len)
            k = self.keys[:, :, :self.tail_len]
            v = self.values[:, :, :self.tail_len]
        # the attention function recognises pooled layers by this marker
        k._pkv_layer = (self, n)
        v._pkv_layer = (self, n)
        return k, v

    def sync_lengths(self) -> None:
        """Re-read the tail length from the device (after CUDA-graph replays)."""
        if self._len_t is not None:
            self.tail_len = int(self._len_t[0].item())

    def get_mask_sizes(self, query_length: int) -> tuple[int, int]:
        return self.prefix_len + self.tail_len + query_length, 0

    def get_seq_length(self) -> int:
        return self.prefix_len + self.tail_len

    def get_max_cache_shape(self) -> int:
        return -1

    def reset(self) -> None:
        self.tail_len = 0
        if self._len_t is not None:
            self._len_t.zero_()

    def materialize(self, dtype: torch.dtype) -> tuple[torch.Tensor, torch.Tensor]:
        """[B, H, prefix + tail, D] K/V: fresh pool decode + the tail (prefill path only)."""
        out = torch.bfloat16 if self.decode_bits == 16 else torch.float32
        (pk, pv), = self.pool.decode_layers([self.layer_idx], out)
        B = self.keys.shape[0]
        k = torch.cat([pk.to(dtype).expand(B, -1, -1, -1), self.keys[:, :, :self.tail_len].to(dtype)], dim=2)
        v = torch.cat([pv.to(dtype).expand(B, -1, -1, -1), self.values[:, :, :self.tail_len].to(dtype)], dim=2)
        return k, v


class PooledCache(Cache):
    """Cache for a batch of agents over one sealed SharedPool."""

    def __init__(self, pool: SharedPool, batch: int = 1, tail_capacity: int = 256, decode_bits: int = 16):
        if not pool.sealed:
            raise ValueError("PooledCache needs a sealed pool")
        if pool.geometry.batch != 1:
            raise ValueError("the shared prefix pool must have batch 1")
        layers = [PooledLayer(pool, i, batch, tail_capacity, decode_bits) for i in range(pool.num_layers)]
        super().__init__(layers=layers)
        self.pool = pool
        self.batch = batch

    def sync_lengths(self) -> None:
        for layer in self.layers:
            layer.sync_lengths()


def pooled_attention_forward(module, query: torch.Tensor, key: torch.Tensor, value: torch.Tensor,
                             attention_mask, scaling: float | None = None, dropout: float = 0.0, **kwargs):
    """AttentionInterface entry "polykv" (called at modeling_llama.py:272-283).

    Every step runs pkv_decode_attention over the packed pool + the agents'
    bf16 tails: a decode step (one new token per agent) and a multi-token
    step (a prompt suffix on top of the pool) alike -- the latter as q_len
    query positions per agent with a causal limit on the tail, so no
    per-agent copy of the prefix is ever materialised. Layers that are not
    pooled fall back to SDPA.
    """
    from transformers.integrations.sdpa_attention import sdpa_attention_forward

    marker = getattr(key, "_pkv_layer", None)
    if marker is None:
        return sdpa_attention_forward(module, query, key, value, attention_mask, scaling=scaling,
                                      dropout=dropout, **kwargs)
    layer, n_new = marker
    B, Hq, q_len, D = query.shape
    Hkv = layer.pool.geometry.kv_heads
    scale = scaling if scaling is not None else D ** -0.5
    # query [B, Hq, q_len, D] with Hq = Hkv * G (query head h*G+g reads kv head h,
    # repeat_kv) -> [B, Hkv, G * q_len, D]: row g * q_len + i is position i
    G = Hq // Hkv
    q = query.reshape(B, Hkv, G * q_len, D)
    out = decode_attention(layer.pool, layer.layer_idx, q, tail_k=layer.keys, tail_v=layer.values,
                           tail_len=layer._len_t, softmax_scale=scale, out_dtype=query.dtype, q_len=q_len)
    return out.reshape(B, Hq, q_len, D).transpose(1, 2), None


AttentionInterface.register(ATTN_IMPLEMENTATION, pooled_attention_forward)


def use_pooled_attention(model) -> None:
    """Route the model's attention through "polykv" (pooled layers) / SDPA (others)."""
    if hasattr(model, "set_attn_implementation"):
        model.set_attn_implementation(ATTN_IMPLEMENTATION)
    else:  # pragma: no cover - older transformers
        model.config._attn_implementation = ATTN_IMPLEMENTATION


def greedy_continuation(model, full_ids: torch.Tensor, src, max_new_tokens: int, *, mode: str = "stream",
                        batch: int | None = None) -> torch.Tensor:
    """Greedy-decode `max_new_tokens` after `full_ids` with the pool injected
    for its prefix (evaluator.py:112-132 without the tokenizer round trip).

    Returns the new token ids [batch, max_new_tokens]. A manual loop (one
    forward per token) so that the same code path serves both modes.
    """
    ids = torch.atleast_2d(torch.as_tensor(full_ids, device=model.device))
    B = batch or ids.shape[0]
    if ids.shape[0] != B:
        ids = ids.expand(B, -1)
    view = _as_view(src)
    prefix = view.pool.geometry.seq_len
    if ids.shape[1] <= prefix:
        raise ValueError("full_ids must extend past the pooled prefix")
    dt = next(model.parameters()).dtype
    cache = build_cache(view, mode, batch=B, dtype=dt)
    if mode == "stream":
        use_pooled_attention(model)
    out = []
    with torch.no_grad():
        step = ids[:, prefix:]
        pos = prefix
        for _ in range(max_new_tokens):
            position_ids = torch.arange(pos, pos + step.shape[1], device=ids.device).unsqueeze(0).expand(B, -1)
            logits = model(step, past_key_values=cache, position_ids=position_ids, use_cache=True).logits
            nxt = logits[:, -1].argmax(-1, keepdim=True)
            out.append(nxt)
            pos += step.shape[1]
            step = nxt
    return torch.cat(out, dim=1)


__all__ = [
    "ATTN_IMPLEMENTATION", "CacheLayoutError", "PooledCache", "PooledLayer", "build_cache",
    "build_dynamic_cache", "cache_layers", "greedy_continuation", "model_kv_geometry",
    "pooled_attention_forward", "use_pooled_attention",
]
