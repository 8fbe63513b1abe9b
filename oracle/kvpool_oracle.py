"""CPU oracle for the SharedKVPool compress/inject hot path.

TEST INFRASTRUCTURE ONLY. This module is the parity checker: only tests/,
__graft_entry__.smoke() and bench.py's cpu_baseline / --impl reference leg
may import it. The product package (paper_2604_24971_b200) never does; its
codec runs exclusively in libpolykv.so on the GPU.

It restates, with numpy, the algorithm of the reference's pure-Python
`kvpool` package (/root/reference/pkg/src/kvpool). Every function cites the
reference lines it follows. numpy itself (2.3.x here; the reference pins only
numpy>=1.24, pkg/pyproject.toml:12) is part of the oracle: the f64 pairwise
summation behind np.mean (valuequant.py:207) decides value scales and codes.

Pinning: tests/test_oracle_golden.py checks this module against
  * golden vectors produced by the reference itself (tests/golden/*.npz,
    written by tests/golden/make_golden.py, which imports /root/reference),
  * the reference's own known-answer tests (pkg/tests/test_keyquant.py,
    test_valuequant.py, test_pool.py, test_acceptance.py) restated.

Where the reference has no function (per-32-block fp16 key scales; attention
over a compressed pool) this module defines the semantics, and says so.
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np

# valuequant.py:31-34 — Lloyd-Max centroids of N(0,1) at 3 bits
GAUSSIAN_3BIT_CENTROIDS = np.array(
    [-2.152, -1.344, -0.756, -0.245, 0.245, 0.756, 1.344, 2.152], dtype=np.float64
)
INT8_LEVELS = 127  # keyquant.py:19


def pinned_midpoints(centroids) -> np.ndarray:
    """Cell boundaries: largest float64 not above each exact rational midpoint.

    valuequant.py:60-71 (Codebook.__post_init__).
    """
    c = np.asarray(centroids, dtype=np.float64)
    out = np.empty(c.size - 1, dtype=np.float64)
    for i in range(c.size - 1):
        exact = (Fraction(float(c[i])) + Fraction(float(c[i + 1]))) / 2
        m = float((c[i] + c[i + 1]) / 2.0)
        while Fraction(m) > exact:
            m = float(np.nextafter(m, -np.inf))
        out[i] = m
    return out


GAUSSIAN_3BIT_MIDPOINTS = pinned_midpoints(GAUSSIAN_3BIT_CENTROIDS)


# ---------------------------------------------------------------------------
# rotation (fwht.py)
# ---------------------------------------------------------------------------

def fwht_last_axis(arr: np.ndarray) -> np.ndarray:
    """Unnormalised Sylvester FWHT of the last axis, returned as a new array.

    fwht.py:24-41: stages half = 1, 2, 4, ...; at each stage the pair
    (lo, hi) = (x[i], x[i + half]) becomes (lo + hi, lo - hi).
    """
    x = np.array(arr, copy=True, order="C")
    d = x.shape[-1]
    if d < 1 or d & (d - 1):
        raise ValueError(f"transform length must be a power of two, got {d}")
    lead = x.shape[:-1]
    h = 1
    while h < d:
        # coordinate i = (block, bit h of i, offset): lo = bit clear, hi = set
        view = x.reshape(lead + (d // (2 * h), 2, h))
        a = view[..., 0, :]
        b = view[..., 1, :]
        s, t = a + b, a - b
        view[..., 0, :] = s
        view[..., 1, :] = t
        h <<= 1
    return x


def rotate(arr: np.ndarray) -> np.ndarray:
    """H x / sqrt(d) in the input's float dtype (f32 stays f32, else f64).

    fwht.py:44-61 (rotate_forward == rotate_inverse).
    """
    a = np.asarray(arr)
    dt = a.dtype if a.dtype in (np.float32, np.float64) else np.dtype(np.float64)
    y = fwht_last_axis(a.astype(dt, copy=True))
    y /= dt.type(np.sqrt(a.shape[-1]))
    return y


def sign_diagonal(seed: int, head_dim: int) -> np.ndarray:
    """valuequant.py:183-190: default_rng(seed).integers(0, 2, d) * 2 - 1, f64."""
    rng = np.random.default_rng(seed)
    return (rng.integers(0, 2, size=head_dim) * 2 - 1).astype(np.float64)


def sign_bits(seed: int | None, head_dim: int) -> np.ndarray | None:
    """The sign diagonal as LSB-first uint32 words (bit set = -1), the C ABI form."""
    if seed is None:
        return None
    neg = sign_diagonal(seed, head_dim) < 0
    words = np.zeros((head_dim + 31) // 32, dtype=np.uint32)
    for i in np.flatnonzero(neg):
        words[i // 32] |= np.uint32(1 << (i % 32))
    return words


# ---------------------------------------------------------------------------
# keys (keyquant.py)
# ---------------------------------------------------------------------------

def quantize_k_tensor(values: np.ndarray) -> tuple[float, np.ndarray]:
    """Per-tensor q8_0 keys. keyquant.py:52-65.

    scale = f32(max|K| / 127); code = clip(floor(|K/s| + 0.5) * sign, -128, 127)
    with K/s evaluated in f64. An all-zero tensor gets scale 0, codes 0.
    """
    x = np.asarray(values, dtype=np.float32)
    peak = float(np.max(np.abs(x))) if x.size else 0.0
    if peak == 0.0:
        return 0.0, np.zeros(x.shape, dtype=np.int8)
    scale = float(np.float32(peak / INT8_LEVELS))
    q = x.astype(np.float64) / scale
    r = np.floor(np.abs(q) + 0.5) * np.sign(q)
    return scale, np.clip(r, -128, 127).astype(np.int8)


def dequantize_k_tensor(codes: np.ndarray, scale: float) -> np.ndarray:
    """keyquant.py:68-71: codes (as f32) * f32(scale)."""
    return np.asarray(codes).astype(np.float32) * np.float32(scale)


def quantize_k_block32(values: np.ndarray) -> tuple[np.ndarray, np.ndarray]:
    """Per-32-element q8_0 keys with fp16 scales (NOT in the reference).

    The north star asks for ggml-style q8_0 blocks; the reference has only a
    per-tensor scale (keyquant.py:1-7). Semantics defined here and used by the
    GPU kernel: blocks are 32 consecutive elements of the flattened tensor
    (the last block may be short); for each block
        s32 = f32(peak / 127)                       (as keyquant.py:60)
        s16 = fp16 round-to-nearest(s32); if peak > 0 and s16 == 0 -> 2^-24
        code = clip(floor(|x / f32(s16)| + 0.5) * sign, -127, 127)  (f64 quotient)
    Dequant is code * f32(s16). Returns (fp16 scales [ceil(n/32)], int8 codes).
    A scale that overflows fp16 is an error (returned as inf here).
    """
    x = np.asarray(values, dtype=np.float32)
    flat = x.reshape(-1)
    n = flat.size
    nb = (n + 31) // 32
    pad = np.zeros(nb * 32, dtype=np.float32)
    pad[:n] = flat
    blocks = pad.reshape(nb, 32)
    peak = np.max(np.abs(blocks), axis=1).astype(np.float64)
    s32 = (peak / INT8_LEVELS).astype(np.float32)
    s16 = s32.astype(np.float16)
    tiny = (peak > 0) & (s16 == 0)
    s16[tiny] = np.float16(2.0**-24)
    sf = s16.astype(np.float64)
    with np.errstate(divide="ignore", invalid="ignore"):
        q = blocks.astype(np.float64) / np.where(sf > 0, sf, 1.0)[:, None]
    r = np.floor(np.abs(q) + 0.5) * np.sign(q)
    r[sf == 0] = 0.0
    codes = np.clip(r, -127, 127).astype(np.int8).reshape(-1)[:n].reshape(x.shape)
    return s16, codes


def dequantize_k_block32(codes: np.ndarray, scales16: np.ndarray) -> np.ndarray:
    c = np.asarray(codes)
    flat = c.reshape(-1).astype(np.float32)
    s = np.repeat(np.asarray(scales16, dtype=np.float16).astype(np.float32), 32)[: flat.size]
    return (flat * s).reshape(c.shape)


# ---------------------------------------------------------------------------
# values (valuequant.py)
# ---------------------------------------------------------------------------

def quantize_v(values: np.ndarray, sign_seed: int | None = None,
               midpoints: np.ndarray = GAUSSIAN_3BIT_MIDPOINTS) -> tuple[np.ndarray, np.ndarray]:
    """valuequant.py:193-219. Returns (uint8 codes [..., d], f32 scales [...]).

    f64 all the way: (x * sign) -> FWHT / sqrt(d) -> rms = sqrt(mean(rot^2))
    (numpy pairwise mean) -> scale = f32(rms) -> z = rot / rms (f64 rms, 1 for
    zero rows) -> code = #{midpoints < z} -> rows with f32 scale 0 get code 0.
    """
    x = np.asarray(values, dtype=np.float32).astype(np.float64)
    d = x.shape[-1]
    if sign_seed is not None:
        x = x * sign_diagonal(sign_seed, d)
    rot = rotate(x)
    rms = np.sqrt(np.mean(np.square(rot), axis=-1))
    scales = rms.astype(np.float32)
    z = rot / np.where(rms > 0.0, rms, 1.0)[..., None]
    codes = np.searchsorted(midpoints, z, side="left").astype(np.uint8)
    codes[scales == 0.0] = 0
    return codes, scales


def dequantize_v(codes: np.ndarray, scales: np.ndarray, sign_seed: int | None = None,
                 centroids: np.ndarray = GAUSSIAN_3BIT_CENTROIDS) -> np.ndarray:
    """valuequant.py:222-238: f32 table[code] * scale -> f32 rotation -> * sign."""
    table = np.asarray(centroids).astype(np.float32)
    y = table[np.asarray(codes)]
    y *= np.asarray(scales, dtype=np.float32)[..., None]
    out = rotate(y)
    if sign_seed is not None:
        out *= sign_diagonal(sign_seed, out.shape[-1]).astype(np.float32)
    return out


def pack3(codes: np.ndarray) -> bytes:
    """valuequant.py:312-328: 8 codes -> 24-bit LE word (code i at bits 3i..3i+2)."""
    flat = np.ascontiguousarray(codes, dtype=np.uint8).reshape(-1)
    if flat.size and int(flat.max()) > 7:
        raise ValueError("3-bit packing needs codes in [0, 7]")
    n = flat.size
    groups = np.zeros(((n + 7) // 8) * 8, dtype=np.uint32)
    groups[:n] = flat
    g = groups.reshape(-1, 8)
    shifts = (3 * np.arange(8, dtype=np.uint32))[None, :]
    words = np.bitwise_or.reduce(g << shifts, axis=1).astype(np.uint32)
    b = np.stack([words & 0xFF, (words >> 8) & 0xFF, (words >> 16) & 0xFF], axis=1)
    return b.astype(np.uint8).tobytes()


def unpack3(packed: bytes | np.ndarray, count: int) -> np.ndarray:
    """valuequant.py:331-345."""
    raw = np.frombuffer(bytes(packed), dtype=np.uint8) if not isinstance(packed, np.ndarray) \
        else np.asarray(packed, dtype=np.uint8).reshape(-1)
    if raw.size != 3 * ((count + 7) // 8):
        raise ValueError(f"packed length {raw.size} does not fit {count} 3-bit codes")
    t = raw.reshape(-1, 3).astype(np.uint32)
    words = t[:, 0] | (t[:, 1] << 8) | (t[:, 2] << 16)
    shifts = (3 * np.arange(8, dtype=np.uint32))[None, :]
    codes = ((words[:, None] >> shifts) & 0x7).astype(np.uint8).reshape(-1)
    return codes[:count].copy()


# ---------------------------------------------------------------------------
# pool read side (pool.py)
# ---------------------------------------------------------------------------

def round_to_bfloat16(values: np.ndarray) -> np.ndarray:
    """pool.py:66-76: RNE on the upper 16 bits of the f32 pattern, kept as f32."""
    u = np.ascontiguousarray(values, dtype=np.float32).view(np.uint32)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return r.view(np.float32)


def decode_layer(k_codes, k_scale, v_codes, v_scales, decode_bits=16, sign_seed=None,
                 k_block_scales=None):
    """pool.py:229-237 get_kv_for_layer: (K, V) f32, bf16-rounded at 16 bits."""
    if k_block_scales is None:
        k = dequantize_k_tensor(k_codes, k_scale)
    else:
        k = dequantize_k_block32(k_codes, k_block_scales)
    v = dequantize_v(v_codes, v_scales, sign_seed)
    if decode_bits == 16:
        k, v = round_to_bfloat16(k), round_to_bfloat16(v)
    return k, v


FNV64_OFFSET = 0xCBF29CE484222325  # checksum.py:13-14
FNV64_PRIME = 0x100000001B3


def fnv1a64(data: bytes) -> int:
    """checksum.py:44-52 (pure Python; small inputs only)."""
    h = FNV64_OFFSET
    for b in data:
        h = ((h ^ b) * FNV64_PRIME) & 0xFFFFFFFFFFFFFFFF
    return h


def tensor_checksum(values: np.ndarray) -> int:
    """checksum.py:55-62: FNV-1a over the little-endian f32 image."""
    return fnv1a64(np.ascontiguousarray(values, dtype="<f4").tobytes())


# ---------------------------------------------------------------------------
# inputs (model.py) and accounting (metrics.py)
# ---------------------------------------------------------------------------

def synth_dump(num_layers, kv_heads, head_dim, seq_len, batch=1, seed=0, variance=None):
    """model.py:250-273: default_rng(seed).normal(0, sqrt(var), shape) as f32,
    K then V for each layer in order. Returns a list of (K, V)."""
    var = 1.0 / head_dim if variance is None else variance
    rng = np.random.default_rng(seed)
    std = float(np.sqrt(var))
    shape = (batch, kv_heads, seq_len, head_dim)
    out = []
    for _ in range(num_layers):
        k = rng.normal(0.0, std, size=shape).astype(np.float32)
        v = rng.normal(0.0, std, size=shape).astype(np.float32)
        out.append((k, v))
    return out


def compression_ratio_exact(k_bits: int, v_bits: int, baseline_bits: int) -> Fraction:
    """metrics.py:26-36: 2 * baseline / (k + v)."""
    return Fraction(2 * baseline_bits, k_bits + v_bits)


# ---------------------------------------------------------------------------
# attention over a compressed pool (NOT in the reference)
# ---------------------------------------------------------------------------

def attention_over_pool(q: np.ndarray, k_deq: np.ndarray, v_deq: np.ndarray,
                        softmax_scale: float, tail_k=None, tail_v=None) -> np.ndarray:
    """f64 GQA decode attention, the semantics of eager attention with repeat_kv
    (transformers modeling_llama.py:187-230) over the reference-dequantised
    pool K/V (+ an optional per-agent tail appended after the prefix).

    q [R, Hkv, G, D]; k_deq, v_deq [Hkv, T, D]; tails [R, Hkv, t, D].
    Returns [R, Hkv, G, D] f64.
    """
    q = np.asarray(q, dtype=np.float64)
    R, H, G, D = q.shape
    out = np.empty_like(q)
    for r in range(R):
        for h in range(H):
            k = np.asarray(k_deq[h], dtype=np.float64)
            v = np.asarray(v_deq[h], dtype=np.float64)
            if tail_k is not None and tail_k[r].shape[1] > 0:
                k = np.concatenate([k, np.asarray(tail_k[r][h], dtype=np.float64)], axis=0)
                v = np.concatenate([v, np.asarray(tail_v[r][h], dtype=np.float64)], axis=0)
            s = (q[r, h] @ k.T) * softmax_scale  # [G, T]
            s -= s.max(axis=-1, keepdims=True)
            p = np.exp(s)
            p /= p.sum(axis=-1, keepdims=True)
            out[r, h] = p @ v
    return out


# ---------------------------------------------------------------------------
# PKVP v1 snapshots (pool.py:14-25, 57-63, 301-432)
# ---------------------------------------------------------------------------

PKVP_HEADER = "<4sHHIIIIIHQ6x"  # magic, version, flags, L, B, H, T, D, baseline_bits, sign seed (44 bytes)


def read_pkvp(data: bytes) -> dict:
    """Parse a PKVP v1 file: per layer f32 key scale, int8 key codes, f32
    value scales, then uint8 value codes (flag 0x1: packed 8 codes / 3 bytes)."""
    import struct

    magic, version, flags, L, B, H, T, D, bits, seed = struct.unpack_from(PKVP_HEADER, data, 0)
    if magic != b"PKVP" or version != 1:
        raise ValueError("not a PKVP v1 file")
    e, vecs = B * H * T * D, B * H * T
    packed = bool(flags & 0x1)
    off = struct.calcsize(PKVP_HEADER)
    layers = []
    for _ in range(L):
        (scale,) = struct.unpack_from("<f", data, off)
        off += 4
        kc = np.frombuffer(data, np.int8, e, off).reshape(B, H, T, D)
        off += e
        vs = np.frombuffer(data, "<f4", vecs, off).reshape(B, H, T).astype(np.float32)
        off += 4 * vecs
        nv = 3 * ((e + 7) // 8) if packed else e
        raw = np.frombuffer(data, np.uint8, nv, off)
        off += nv
        vc = (unpack3(raw, e) if packed else raw.copy()).reshape(B, H, T, D)
        layers.append((float(scale), kc.copy(), vc, vs))
    if off != len(data):
        raise ValueError(f"{len(data) - off} trailing bytes")
    return {"geom": (L, B, H, T, D), "flags": flags, "sign_seed": seed if flags & 0x2 else None, "layers": layers}
