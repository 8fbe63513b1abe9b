"""Value path: 3-bit Lloyd-Max codebook over FWHT-rotated, RMS-normalised vectors.

API-compatible with kvpool.valuequant (/root/reference/pkg/src/kvpool/
valuequant.py). quantize_v / dequantize_v run the fused sm_100a kernels of
libpolykv.so (rotate -> RMS -> code -> 3-bit pack, and unpack -> lookup ->
inverse rotate); codes and scales are bit-identical to the reference.

A QuantizedValueBlock stores its codes *packed* on the device (8 codes per
3 bytes, the PKVP packed payload, valuequant.py:312-328); `.codes` unpacks on
demand to the reference's canonical uint8 form.
"""

from __future__ import annotations

import math
import warnings
from dataclasses import dataclass, field
from fractions import Fraction

import numpy as np
import torch

from . import _codec
from .errors import CorruptBlockError, GeometryError, KvPoolError
from .model import KvTensor, ModelGeometry

GAUSSIAN_3BIT_NAME = "gaussian-3bit-v1"
_GAUSSIAN_3BIT_CENTROIDS = (-2.152, -1.344, -0.756, -0.245, 0.245, 0.756, 1.344, 2.152)


@dataclass(frozen=True)
class Codebook:
    """Strictly increasing centroids plus pinned cell midpoints (valuequant.py:37-82)."""

    bits: int
    centroids: np.ndarray
    name: str = "unnamed"
    midpoints: np.ndarray = field(init=False, repr=False)

    def __post_init__(self):
        if not 1 <= self.bits <= 8:
            raise ValueError(f"bits must be in [1, 8], got {self.bits}")
        c = np.ascontiguousarray(self.centroids, dtype=np.float64).copy()
        if c.ndim != 1 or c.size != 1 << self.bits:
            raise ValueError(f"need {1 << self.bits} centroids for {self.bits} bits, got shape {c.shape}")
        if not np.isfinite(c).all():
            raise ValueError("centroids must be finite")
        if not (np.diff(c) > 0).all():
            raise ValueError("centroids must be strictly increasing")
        mids = np.empty(c.size - 1, dtype=np.float64)
        for i in range(mids.size):
            # largest float64 not above the exact rational midpoint, so that
            # "#boundaries < z" is nearest-centroid with ties to the lower cell
            exact = (Fraction(float(c[i])) + Fraction(float(c[i + 1]))) / 2
            m = float((c[i] + c[i + 1]) / 2.0)
            while Fraction(m) > exact:
                m = float(np.nextafter(m, -np.inf))
            mids[i] = m
        c.flags.writeable = False
        mids.flags.writeable = False
        object.__setattr__(self, "centroids", c)
        object.__setattr__(self, "midpoints", mids)

    @property
    def levels(self) -> int:
        return 1 << self.bits

    def is_symmetric(self, atol: float = 0.0) -> bool:
        return bool(np.allclose(self.centroids, -self.centroids[::-1], atol=atol, rtol=0.0))


GAUSSIAN_3BIT = Codebook(bits=3, centroids=np.array(_GAUSSIAN_3BIT_CENTROIDS), name=GAUSSIAN_3BIT_NAME)


@dataclass(frozen=True)
class DistortionBound:
    """High-resolution ceiling (sqrt(3)*pi/2) * 4**-b per unit-variance coordinate."""

    bits: int
    bound: float = field(init=False)

    def __post_init__(self):
        if self.bits < 1:
            raise ValueError(f"bits must be >= 1, got {self.bits}")
        object.__setattr__(self, "bound", (math.sqrt(3.0) * math.pi / 2.0) * 4.0 ** (-self.bits))


def nearest_centroid(x: float, codebook: Codebook) -> int:
    """Scalar coder (host utility): count of midpoints strictly below x."""
    return int(np.searchsorted(codebook.midpoints, x, side="left"))


def encode_coordinates(z, codebook: Codebook) -> np.ndarray:
    return np.searchsorted(codebook.midpoints, np.asarray(z), side="left").astype(np.uint8)


def sign_diagonal(seed: int, head_dim: int) -> np.ndarray:
    """Seeded +-1 diagonal (valuequant.py:183-190), identical draws."""
    rng = np.random.default_rng(seed)
    return (rng.integers(0, 2, size=head_dim) * 2 - 1).astype(np.float64)


def _require_3bit(codebook: Codebook) -> None:
    if codebook.bits != 3:
        raise KvPoolError(
            f"the B200 pool stores 3-bit packed codes; codebook {codebook.name!r} has "
            f"{codebook.bits} bits"
        )


def packed_nbytes(count: int) -> int:
    return 3 * ((count + 7) // 8)


class QuantizedValueBlock:
    """One layer's quantized V: packed 3-bit codes + f32 RMS per head vector.

    Constructor mirrors valuequant.py:124-180 (geometry, codebook_name, bits,
    codes, scales, sign_seed) and validates the same invariants; pass
    `packed=` instead of `codes=` to wrap an existing packed payload.
    """

    def __init__(self, geometry: ModelGeometry, codebook_name: str, bits: int, codes=None,
                 scales=None, sign_seed: int | None = None, *, packed: torch.Tensor | None = None,
                 _trusted: bool = False):
        self.geometry = geometry
        self.codebook_name = codebook_name
        self.bits = bits
        self.sign_seed = sign_seed
        n = geometry.elements_per_tensor
        if bits != 3:
            raise KvPoolError("the B200 pool stores 3-bit packed codes only")
        if scales is None:
            raise CorruptBlockError("scales are required")
        if isinstance(scales, np.ndarray):
            if scales.dtype != np.float32:
                raise CorruptBlockError(
                    f"scales must be float32 with shape {geometry.tensor_shape[:-1]}, got "
                    f"{scales.dtype} {scales.shape}")
            scales = torch.from_numpy(np.ascontiguousarray(scales).copy())
        if scales.dtype != torch.float32 or tuple(scales.shape) != geometry.tensor_shape[:-1]:
            raise CorruptBlockError(
                f"scales must be float32 with shape {geometry.tensor_shape[:-1]}, got "
                f"{scales.dtype} {tuple(scales.shape)}")
        if packed is None:
            if codes is None:
                raise CorruptBlockError("need codes or packed")
            if isinstance(codes, np.ndarray):
                if codes.dtype != np.uint8:
                    raise CorruptBlockError(f"value codes must be uint8, got {codes.dtype}")
                codes = torch.from_numpy(np.ascontiguousarray(codes).copy())
            if codes.dtype != torch.uint8:
                raise CorruptBlockError(f"value codes must be uint8, got {codes.dtype}")
            if tuple(codes.shape) != geometry.tensor_shape:
                raise GeometryError(
                    f"value codes shape {tuple(codes.shape)} does not match geometry "
                    f"{geometry.tensor_shape}")
            device = _codec.require_device(scales.device if scales.is_cuda else None)
            codes = codes.to(device).contiguous()
            scales = scales.to(device)
            if not _trusted:
                self._validate(codes, scales)
            packed = torch.empty(packed_nbytes(n), dtype=torch.uint8, device=device)
            bad = torch.zeros(1, dtype=torch.int32, device=device)
            _codec.pack_codes(codes, n, packed, bad)
        else:
            if packed.dtype != torch.uint8 or packed.numel() < packed_nbytes(n):
                raise CorruptBlockError("packed payload has the wrong dtype or size")
            if not _trusted:
                device = packed.device
                self._validate(None, scales.to(device), packed=packed)
        self.packed = packed
        self.scales = scales.to(packed.device).contiguous()

    def _validate(self, codes, scales, packed=None) -> None:
        # valuequant.py:141-166 (one device reduction + sync; user-built blocks only)
        if codes is None:
            n = self.geometry.elements_per_tensor
            codes = torch.empty(n, dtype=torch.uint8, device=packed.device)
            _codec.unpack_codes(packed, n, codes)
            codes = codes.view(self.geometry.tensor_shape)
        if codes.numel() and int(codes.max()) >= (1 << self.bits):
            raise CorruptBlockError(
                f"corrupt block: code {int(codes.max())} out of range for {self.bits}-bit codebook")
        if not bool(torch.isfinite(scales).all()) or bool((scales < 0).any()):
            raise CorruptBlockError("scales must be finite and >= 0")
        if bool(codes[scales == 0].any()):
            raise CorruptBlockError("zero-scale vector with nonzero codes")

    @property
    def device(self) -> torch.device:
        return self.packed.device

    @property
    def codes(self) -> torch.Tensor:
        """Canonical uint8 codes [B,H,T,D], unpacked on the device."""
        n = self.geometry.elements_per_tensor
        out = torch.empty(n, dtype=torch.uint8, device=self.packed.device)
        _codec.unpack_codes(self.packed, n, out)
        return out.view(self.geometry.tensor_shape)

    @property
    def payload_nbytes(self) -> int:
        """Canonical-form bytes (one per code + f32 scales), as valuequant.py:170-173."""
        return self.geometry.elements_per_tensor + 4 * self.geometry.vectors_per_tensor

    @property
    def packed_payload_nbytes(self) -> int:
        """Packed bytes (8 codes per 3 bytes + scales), valuequant.py:175-180; what HBM holds."""
        return packed_nbytes(self.geometry.elements_per_tensor) + 4 * self.geometry.vectors_per_tensor


def quantize_v(tensor: KvTensor, codebook: Codebook = GAUSSIAN_3BIT,
               sign_seed: int | None = None) -> QuantizedValueBlock:
    """Rotate, RMS-normalise and code one layer's V on the GPU (valuequant.py:193-219)."""
    from .pool import _encode_layers  # single code path shared with build_pool

    _require_3bit(codebook)
    return _encode_layers([None], [tensor], tensor.geometry, codebook, sign_seed, "tensor")[1][0]


def dequantize_v(block: QuantizedValueBlock, codebook: Codebook = GAUSSIAN_3BIT, *,
                 dtype: torch.dtype = torch.float32) -> KvTensor:
    """Centroid lookup * RMS, inverse rotation (valuequant.py:222-238), on the GPU."""
    if codebook.name != block.codebook_name or codebook.bits != block.bits:
        raise CorruptBlockError(
            f"block was coded with {block.codebook_name!r} at {block.bits} bits, "
            f"got {codebook.name!r} at {codebook.bits} bits")
    g = block.geometry
    out = torch.empty(g.tensor_shape, dtype=dtype, device=block.device)
    _codec.decode(
        num_vectors=g.vectors_per_tensor, head_dim=g.head_dim, out_dtype=dtype, k_mode=0,
        k_codes=None, k_scale=None, k_bscale=None, v_packed=[block.packed], v_scales=[block.scales],
        centroids=codebook.centroids, sign_seed=block.sign_seed, k_out=None, v_out=[out],
        device=block.device)
    return KvTensor(g, out)


def lloyd_max_train(samples, bits: int, max_iters: int = 200, tol: float = 1e-7) -> Codebook:
    """Scalar Lloyd-Max codebook for 1-D samples (kvpool.lloyd_max_train,
    valuequant.py:241-300 semantics: quantile start, midpoint cells with
    ties to the lower cell, cell means, empty cells reseeded inside the most
    populated cell with a RuntimeWarning, strictly increasing centroids).

    Offline table building, not on the compress/inject path (
    the pool codes with the frozen GAUSSIAN_3BIT table). Implemented on the
    SORTED samples: every cell is a contiguous run, so one iteration is two
    searchsorted calls over the level boundaries and a prefix-sum difference,
    O(levels log n) instead of a pass over all samples.
    """
    x = np.sort(np.asarray(samples, dtype=np.float64).ravel())
    if not 1 <= bits <= 8:
        raise ValueError(f"bits must be in [1, 8], got {bits}")
    k = 1 << bits
    if x.size < 10 * k:
        raise ValueError(f"need at least {10 * k} samples for {bits} bits, got {x.size}")
    if not np.isfinite(x).all():
        raise ValueError("samples must be finite")
    csum = np.concatenate(([0.0], np.cumsum(x)))

    def monotone(c):  # nudge ties up by one ulp, left to right
        c = np.array(c, dtype=np.float64)
        for i in range(1, c.size):
            if c[i] <= c[i - 1]:
                c[i] = np.nextafter(c[i - 1], np.inf)
        return c

    c = monotone(np.quantile(x, (np.arange(k) + 0.5) / k))
    reseeded = 0
    for _ in range(max_iters):
        mid = 0.5 * (c[1:] + c[:-1])
        edge = np.concatenate(([0], np.searchsorted(x, mid, side="right"), [x.size]))
        n = np.diff(edge)
        total = csum[edge[1:]] - csum[edge[:-1]]
        upd = np.where(n > 0, total / np.maximum(n, 1), c)
        hole = np.flatnonzero(n == 0)
        if hole.size:
            reseeded += hole.size
            full = int(np.argmax(n))
            left = x[0] if full == 0 else mid[full - 1]
            right = x[-1] if full == k - 1 else mid[full]
            upd[hole] = left + (np.arange(1, hole.size + 1) / (hole.size + 1)) * (right - left)
            c = monotone(np.sort(upd))
            continue
        upd = monotone(upd)
        moved = float(np.abs(upd - c).max())
        c = upd
        if moved < tol:
            break
    if reseeded:
        warnings.warn(f"lloyd_max_train repaired {reseeded} empty cell(s)", RuntimeWarning)
    return Codebook(bits=bits, centroids=c, name=f"lloyd-max-{bits}bit-trained")


def pack_indices_3bit(codes) -> bytes:
    """Host byte packer for snapshot files (valuequant.py:312-328 layout)."""
    if isinstance(codes, torch.Tensor):
        codes = codes.detach().cpu().numpy()
    flat = np.ascontiguousarray(codes, dtype=np.uint8).reshape(-1)
    if flat.size and int(flat.max()) > 7:
        raise ValueError("3-bit packing needs codes in [0, 7]")
    n = flat.size
    g = np.zeros(((n + 7) // 8) * 8, dtype=np.uint32)
    g[:n] = flat
    words = np.zeros(g.size // 8, dtype=np.uint32)
    for i in range(8):
        words |= g[i::8] << np.uint32(3 * i)
    b = np.empty((words.size, 3), dtype=np.uint8)
    b[:, 0] = words & 0xFF
    b[:, 1] = (words >> 8) & 0xFF
    b[:, 2] = (words >> 16) & 0xFF
    return b.tobytes()


def unpack_indices_3bit(packed: bytes, count: int) -> np.ndarray:
    raw = np.frombuffer(packed, dtype=np.uint8)
    if raw.size != 3 * ((count + 7) // 8):
        raise ValueError(f"packed length {raw.size} does not fit {count} 3-bit codes")
    if count == 0:
        return np.zeros(0, dtype=np.uint8)
    t = raw.reshape(-1, 3).astype(np.uint32)
    w = t[:, 0] | (t[:, 1] << np.uint32(8)) | (t[:, 2] << np.uint32(16))
    out = np.empty((w.size, 8), dtype=np.uint8)
    for i in range(8):
        out[:, i] = (w >> np.uint32(3 * i)) & 0x7
    return out.reshape(-1)[:count].copy()
