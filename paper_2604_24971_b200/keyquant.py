"""Key path: q8_0 int8 keys, per-tensor f32 scale (reference) or per-32 fp16 scales.

API-compatible with kvpool.keyquant (/root/reference/pkg/src/kvpool/
keyquant.py). k_scale_mode="tensor" (default) reproduces the reference
bit-for-bit; "block32" is the north star's ggml-style q8_0 layout (one fp16
scale per 32 contiguous elements; semantics in oracle/kvpool_oracle.py
quantize_k_block32 and DESIGN.md).
"""

from __future__ import annotations

import numpy as np
import torch

from . import _codec
from .errors import CorruptBlockError, GeometryError
from .model import KvTensor, ModelGeometry

INT8_LEVELS = 127
K_MODES = {"tensor": 0, "block32": 1}


def block32_count(n: int) -> int:
    return (n + 31) // 32


class QuantizedKeyBlock:
    """One layer's int8 key codes plus scale(s), resident on the device.

    QuantizedKeyBlock(geometry, scale, codes) as keyquant.py:22-49. In
    block32 mode `block_scales` holds ceil(n/32) fp16 scales and `scale` is
    their maximum (so the reference's error bound |err| <= scale/2 holds).
    """

    def __init__(self, geometry: ModelGeometry, scale, codes, *, mode: str = "tensor",
                 block_scales: torch.Tensor | None = None, _trusted: bool = False):
        if mode not in K_MODES:
            raise ValueError(f"k_scale_mode must be one of {tuple(K_MODES)}, got {mode!r}")
        self.geometry = geometry
        self.mode = mode
        if isinstance(codes, np.ndarray):
            if codes.dtype != np.int8:
                raise CorruptBlockError(f"key codes must be int8, got {codes.dtype}")
            codes = torch.from_numpy(np.ascontiguousarray(codes).copy())
        if codes.dtype != torch.int8:
            raise CorruptBlockError(f"key codes must be int8, got {codes.dtype}")
        if tuple(codes.shape) != geometry.tensor_shape:
            raise GeometryError(
                f"key codes shape {tuple(codes.shape)} does not match geometry {geometry.tensor_shape}")
        # trusted blocks view an existing arena (any device); user codes move to the GPU
        device = codes.device if (codes.is_cuda or _trusted) else _codec.require_device()
        codes = codes.to(device).contiguous()
        if mode == "tensor":
            if isinstance(scale, torch.Tensor):
                scale_t = scale.to(device=device, dtype=torch.float32).reshape(1)
            else:
                scale_t = torch.tensor([float(scale)], dtype=torch.float32, device=device)
            if not _trusted:
                s = float(scale_t.item())
                if not (np.isfinite(s) and s >= 0.0):
                    raise CorruptBlockError(f"key scale must be finite and >= 0, got {s}")
                if s == 0.0 and bool(codes.any()):
                    raise CorruptBlockError("zero scale with nonzero codes")
            self.scale_t = scale_t
            self.block_scales = None
        else:
            if block_scales is None or block_scales.dtype != torch.float16 or \
                    block_scales.numel() != block32_count(geometry.elements_per_tensor):
                raise CorruptBlockError("block32 keys need ceil(n/32) float16 block_scales")
            self.block_scales = block_scales.to(device).contiguous()
            self.scale_t = None
        self.codes = codes

    @property
    def device(self) -> torch.device:
        return self.codes.device

    @property
    def scale(self) -> float:
        """Per-tensor scale (tensor mode) or the largest block scale (block32). Syncs."""
        if self.mode == "tensor":
            return float(self.scale_t.item())
        return float(self.block_scales.float().max().item())

    @property
    def payload_nbytes(self) -> int:
        """Physical bytes: one per element plus the f32 scale (keyquant.py:46-49),
        or plus one fp16 per 32 elements in block32 mode."""
        n = self.geometry.elements_per_tensor
        return n + (4 if self.mode == "tensor" else 2 * block32_count(n))


def quantize_k(tensor: KvTensor, *, k_scale_mode: str = "tensor") -> QuantizedKeyBlock:
    """Quantize one layer's K to int8 on the GPU (keyquant.py:52-65)."""
    from .pool import _encode_layers

    return _encode_layers([tensor], [None], tensor.geometry, None, None, k_scale_mode)[0][0]


def dequantize_k(block: QuantizedKeyBlock, *, dtype: torch.dtype = torch.float32) -> KvTensor:
    """codes * scale in f32 (keyquant.py:68-71), on the GPU."""
    g = block.geometry
    out = torch.empty(g.tensor_shape, dtype=dtype, device=block.device)
    _codec.decode(
        num_vectors=g.vectors_per_tensor, head_dim=g.head_dim, out_dtype=dtype,
        k_mode=K_MODES[block.mode], k_codes=[block.codes],
        k_scale=[block.scale_t] if block.mode == "tensor" else None,
        k_bscale=[block.block_scales] if block.mode == "block32" else None,
        v_packed=None, v_scales=None, centroids=np.zeros(8), sign_seed=None,
        k_out=[out], v_out=None, device=block.device)
    return KvTensor(g, out)
