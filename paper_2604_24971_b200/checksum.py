"""64-bit FNV-1a fingerprints (kvpool/checksum.py API), computed by libpolykv.so's
host code. FNV-1a is byte-serial, so it stays on the CPU after a D2H copy."""

from __future__ import annotations

import numpy as np
import torch

from . import _codec

FNV64_OFFSET = 0xCBF29CE484222325
FNV64_PRIME = 0x100000001B3


def fnv1a64(buf) -> int:
    """FNV-1a 64-bit hash of a byte buffer or array's bytes."""
    if isinstance(buf, torch.Tensor):
        buf = buf.detach().cpu().contiguous().view(torch.uint8).numpy()
    return _codec.fnv1a64_bytes(buf)


def tensor_checksum(values) -> int:
    """FNV-1a over the little-endian f32 image, row-major (checksum.py:55-62).

    bf16 tensors hash as their exact f32 widening, so a decode_bits=16 view
    fingerprints exactly like the reference's bf16-rounded f32 arrays.
    """
    if isinstance(values, torch.Tensor):
        return _codec.fnv1a64_tensor_f32_image(values.detach())
    arr = np.ascontiguousarray(values, dtype="<f4")
    return _codec.fnv1a64_bytes(arr)
