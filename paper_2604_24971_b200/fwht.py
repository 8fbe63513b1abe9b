"""Standalone Walsh-Hadamard rotation helpers (kvpool/fwht.py API).

The hot path never calls these: the rotation is fused into the encode and
decode kernels. They exist so code written against kvpool keeps working;
numpy inputs are transformed on the host exactly as the reference does,
torch inputs on their own device with the same stage order.
"""

from __future__ import annotations

import numpy as np
import torch


def hadamard_order(d: int) -> int:
    if d < 1 or d & (d - 1):
        raise ValueError(f"transform length must be a power of two, got {d}")
    return d


def _fwht_torch(x: torch.Tensor) -> torch.Tensor:
    d = hadamard_order(x.shape[-1])
    y = x.contiguous().clone()
    h = 1
    while h < d:
        v = y.view(*y.shape[:-1], d // (2 * h), 2, h)
        lo = v[..., 0, :].clone()
        hi = v[..., 1, :]
        v[..., 0, :] = lo + hi
        v[..., 1, :] = lo - hi
        h *= 2
    return y


def _fwht_numpy(x: np.ndarray) -> np.ndarray:
    d = hadamard_order(x.shape[-1])
    y = np.array(x, copy=True, order="C")
    h = 1
    while h < d:
        v = y.reshape(y.shape[:-1] + (d // (2 * h), 2, h))
        lo = v[..., 0, :].copy()
        hi = v[..., 1, :]
        v[..., 0, :] = lo + hi
        v[..., 1, :] = lo - hi
        h *= 2
    return y


def fwht_inplace(vec) -> None:
    """Unnormalised FWHT of the last axis, in place (fwht.py:24-41)."""
    if isinstance(vec, torch.Tensor):
        vec.copy_(_fwht_torch(vec))
    else:
        vec[...] = _fwht_numpy(np.asarray(vec))


def _rotate(vec):
    if isinstance(vec, torch.Tensor):
        dt = vec.dtype if vec.dtype in (torch.float32, torch.float64) else torch.float64
        y = _fwht_torch(vec.to(dt))
        return y / torch.tensor(float(np.sqrt(vec.shape[-1])), dtype=dt, device=vec.device)
    arr = np.asarray(vec)
    dt = arr.dtype if arr.dtype in (np.float32, np.float64) else np.dtype(np.float64)
    y = _fwht_numpy(arr.astype(dt))
    y /= dt.type(np.sqrt(arr.shape[-1]))
    return y


def rotate_forward(vec):
    """H x / sqrt(d) (orthogonal, norm preserving)."""
    return _rotate(vec)


def rotate_inverse(vec):
    """Inverse of rotate_forward (the rotation is an involution)."""
    return _rotate(vec)
