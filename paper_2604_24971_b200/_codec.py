"""torch <-> libpolykv.so glue: every codec call of the package goes through here.

Tensors are handed to the C ABI as raw device pointers together with the
caller's current CUDA stream; the library only enqueues work. There is no
host implementation behind any of these functions.
"""

from __future__ import annotations

import ctypes

import numpy as np
import torch

from . import _lib
from ._lib import PKV_BF16, PKV_F32, check, load, ptr_array

_DTYPE_CODE = {torch.float32: PKV_F32, torch.bfloat16: PKV_BF16}


class CudaRequiredError(RuntimeError):
    """The codec runs only on a CUDA device; there is no CPU fallback."""


def require_device(device=None) -> torch.device:
    if not torch.cuda.is_available():
        raise CudaRequiredError(
            "paper_2604_24971_b200 runs its codec on a CUDA (sm_100a) device only; "
            "no CUDA device is visible"
        )
    load()
    if device is None:
        return torch.device("cuda", torch.cuda.current_device())
    d = torch.device(device)
    if d.type != "cuda":
        raise CudaRequiredError(f"device {d} is not a CUDA device")
    return d if d.index is not None else torch.device("cuda", torch.cuda.current_device())


def stream_ptr(device: torch.device) -> int:
    return torch.cuda.current_stream(device).cuda_stream


def dtype_code(t: torch.Tensor) -> int:
    try:
        return _DTYPE_CODE[t.dtype]
    except KeyError:
        raise TypeError(f"unsupported tensor dtype {t.dtype}; use float32 or bfloat16") from None


def centroid_array(centroids) -> ctypes.Array:
    c = np.asarray(centroids, dtype=np.float64).reshape(-1)
    if c.size != 8:
        raise ValueError("the B200 codec stores 3-bit codes: need exactly 8 centroids")
    return (ctypes.c_double * 8)(*[float(x) for x in c])


def sign_word_array(sign_seed, head_dim: int):
    """Sign diagonal (valuequant.py:183-190) as LSB-first uint32 words, or None."""
    if sign_seed is None:
        return None
    rng = np.random.default_rng(sign_seed)
    neg = (rng.integers(0, 2, size=head_dim) * 2 - 1) < 0
    words = [0] * ((head_dim + 31) // 32)
    for i in np.flatnonzero(neg):
        words[i // 32] |= 1 << int(i % 32)
    return (ctypes.c_uint32 * len(words))(*words)


def _p(t: torch.Tensor | None) -> int | None:
    return None if t is None else t.data_ptr()


def encode(
    *,
    num_vectors: int,
    head_dim: int,
    k_in: list[torch.Tensor] | None,
    v_in: list[torch.Tensor] | None,
    k_mode: int,
    k_codes: list[torch.Tensor] | None,
    k_scale: list[torch.Tensor] | None,
    k_bscale: list[torch.Tensor] | None,
    v_packed: list[torch.Tensor] | None,
    v_scales: list[torch.Tensor] | None,
    centroids,
    sign_seed,
    status: torch.Tensor,
    replay: torch.Tensor | None,
    device: torch.device,
    k_layer_max: torch.Tensor | None = None,
) -> None:
    """pkv_encode. k_layer_max: optional int32 [L] device tensor of external
    per-layer max|K| bit patterns (head-sharded pools); None = own pass."""
    lib = load()
    ins = k_in if k_in is not None else v_in
    L = len(ins)
    dt = dtype_code(ins[0])
    for t in (k_in or []) + (v_in or []):
        if t.dtype != ins[0].dtype:
            raise TypeError("all inputs of one encode call must share a dtype")
        if t.device != device or not t.is_contiguous():
            raise ValueError("encode inputs must be contiguous tensors on the pool device")
    ws_bytes = lib.pkv_encode_workspace_bytes(L, num_vectors, head_dim)
    ws = torch.empty((ws_bytes + 3) // 4, dtype=torch.int32, device=device)
    arr = lambda ts: None if ts is None else ptr_array([_p(t) for t in ts])  # noqa: E731
    with torch.cuda.device(device):  # the library launches on the current device
        rc = lib.pkv_encode(
            L, num_vectors, head_dim, dt,
            arr(k_in), arr(v_in), k_mode,
            arr(k_codes), arr(k_scale), arr(k_bscale), arr(v_packed), arr(v_scales),
            centroid_array(centroids), sign_word_array(sign_seed, head_dim),
            status.data_ptr(), _p(replay), _p(k_layer_max), ws.data_ptr(), ws_bytes, stream_ptr(device),
        )
    check(rc, "pkv_encode")


def k_absmax(k_in: list[torch.Tensor], out: torch.Tensor, device: torch.device) -> torch.Tensor:
    """pkv_k_absmax: out[l] = f32 bit pattern of max|k_in[l]| (int32 [L] on device)."""
    lib = load()
    for t in k_in:
        if t.device != device or not t.is_contiguous() or t.dtype != k_in[0].dtype:
            raise ValueError("absmax inputs must be contiguous same-dtype tensors on the device")
    with torch.cuda.device(device):
        rc = lib.pkv_k_absmax(len(k_in), k_in[0].numel(), dtype_code(k_in[0]),
                              ptr_array([t.data_ptr() for t in k_in]), out.data_ptr(), stream_ptr(device))
    check(rc, "pkv_k_absmax")
    return out


def decode(
    *,
    num_vectors: int,
    head_dim: int,
    out_dtype: torch.dtype,
    k_mode: int,
    k_codes: list[torch.Tensor] | None,
    k_scale: list[torch.Tensor] | None,
    k_bscale: list[torch.Tensor] | None,
    v_packed: list[torch.Tensor] | None,
    v_scales: list[torch.Tensor] | None,
    centroids,
    sign_seed,
    k_out: list[torch.Tensor] | None,
    v_out: list[torch.Tensor] | None,
    device: torch.device,
) -> None:
    lib = load()
    L = len(k_codes if k_codes is not None else v_packed)
    arr = lambda ts: None if ts is None else ptr_array([_p(t) for t in ts])  # noqa: E731
    with torch.cuda.device(device):
        rc = lib.pkv_decode(
            L, num_vectors, head_dim, _DTYPE_CODE[out_dtype], k_mode,
            arr(k_codes), arr(k_scale), arr(k_bscale), arr(v_packed), arr(v_scales),
            centroid_array(centroids), sign_word_array(sign_seed, head_dim),
            arr(k_out), arr(v_out), stream_ptr(device),
        )
    check(rc, "pkv_decode")


def unpack_codes(packed: torch.Tensor, count: int, out: torch.Tensor) -> None:
    with torch.cuda.device(packed.device):
        rc = load().pkv_unpack_codes(packed.data_ptr(), count, out.data_ptr(), stream_ptr(packed.device))
    check(rc, "pkv_unpack_codes")


def pack_codes(codes: torch.Tensor, count: int, out: torch.Tensor, bad: torch.Tensor) -> None:
    with torch.cuda.device(codes.device):
        rc = load().pkv_pack_codes(codes.data_ptr(), count, out.data_ptr(), bad.data_ptr(),
                                   stream_ptr(codes.device))
    check(rc, "pkv_pack_codes")


def fnv1a64_bytes(buf: bytes | bytearray | memoryview | np.ndarray) -> int:
    arr = np.ascontiguousarray(np.frombuffer(buf, dtype=np.uint8) if not isinstance(buf, np.ndarray)
                               else buf.view(np.uint8).reshape(-1))
    return int(load().pkv_fnv1a64(arr.ctypes.data, arr.size))


def fnv1a64_tensor_f32_image(t: torch.Tensor) -> int:
    """FNV-1a of the LE f32 image of a (host) f32 or bf16 tensor."""
    t = t.contiguous()
    if t.device.type != "cpu":
        t = t.cpu()
    if t.dtype == torch.bfloat16:
        u16 = t.view(torch.int16).numpy()
        return int(load().pkv_fnv1a64_bf16_as_f32(u16.ctypes.data, u16.size))
    a = t.to(torch.float32).numpy()
    return int(load().pkv_fnv1a64(a.ctypes.data, a.nbytes))


__all__ = [
    "CudaRequiredError", "require_device", "encode", "decode", "unpack_codes", "pack_codes",
    "fnv1a64_bytes", "fnv1a64_tensor_f32_image", "sign_word_array", "centroid_array", "_lib",
]
