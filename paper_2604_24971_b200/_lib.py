"""ctypes binding of libpolykv.so (include/polykv.h).

The product path has no CPU fallback: if the library is missing or a CUDA
device is absent, codec entry points raise instead of computing anything on
the host.
"""

from __future__ import annotations

import ctypes
import os
import threading
from pathlib import Path

from ._build import LIB_PATH

PKV_OK = 0
PKV_ERR_CUDA = -3
PKV_F32 = 0
PKV_BF16 = 1
PKV_K_TENSOR = 0
PKV_K_BLOCK32 = 1
PKV_FLAG_K_NONFINITE = 0x1
PKV_FLAG_V_NONFINITE = 0x2
PKV_FLAG_K_SCALE_OVERFLOW = 0x4
PKV_FLAG_BAD_CODE = 0x8
PKV_MAX_LAYERS_PER_LAUNCH = 64

_lock = threading.Lock()
_lib: ctypes.CDLL | None = None

c_void_p = ctypes.c_void_p
c_int = ctypes.c_int
c_i64 = ctypes.c_int64
c_size = ctypes.c_size_t
c_u64 = ctypes.c_uint64
P = ctypes.POINTER

# symbol -> (restype, argtypes); mirrors include/polykv.h
SIGNATURES: dict[str, tuple] = {
    "pkv_abi_version": (c_int, []),
    "pkv_status_string": (ctypes.c_char_p, [c_int]),
    "pkv_reload_tuning": (c_int, []),
    "pkv_last_cuda_error": (ctypes.c_char_p, []),
    "pkv_v_head_dim_supported": (c_int, [c_int]),
    "pkv_encode_workspace_bytes": (c_size, [c_int, c_i64, c_int]),
    "pkv_encode": (
        c_int,
        [c_int, c_i64, c_int, c_int, P(c_void_p), P(c_void_p), c_int, P(c_void_p), P(c_void_p),
         P(c_void_p), P(c_void_p), P(c_void_p), P(ctypes.c_double), P(ctypes.c_uint32), c_void_p,
         c_void_p, c_void_p, c_void_p, c_size, c_void_p],
    ),
    "pkv_k_absmax": (c_int, [c_int, c_i64, c_int, P(c_void_p), c_void_p, c_void_p]),
    "pkv_layer_stats_workspace_bytes": (c_size, [c_int, c_i64]),
    "pkv_layer_stats": (c_int, [c_int, c_i64, c_int, P(c_void_p), P(c_void_p), P(c_void_p), P(c_void_p), c_void_p,
                                c_void_p, c_size, c_void_p]),
    "pkv_decode": (
        c_int,
        [c_int, c_i64, c_int, c_int, c_int, P(c_void_p), P(c_void_p), P(c_void_p), P(c_void_p),
         P(c_void_p), P(ctypes.c_double), P(ctypes.c_uint32), P(c_void_p), P(c_void_p), c_void_p],
    ),
    "pkv_unpack_codes": (c_int, [c_void_p, c_i64, c_void_p, c_void_p]),
    "pkv_pack_codes": (c_int, [c_void_p, c_i64, c_void_p, c_void_p, c_void_p]),
    "pkv_attention_workspace_bytes": (c_size, [c_int, c_int, c_int, c_int, c_i64]),
    "pkv_decode_attention": (
        c_int,
        [c_int, c_int, c_int, c_int, c_i64, c_int, c_void_p, c_int, c_void_p, c_void_p, c_void_p,
         c_void_p, c_void_p, P(ctypes.c_double), P(ctypes.c_uint32), c_void_p, c_void_p, c_void_p,
         c_int, c_int, ctypes.c_float, c_int, c_void_p, c_void_p, c_size, c_void_p],
    ),
    "pkv_selftest": (c_i64, [c_int, c_void_p, c_size, c_void_p]),
    "pkv_fnv1a64": (c_u64, [c_void_p, c_size]),
    "pkv_fnv1a64_bf16_as_f32": (c_u64, [c_void_p, c_size]),
}


class LibraryError(RuntimeError):
    """libpolykv.so is missing, stale, or returned an error status."""


def library_path() -> Path:
    """lib/libpolykv.so, or lib/variants/libpolykv_<name>.so when
    PKV_LIB_VARIANT=<name> is set (tuning builds from _build.build_variant)."""
    name = os.environ.get("PKV_LIB_VARIANT") or None
    return LIB_PATH.parent / "variants" / f"libpolykv_{name}.so" if name else LIB_PATH


def load() -> ctypes.CDLL:
    """Load (never build) libpolykv.so and bind every C ABI symbol."""
    global _lib
    if _lib is not None:
        return _lib
    with _lock:
        if _lib is not None:
            return _lib
        path = library_path()
        if not path.exists():
            raise LibraryError(
                f"{path} not found: build it with `python -m paper_2604_24971_b200._build` "
                "or __graft_entry__.build(); there is no CPU fallback"
            )
        lib = ctypes.CDLL(str(path))
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def reload_tuning() -> None:
    """Re-read the PKV_* scheduling knobs from os.environ (they are otherwise
    read once per process; see include/polykv.h pkv_reload_tuning)."""
    load().pkv_reload_tuning()


def check(status: int, what: str) -> None:
    if status != PKV_OK:
        lib = load()
        msg = lib.pkv_status_string(status).decode()
        if status == PKV_ERR_CUDA:
            msg += f" [{lib.pkv_last_cuda_error().decode()}]"
        raise LibraryError(f"{what} failed: {msg} (status {status})")


def ptr_array(ptrs) -> ctypes.Array:
    arr = (c_void_p * max(1, len(ptrs)))()
    for i, p in enumerate(ptrs):
        arr[i] = p
    return arr
