"""The C-ABI library: loads, exports every symbol include/polykv.h declares,
and its host-only entry points (FNV-1a, status strings) behave. No GPU."""

from __future__ import annotations

import ctypes
import re
from pathlib import Path

import numpy as np
import pytest

from oracle import kvpool_oracle as O
from paper_2604_24971_b200 import _lib

HEADER = Path(__file__).resolve().parents[1] / "include" / "polykv.h"


def declared_symbols() -> list[str]:
    text = HEADER.read_text()
    text = re.sub(r"/\*.*?\*/", "", text, flags=re.S)
    return sorted(set(re.findall(r"\b(pkv_[a-z0-9_]+)\s*\(", text)))


@pytest.fixture(scope="module")
def lib():
    from paper_2604_24971_b200 import _build

    _build.build()
    return _lib.load()


def test_header_declares_expected_entry_points():
    syms = declared_symbols()
    for s in ("pkv_encode", "pkv_decode", "pkv_decode_attention", "pkv_fnv1a64"):
        assert s in syms
    assert set(syms) == set(_lib.SIGNATURES), "ctypes binding must mirror include/polykv.h"


def test_library_exports_every_declared_symbol(lib):
    raw = ctypes.CDLL(str(_lib.library_path()))
    for s in declared_symbols():
        assert hasattr(raw, s), s


def test_abi_and_status(lib):
    assert lib.pkv_abi_version() == 2
    assert lib.pkv_status_string(0) == b"ok"
    assert b"head_dim" in lib.pkv_status_string(-2)
    assert lib.pkv_v_head_dim_supported(128) == 1 and lib.pkv_v_head_dim_supported(4) == 0
    # per layer: u32 max + u32 published-CTA count (+16); the warp path needs 2L+2 words
    assert lib.pkv_encode_workspace_bytes(32, 8 * 4096, 128) == 32 * 8 + 16
    assert lib.pkv_encode_workspace_bytes(2, 3, 4) == 2 * 8 + 16


def test_invalid_arguments_fail_without_touching_the_device(lib):
    # bad dtype / mode / negative sizes are rejected before any CUDA call
    assert lib.pkv_encode(1, 8, 128, 7, None, None, 0, None, None, None, None, None, None, None,
                          None, None, None, 0, None) == -1
    assert lib.pkv_decode(-1, 8, 128, 0, 0, None, None, None, None, None, None, None, None, None,
                          None) == -1
    assert lib.pkv_decode_attention(1, 8, 4, 96, 10, 0, None, 0, None, None, None, None, None, None,
                                    None, None, None, None, 0, 1.0, 0, None, None, 0, None) == -2


def test_fnv_host_functions_match_oracle(lib):
    rng = np.random.default_rng(0)
    data = rng.integers(0, 256, size=4097, dtype=np.uint8)
    assert lib.pkv_fnv1a64(data.ctypes.data, data.size) == O.fnv1a64(data.tobytes())
    f = rng.normal(size=333).astype(np.float32)
    bf = O.round_to_bfloat16(f)
    u16 = (bf.view(np.uint32) >> 16).astype(np.uint16)
    assert lib.pkv_fnv1a64_bf16_as_f32(u16.ctypes.data, u16.size) == O.tensor_checksum(bf)
