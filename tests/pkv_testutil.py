"""Shared helpers for the test suite (importable as a top-level module)."""

from __future__ import annotations


def golden_case(golden, name):
    L, B, H, T, D, seed = (int(x) for x in golden[f"{name}/geom"])
    return dict(L=L, B=B, H=H, T=T, D=D, sign_seed=None if seed < 0 else seed)


def oracle_layer(args):
    """Worker (spawn-safe): the oracle's codes for one layer.
    args = (k f32, v f32, sign_seed, k_mode) -> dict of arrays."""
    import numpy as np

    from oracle import kvpool_oracle as O

    k, v, sign_seed, k_mode = args
    out = {}
    if k_mode == "tensor":
        out["k_scale"], out["k_codes"] = O.quantize_k_tensor(k)
    else:
        out["k_bscale"], out["k_codes"] = O.quantize_k_block32(k)
    out["v_codes"], out["v_scales"] = O.quantize_v(v, sign_seed=sign_seed)
    out["v_scales"] = np.ascontiguousarray(out["v_scales"])
    return out


def oracle_layers(pairs, sign_seed=None, k_mode="tensor", procs=None):
    """oracle_layer over [(k, v)] on a spawn process pool (CUDA-safe)."""
    import multiprocessing as mp
    import os
    from concurrent.futures import ProcessPoolExecutor

    procs = procs or min(len(pairs), max(1, (os.cpu_count() or 2) - 1), 16)
    work = [(k, v, sign_seed, k_mode) for k, v in pairs]
    if procs <= 1:
        return [oracle_layer(w) for w in work]
    with ProcessPoolExecutor(max_workers=procs, mp_context=mp.get_context("spawn")) as ex:
        return list(ex.map(oracle_layer, work))
