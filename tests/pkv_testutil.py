"""Shared helpers for the test suite (importable as a top-level module)."""

from __future__ import annotations


def golden_case(golden, name):
    L, B, H, T, D, seed = (int(x) for x in golden[f"{name}/geom"])
    return dict(L=L, B=B, H=H, T=T, D=D, sign_seed=None if seed < 0 else seed)
