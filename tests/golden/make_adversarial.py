"""Adversarial value vectors for the exact fp64 replay.

Each vector's RMS lands within a few fp64 ulps of an f32 rounding midpoint,
so (a) the GPU fast path cannot decide the f32 scale and hands the vector to
the fp64 replay (kvpool/valuequant.py:203-211 in numpy's exact order), and
(b) numpy's sum of squares (np.square rounded, then the pairwise add,
valuequant.py:207) and an FMA-contracted sum (r = fma(v, v, r), what nvcc
emits for `r += v * v` by default) give DIFFERENT f32 scales. A replay that
contracts fails on every vector here; the numpy-order replay passes.

Run in the build container (imports the reference read-only):

    NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_adversarial.py

Writes tests/golden/adversarial_fma.npz: v_in [1, 1, N, 128] f32 and the
reference's quantize_v codes / scales for it.
"""

from __future__ import annotations

import os
import sys
from fractions import Fraction
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "adversarial_fma.npz"
D = 128


def fma_exact(a: float, b: float, c: float) -> float:
    """fl(a * b + c) with one rounding (float(Fraction) rounds to nearest even)."""
    return float(Fraction(a) * Fraction(b) + Fraction(c))


def sumsq_numpy_order(rot: np.ndarray) -> float:
    """numpy's pairwise sum of np.square(rot) for n == 128 (8 accumulators)."""
    sq = [float(x) * float(x) for x in rot]  # np.square: one rounding each
    r = sq[:8]
    for i in range(8, len(sq), 8):
        r = [r[j] + sq[i + j] for j in range(8)]
    return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))


def sumsq_contracted(rot: np.ndarray) -> float:
    """The same order with r[j] += v * v contracted to one fma rounding."""
    v = [float(x) for x in rot]
    r = [v[j] * v[j] for j in range(8)]
    for i in range(8, len(v), 8):
        r = [fma_exact(v[i + j], v[i + j], r[j]) for j in range(8)]
    return ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))


def f32_scale(S: float) -> np.float32:
    return np.float32(np.sqrt(np.float64(S) / D))


def search(rotate_forward, n_want: int, seed: int = 2024) -> list[np.ndarray]:
    rng = np.random.default_rng(seed)
    found: list[np.ndarray] = []
    tries = 0
    while len(found) < n_want and tries < 4000:
        tries += 1
        x = rng.normal(0.0, np.sqrt(1.0 / D), size=D).astype(np.float32)
        x[1] = 0.0
        S = float(np.sum(x.astype(np.float64) ** 2))
        rr = np.sqrt(S / D)
        # nearest f32 rounding midpoint of the rms, as a target sum of squares
        f = np.float32(rr)
        nb = np.nextafter(f, np.float32(np.inf) if rr >= float(f) else np.float32(0))
        mid = (float(f) + float(nb)) / 2.0
        target = D * mid * mid
        # coarse: x0 so that the sum sits just below the target
        rest = S - float(x[0]) ** 2
        x0 = np.float32(np.sqrt(max(target - rest, 0.0)))
        while rest + float(x0) ** 2 > target:
            x0 = np.nextafter(x0, np.float32(0))
        x[0] = x0
        gap = target - float(np.sum(x.astype(np.float64) ** 2))
        if gap <= 0:
            continue
        # fine: a small coordinate walks the sum across the target in ~ulp steps
        x1 = np.float32(np.sqrt(gap))
        ups, downs = [x1], [x1]
        for _ in range(300):
            ups.append(np.nextafter(ups[-1], np.float32(np.inf)))
            downs.append(np.nextafter(downs[-1], np.float32(0)))
        for t in [v for pair in zip(ups, downs[1:]) for v in pair]:
            x[1] = t
            rot = rotate_forward(x.astype(np.float64).reshape(1, D))[0]
            s_np, s_fma = sumsq_numpy_order(rot), sumsq_contracted(rot)
            if f32_scale(s_np) != f32_scale(s_fma):
                found.append(x.copy())
                break
    return found


def main() -> None:
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_golden")
    sys.path.insert(0, str(REF))
    from kvpool import KvTensor, ModelGeometry, quantize_v, rotate_forward  # noqa: E402  (the reference)

    vecs = search(rotate_forward, n_want=24)
    assert len(vecs) >= 8, f"only {len(vecs)} adversarial vectors found"
    v = np.stack(vecs).reshape(1, 1, len(vecs), D).astype(np.float32)
    g = ModelGeometry(num_layers=1, kv_heads=1, head_dim=D, seq_len=len(vecs))
    vq = quantize_v(KvTensor(g, v))
    # the numpy-order emulation above must agree with the reference itself
    for i in range(len(vecs)):
        rot = rotate_forward(v[0, 0, i].astype(np.float64).reshape(1, D))[0]
        assert f32_scale(sumsq_numpy_order(rot)) == vq.scales[0, 0, i]
        assert f32_scale(sumsq_contracted(rot)) != vq.scales[0, 0, i]
    np.savez_compressed(OUT, v_in=v, v_codes=vq.codes, v_scales=vq.scales)
    print(f"wrote {OUT}: {len(vecs)} vectors")


if __name__ == "__main__":
    main()
