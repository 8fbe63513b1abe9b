"""PKVP v1 snapshots written by the reference's own save_pool (VERDICT r01
missing #5; kvpool/pool.py:301-345, pinned by pkg/tests/test_pool.py:205-247).

Run in the build container (imports the reference read-only):

    NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_pkvp.py

Writes tests/golden/pkvp/{unpacked,packed,packed_sign}.pkvp plus
tests/golden/pkvp/expect.npz: the dump the pools were built from and the
reference's get_kv_for_layer output at 16 and 32 bits for every layer.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "pkvp"
CASES = {"unpacked": (False, None), "packed": (True, None), "packed_sign": (True, 9)}


def main() -> None:
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_golden")
    sys.path.insert(0, str(REF))
    from kvpool import ModelGeometry, build_pool, load_pool, save_pool, synth_gaussian_dump  # noqa: E402

    OUT.mkdir(exist_ok=True)
    g = ModelGeometry(num_layers=2, kv_heads=2, head_dim=64, seq_len=40)
    dump = synth_gaussian_dump(g, seed=3)
    out = {"geom": np.array([g.num_layers, g.batch, g.kv_heads, g.seq_len, g.head_dim])}
    for li, (k, v) in enumerate(dump.layers):
        out[f"k_in/{li}"] = k.values
        out[f"v_in/{li}"] = v.values
    for name, (packed, seed) in CASES.items():
        pool = build_pool(dump, sign_seed=seed)
        path = OUT / f"{name}.pkvp"
        save_pool(pool, path, packed=packed)
        back = load_pool(path)  # the reference reads its own file back
        for bits in (16, 32):
            view = back.attach(bits)
            for li in range(g.num_layers):
                kd, vd = view.get_kv_for_layer(li)
                out[f"{name}/k{bits}/{li}"] = kd.values
                out[f"{name}/v{bits}/{li}"] = vd.values
    np.savez_compressed(OUT / "expect.npz", **out)
    print("wrote", sorted(p.name for p in OUT.iterdir()))


if __name__ == "__main__":
    main()
