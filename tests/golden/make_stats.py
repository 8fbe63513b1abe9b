"""LayerStats goldens from the reference's build_pool (kvpool/pool.py:274-288).

Run in the build container (imports the reference read-only):

    NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_stats.py

Writes tests/golden/stats.npz: for each case the input dump and, per layer,
(k_scale, k_mse, k_max_err, v_mse, v_nmse) as float64.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "stats.npz"
# name: (L, H, d, T, seed, sign_seed, bf16-valued inputs)
CASES = {"d128": (2, 2, 128, 100, 5, None, False), "d64_sign": (2, 2, 64, 129, 6, 7, False),
         "bf16vals": (2, 2, 128, 64, 8, None, True)}


def main() -> None:
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_golden")
    sys.path.insert(0, str(REF))
    from kvpool import KvDump, KvTensor, ModelGeometry, build_pool, synth_gaussian_dump  # noqa: E402

    out = {}
    for name, (L, H, d, T, seed, sign, bf16) in CASES.items():
        g = ModelGeometry(num_layers=L, kv_heads=H, head_dim=d, seq_len=T)
        dump = synth_gaussian_dump(g, seed=seed)
        if bf16:  # values exactly representable in bf16 (the bf16-input path)
            def rb(x):
                u = x.view(np.uint32)
                return ((u + 0x7FFF + ((u >> 16) & 1)) & 0xFFFF0000).astype(np.uint32).view(np.float32)
            dump = KvDump(g, tuple((KvTensor(g, rb(k.values)), KvTensor(g, rb(v.values))) for k, v in dump.layers))
        pool = build_pool(dump, sign_seed=sign)
        out[f"{name}/geom"] = np.array([L, H, d, T, -1 if sign is None else sign, int(bf16)])
        for li, (k, v) in enumerate(dump.layers):
            out[f"{name}/k_in/{li}"] = k.values
            out[f"{name}/v_in/{li}"] = v.values
            st = pool.build_stats[li]
            out[f"{name}/stats/{li}"] = np.array([st.k_scale, st.k_mse, st.k_max_err, st.v_mse, st.v_nmse])
    np.savez_compressed(OUT, **out)
    print("wrote", OUT)


if __name__ == "__main__":
    main()
