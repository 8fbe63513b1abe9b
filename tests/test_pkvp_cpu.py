"""PKVP v1 snapshots written by the reference (tests/golden/make_pkvp.py):
the oracle's reader decodes them to exactly the reference's own
get_kv_for_layer output (kvpool/pool.py:229-237, 348-432). CPU only; the GPU
load / byte-identical save is tests/test_gpu_pkvp.py."""

from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from oracle import kvpool_oracle as O

PK = Path(__file__).resolve().parent / "golden" / "pkvp"


@pytest.mark.parametrize("name", ["unpacked", "packed", "packed_sign"])
@pytest.mark.parametrize("bits", [16, 32])
def test_reference_snapshot_decodes_to_reference_output(name, bits):
    snap = O.read_pkvp((PK / f"{name}.pkvp").read_bytes())
    with np.load(PK / "expect.npz") as z:
        for li, (scale, kc, vc, vs) in enumerate(snap["layers"]):
            kd, vd = O.decode_layer(kc, scale, vc, vs, bits, sign_seed=snap["sign_seed"])
            assert np.array_equal(kd.view(np.uint32), z[f"{name}/k{bits}/{li}"].view(np.uint32))
            assert np.array_equal(vd.view(np.uint32), z[f"{name}/v{bits}/{li}"].view(np.uint32))


def test_snapshot_codes_are_the_oracle_codes():
    snap = O.read_pkvp((PK / "packed_sign.pkvp").read_bytes())
    with np.load(PK / "expect.npz") as z:
        for li, (scale, kc, vc, vs) in enumerate(snap["layers"]):
            s, k = O.quantize_k_tensor(z[f"k_in/{li}"])
            c, sc = O.quantize_v(z[f"v_in/{li}"], sign_seed=9)
            assert scale == s and np.array_equal(kc, k) and np.array_equal(vc, c)
            assert np.array_equal(vs.view(np.uint32), sc.view(np.uint32))
