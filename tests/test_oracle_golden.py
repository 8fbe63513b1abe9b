"""Pin the CPU oracle (oracle/kvpool_oracle.py) before trusting it as the checker.

Against (a) golden vectors produced by the reference kvpool itself
(tests/golden/make_golden.py) and (b) the reference's own known-answer tests,
restated (pkg/tests/test_keyquant.py, test_valuequant.py, test_pool.py,
test_fwht.py, test_acceptance.py).
"""

from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest

from oracle import kvpool_oracle as O
from pkv_testutil import golden_case

POOL_CASES = ["c1mini", "d128", "d128_sign", "d64_batch2", "d8", "d16", "d32", "d256", "bf16in", "laplace"]


@pytest.mark.parametrize("name", POOL_CASES)
def test_oracle_codec_matches_reference_goldens(golden, name):
    c = golden_case(golden, name)
    for li in range(c["L"]):
        k = golden[f"{name}/k_in/{li}"]
        v = golden[f"{name}/v_in/{li}"]
        scale, kc = O.quantize_k_tensor(k)
        assert scale == float(golden[f"{name}/k_scale/{li}"][0])
        assert np.array_equal(kc, golden[f"{name}/k_codes/{li}"])
        vc, vs = O.quantize_v(v, c["sign_seed"])
        assert np.array_equal(vc, golden[f"{name}/v_codes/{li}"])
        assert np.array_equal(vs.view(np.uint32), golden[f"{name}/v_scales/{li}"].view(np.uint32))
        assert O.pack3(vc) == golden[f"{name}/v_packed/{li}"].tobytes()
        assert np.array_equal(O.unpack3(O.pack3(vc), vc.size).reshape(vc.shape), vc)
        for bits in (16, 32):
            kd, vd = O.decode_layer(kc, scale, vc, vs, bits, c["sign_seed"])
            assert np.array_equal(kd.view(np.uint32), golden[f"{name}/k{bits}/{li}"].view(np.uint32))
            assert np.array_equal(vd.view(np.uint32), golden[f"{name}/v{bits}/{li}"].view(np.uint32))


@pytest.mark.parametrize("name", ["c1mini", "d128_sign", "d8"])
def test_oracle_transcript_checksums(golden, name):
    c = golden_case(golden, name)
    sums = []
    for li in range(c["L"]):
        sums.append((O.tensor_checksum(golden[f"{name}/k16/{li}"]), O.tensor_checksum(golden[f"{name}/v16/{li}"])))
    assert np.array_equal(np.array(sums, dtype=np.uint64), golden[f"{name}/checksums16"])


def test_oracle_value_ties(golden):
    vc, vs = O.quantize_v(golden["tie/v_in"])
    assert np.array_equal(vc, golden["tie/v_codes"])
    assert np.array_equal(vs, golden["tie/v_scales"])


@pytest.mark.parametrize("kat", ["sym", "grid", "half", "halfgrid_all"])
def test_oracle_key_known_answers(golden, kat):
    vals = golden[f"kat/{kat}/in"]
    s, c = O.quantize_k_tensor(vals.reshape(1, 1, -1, 1))
    assert s == float(golden[f"kat/{kat}/scale"][0])
    assert np.array_equal(c.reshape(-1), golden[f"kat/{kat}/codes"])


def test_key_kats_restated():
    # pkg/tests/test_keyquant.py:41-78
    s, c = O.quantize_k_tensor(np.array([-2.54, 0.0, 2.54], dtype=np.float32))
    assert s == pytest.approx(0.02, rel=1e-6) and c.tolist() == [-127, 0, 127]
    s, c = O.quantize_k_tensor(np.array([127, 2.5, -2.5, 0.5, -0.5, 10.5]) * 2.0**-6)
    assert s == 2.0**-6 and c.tolist() == [127, 3, -3, 1, -1, 11]
    s, c = O.quantize_k_tensor(np.zeros(3, dtype=np.float32))
    assert s == 0.0 and not c.any()


def test_pinned_midpoints_and_table():
    # pkg/tests/test_valuequant.py:24-25, 56-59, 91-94
    mids = O.GAUSSIAN_3BIT_MIDPOINTS
    assert np.allclose(mids, [-1.748, -1.05, -0.5005, 0.0, 0.5005, 1.05, 1.748])
    c = O.GAUSSIAN_3BIT_CENTROIDS
    for i, m in enumerate(mids):
        exact = (Fraction(float(c[i])) + Fraction(float(c[i + 1]))) / 2
        assert Fraction(float(m)) <= exact < Fraction(float(np.nextafter(m, np.inf)))
        assert int(np.searchsorted(mids, m, side="left")) == i
        assert int(np.searchsorted(mids, np.nextafter(m, np.inf), side="left")) == i + 1


def test_pairwise_sum_order_is_numpy_mean():
    # the GPU replay (pkv_common.cuh pairwise_sumsq) follows numpy's pairwise
    # summation; restate it in Python and check against np.mean bit for bit
    def pw(a):
        n = len(a)
        if n < 8:
            r = 0.0
            for x in a:
                r += x * x
            return r
        if n <= 128:
            r = [a[j] * a[j] for j in range(8)]
            i = 8
            while i < n - (n % 8):
                for j in range(8):
                    r[j] += a[i + j] * a[i + j]
                i += 8
            res = ((r[0] + r[1]) + (r[2] + r[3])) + ((r[4] + r[5]) + (r[6] + r[7]))
            while i < n:
                res += a[i] * a[i]
                i += 1
            return res
        n2 = n // 2
        n2 -= n2 % 8
        return pw(a[:n2]) + pw(a[n2:])

    rng = np.random.default_rng(1)
    for d in (8, 16, 32, 64, 128, 256):
        x = rng.normal(size=(40, d))
        want = np.mean(np.square(x), axis=-1)
        got = np.array([pw([float(t) for t in row]) / d for row in x])
        assert np.array_equal(got, want), d


def test_fwht_matches_dense_hadamard():
    # pkg/tests/test_fwht.py:22-37
    from scipy.linalg import hadamard

    rng = np.random.default_rng(0)
    for d in (2, 8, 64, 128):
        x = rng.normal(size=(5, d))
        assert np.allclose(O.fwht_last_axis(x), x @ hadamard(d).T)
        assert np.allclose(O.rotate(O.rotate(x)), x)


def test_block32_oracle_properties():
    rng = np.random.default_rng(5)
    x = rng.normal(0, 0.3, size=(1, 4, 33, 64)).astype(np.float32)
    x[0, 0, 0, :32] = 0.0  # an all-zero block
    s16, codes = O.quantize_k_block32(x)
    assert s16.dtype == np.float16 and s16.size == x.size // 32
    assert np.abs(codes.astype(np.int32)).max() <= 127
    back = O.dequantize_k_block32(codes, s16)
    err = np.abs(back - x).reshape(-1, 32).max(axis=1)
    assert (err <= s16.astype(np.float64) / 2 * (1 + 1e-6)).all()
    assert s16[0] == 0 and not codes.reshape(-1)[:32].any()


def test_guard_band_covers_fp32_fast_path_error():
    # the encode kernel's fast path computes z in fp32 (FWHT of f32 inputs,
    # times f32 1/||x||). The bound behind its guard band must cover the
    # observed error with margin.
    rng = np.random.default_rng(3)
    for d in (64, 128, 256):
        x = rng.normal(size=(4000, d)).astype(np.float32)
        u32 = O.fwht_last_axis(x)  # f32 arithmetic, same stage order
        n64 = np.sqrt(np.sum(x.astype(np.float64) ** 2, axis=-1))
        z32 = u32 * (1.0 / n64).astype(np.float32)[:, None]
        z64 = O.rotate(x.astype(np.float64)) / (n64 / np.sqrt(d))[:, None]
        err = np.abs(z32.astype(np.float64) - z64).max()
        u = 2.0**-24
        bound = u * (np.log2(d) * np.sqrt(d) + 6.0)
        assert err < bound / 2, (d, err, bound)


def test_compression_ratio_is_32_over_11():
    # pkg/tests/test_acceptance.py:57-61
    r = O.compression_ratio_exact(8, 3, 16)
    assert r == Fraction(32, 11) and f"{float(r):.2f}" == "2.91"


def test_fma_adversarial_fixture_is_adversarial():
    """tests/golden/adversarial_fma.npz (make_adversarial.py, from the
    reference's quantize_v): the oracle reproduces it, and for every vector a
    sum of squares with r += v*v contracted to one fma rounding gives a
    different f32 scale than numpy's order (valuequant.py:207)."""
    import importlib.util
    from pathlib import Path

    here = Path(__file__).resolve().parent / "golden"
    spec = importlib.util.spec_from_file_location("make_adversarial", here / "make_adversarial.py")
    M = importlib.util.module_from_spec(spec)
    spec.loader.exec_module(M)
    with np.load(here / "adversarial_fma.npz") as z:
        v, codes, scales = z["v_in"], z["v_codes"], z["v_scales"]
    assert v.shape[2] >= 8
    c, s = O.quantize_v(v)
    assert np.array_equal(c, codes) and np.array_equal(s.view(np.uint32), scales.view(np.uint32))
    for i in range(v.shape[2]):
        rot = O.rotate(v[0, 0, i].astype(np.float64))
        assert M.f32_scale(M.sumsq_numpy_order(rot)) == scales[0, 0, i]
        assert M.f32_scale(M.sumsq_contracted(rot)) != scales[0, 0, i]
