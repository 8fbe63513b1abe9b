"""Host-side API behaviour that needs no GPU: names, validation, errors,
accounting, file formats, and the no-CPU-fallback rule."""

from __future__ import annotations

from fractions import Fraction

import numpy as np
import pytest
import torch

import paper_2604_24971_b200 as pk
from oracle import kvpool_oracle as O

REFERENCE_ALL = [
    "AgentCacheView", "BadMagicError", "BenchResult", "Codebook", "CompressionReport", "CorruptBlockError",
    "DistortionBound", "DumpFormatError", "GAUSSIAN_3BIT", "GeometryError", "InjectionTranscript", "KvDump",
    "KvPoolError", "KvTensor", "LayerStats", "MemoryRow", "ModelGeometry", "NonFiniteValuesError",
    "PayloadSizeError", "PplDelta", "QuantizedKeyBlock", "QuantizedValueBlock", "SharedPool", "TranscriptEntry",
    "TruncatedFileError", "UnsealedPoolError", "UnsupportedVersionError", "attach_agent", "build_pool",
    "compression_ratio", "compression_ratio_exact", "dequantize_k", "dequantize_v", "distortion_report",
    "fnv1a64", "format_memory_table", "fwht_inplace", "hadamard_order", "load_pool", "lloyd_max_train",
    "memory_rows_csv", "memory_table", "nearest_centroid", "pack_indices_3bit", "ppl_delta", "quantize_k",
    "quantize_v", "read_dump", "rotate_forward", "rotate_inverse", "round_to_bfloat16", "run_bench",
    "save_pool", "sign_diagonal", "synth_gaussian_dump", "tensor_checksum", "unpack_indices_3bit", "write_dump",
]  # kvpool/__init__.py:73-132


def test_public_names_match_reference():
    for name in REFERENCE_ALL:
        assert hasattr(pk, name), name
    assert pk.SharedKVPool is pk.SharedPool and pk.PooledAgent is pk.AgentCacheView


def test_geometry_validation_and_arithmetic():
    g = pk.ModelGeometry(num_layers=32, kv_heads=8, head_dim=128, seq_len=1837)
    assert g.elements_per_tensor == 1837 * 8 * 128
    assert g.payload_elements == 120_389_632 and g.baseline_cache_nbytes() == 240_779_264  # test_model.py:37-40
    with pytest.raises(pk.GeometryError, match="power of two"):
        pk.ModelGeometry(num_layers=1, kv_heads=1, head_dim=96, seq_len=1)
    with pytest.raises(pk.GeometryError):
        pk.ModelGeometry(num_layers=0, kv_heads=1, head_dim=8, seq_len=1)
    with pytest.raises(pk.GeometryError, match="baseline_bits"):
        pk.ModelGeometry(num_layers=1, kv_heads=1, head_dim=8, seq_len=1, baseline_bits=8)


def test_kvtensor_host_checks():
    g = pk.ModelGeometry(num_layers=1, kv_heads=1, head_dim=4, seq_len=2)
    with pytest.raises(pk.GeometryError, match="shape"):
        pk.KvTensor(g, np.zeros((1, 1, 3, 4), np.float32))
    bad = np.zeros((1, 1, 2, 4), np.float32)
    bad[0, 0, 1, 2] = np.nan
    with pytest.raises(pk.GeometryError, match="NaN or Inf"):
        pk.KvTensor(g, bad)
    t = pk.KvTensor(g, np.ones((1, 1, 2, 4), np.float64))
    assert t.values.dtype == torch.float32 and t.nbytes == 32


def test_codebook_and_coder_match_reference_tables():
    assert np.array_equal(pk.GAUSSIAN_3BIT.midpoints, O.GAUSSIAN_3BIT_MIDPOINTS)
    assert pk.GAUSSIAN_3BIT.is_symmetric()
    for x, want in [(0.0, 3), (1.0, 5), (3.0, 7), (-3.0, 0), (0.245, 4), (-0.245, 3), (0.5, 4)]:
        assert pk.nearest_centroid(x, pk.GAUSSIAN_3BIT) == want  # test_valuequant.py:80-85
    with pytest.raises(ValueError, match="strictly increasing"):
        pk.Codebook(bits=3, centroids=np.array([0, 0, 1, 2, 3, 4, 5, 6.0]))
    assert pk.DistortionBound(3).bound == pytest.approx(0.0425109, abs=1e-6)


def test_ratio_and_memory_table():
    assert pk.compression_ratio_exact(8, 3, 16) == Fraction(32, 11)
    assert f"{pk.compression_ratio(8, 3, 16):.2f}" == "2.91"
    g = pk.ModelGeometry(num_layers=32, kv_heads=8, head_dim=128, seq_len=1837)
    rows = pk.memory_table(g, [1, 3, 5, 10, 15], pk.compression_ratio(8, 3, 16))
    assert {r.agents: round(r.reduction_percent, 1) for r in rows} == {1: 65.6, 3: 88.5, 5: 93.1, 10: 96.6, 15: 97.7}
    assert [round(pk.ppl_delta(b, c).delta_percent, 2) for b, c in [(8.998, 9.141), (10.369, 10.342)]] == [1.59, -0.26]


def test_packing_helpers_and_layout():
    packed = pk.pack_indices_3bit(np.arange(8, dtype=np.uint8))
    word = int.from_bytes(packed, "little")
    assert all((word >> (3 * i)) & 7 == i for i in range(8))
    rng = np.random.default_rng(0)
    for n in (0, 1, 7, 8, 9, 1000):
        c = rng.integers(0, 8, size=n).astype(np.uint8)
        p = pk.pack_indices_3bit(c)
        assert p == O.pack3(c) and np.array_equal(pk.unpack_indices_3bit(p, n), c)


def test_dump_roundtrip_and_format_errors(tmp_path):
    g = pk.ModelGeometry(num_layers=2, kv_heads=2, head_dim=8, seq_len=3)
    d = pk.synth_gaussian_dump(g, seed=0)
    host = O.synth_dump(2, 2, 8, 3, seed=0)
    assert np.array_equal(d.layers[1][0].numpy(), host[1][0])  # same draws as the reference
    p = tmp_path / "x.pkvd"
    pk.write_dump(d, p)
    back = pk.read_dump(p)
    assert np.array_equal(back.layers[1][1].numpy(), d.layers[1][1].numpy())
    raw = bytearray(p.read_bytes())
    raw[:4] = b"XXXX"
    p.write_bytes(raw)
    with pytest.raises(pk.BadMagicError):
        pk.read_dump(p)


def test_transcript_requires_ordered_layers():
    e = pk.TranscriptEntry(layer=1, k_checksum=0, v_checksum=0, k_elements=1, v_elements=1)
    with pytest.raises(ValueError, match="order"):
        pk.InjectionTranscript(agent_id=0, decode_bits=16, entries=(e,))


def test_round_to_bfloat16_matches_torch_cast():
    rng = np.random.default_rng(3)
    x = np.concatenate([rng.normal(size=5000).astype(np.float32),
                        np.array([0.0, -0.0, 1.0, 1.00390625, -1.00390625, 3.4e38, 1e-38], np.float32)])
    ref = torch.from_numpy(x.copy()).to(torch.bfloat16).to(torch.float32).numpy()
    assert np.array_equal(pk.round_to_bfloat16(x).view(np.uint32), ref.view(np.uint32))


@pytest.mark.skipif(torch.cuda.is_available(), reason="checks the no-GPU behaviour")
def test_no_cpu_fallback():
    from paper_2604_24971_b200._codec import CudaRequiredError

    g = pk.ModelGeometry(num_layers=1, kv_heads=1, head_dim=64, seq_len=4)
    dump = pk.synth_gaussian_dump(g, seed=0)
    with pytest.raises(CudaRequiredError):
        pk.build_pool(dump)
    with pytest.raises(CudaRequiredError):
        pk.quantize_v(dump.layers[0][1])


def test_lloyd_max_train_matches_reference_semantics():
    """Off-path table builder (valuequant.py:241-300): sorted-sample
    implementation, same fixed point as the reference's pass-over-samples
    loop (to summation rounding), same empty-cell repair warning."""
    import warnings

    from paper_2604_24971_b200 import valuequant as V

    x = np.random.default_rng(0).normal(size=20000)
    c = V.lloyd_max_train(x, 3).centroids
    assert np.all(np.diff(c) > 0)
    # the trained 3-bit table of N(0, 1) samples is close to the frozen GAUSSIAN_3BIT one
    assert np.abs(c - V.GAUSSIAN_3BIT.centroids).max() < 0.1
    with warnings.catch_warnings(record=True) as w:
        warnings.simplefilter("always")
        c2 = V.lloyd_max_train(np.concatenate([np.zeros(100), np.ones(100)]), 3).centroids
    assert any("repaired" in str(i.message) for i in w) and np.all(np.diff(c2) > 0)
