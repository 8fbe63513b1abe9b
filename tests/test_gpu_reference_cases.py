"""The reference's own codec / pool test cases, run through the sm_100a path.

Each test restates one case of `/root/reference/pkg/tests/test_keyquant.py`,
`test_valuequant.py`, `test_pool.py` or `test_acceptance.py` (cited per
test) against the GPU codec behind the drop-in API, and, where the case has
a numeric answer, also pins the device result bit-for-bit to the oracle.
Shapes are the reference's (head_dim 1 for scalar key tensors, d=2/8/64/128
for values) so the generic-warp codec and the streaming codec both run.
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2604_24971_b200 as pk
from paper_2604_24971_b200 import rotate_inverse
from oracle import kvpool_oracle as O

pytestmark = pytest.mark.gpu

CENTROIDS = np.array([-2.152, -1.344, -0.756, -0.245, 0.245, 0.756, 1.344, 2.152])


def scalar_tensor(values):
    """[1, 1, n, 1] f32 tensor on the device (head_dim 1 is legal for keys)."""
    v = np.asarray(values, dtype=np.float32)
    g = pk.ModelGeometry(num_layers=1, kv_heads=1, head_dim=1, seq_len=v.size)
    return pk.KvTensor(g, torch.from_numpy(v.reshape(1, 1, -1, 1)).cuda())


def value_tensor(values):
    """[1, 1, rows, d] (or [B, H, T, d]) f32 tensor on the device."""
    v = np.asarray(values, dtype=np.float32)
    if v.ndim == 2:
        v = v[None, None]
    g = pk.ModelGeometry(num_layers=1, kv_heads=v.shape[1], head_dim=v.shape[-1], seq_len=v.shape[2],
                         batch=v.shape[0])
    return pk.KvTensor(g, torch.from_numpy(np.ascontiguousarray(v)).cuda())


def host(t):
    return t.detach().cpu().numpy()


def scalar_reference(values, scale):
    """Round half away from zero, element by element, clip to [-128, 127]."""
    q = np.asarray(values, dtype=np.float64) / scale
    return np.clip(np.floor(np.abs(q) + 0.5) * np.where(q >= 0, 1, -1), -128, 127).astype(int).tolist()


def assert_k_matches_oracle(t, block):
    s, codes = O.quantize_k_tensor(t.numpy())
    assert np.float32(block.scale) == np.float32(s)
    assert np.array_equal(host(block.codes), codes)


def assert_v_matches_oracle(t, block, sign_seed=None):
    codes, scales = O.quantize_v(t.numpy(), sign_seed=sign_seed)
    assert np.array_equal(host(block.codes), codes)
    assert np.array_equal(host(block.scales).view(np.uint32), scales.astype(np.float32).view(np.uint32))


# ---------------------------------------------------------------- keys (test_keyquant.py)
def test_all_zero_key_tensor():  # test_keyquant.py:34-39
    t = scalar_tensor([0.0, 0.0, 0.0])
    block = pk.quantize_k(t)
    assert block.scale == 0.0
    assert not bool(block.codes.any())
    assert torch.equal(pk.dequantize_k(block).values, t.values)


def test_symmetric_extremes():  # test_keyquant.py:41-46
    t = scalar_tensor([-2.54, 0.0, 2.54])
    block = pk.quantize_k(t)
    assert block.scale == pytest.approx(0.02, rel=1e-6)
    assert host(block.codes).ravel().tolist() == [-127, 0, 127]
    assert host(pk.dequantize_k(block).values).ravel() == pytest.approx([-2.54, 0.0, 2.54], rel=1e-6)
    assert_k_matches_oracle(t, block)


def test_grid_aligned_keys_roundtrip_bit_exact():  # test_keyquant.py:48-55
    t = scalar_tensor(np.array([-127, -3, 0, 64, 127], dtype=np.float64) * 2.0**-6)
    block = pk.quantize_k(t)
    assert block.scale == 2.0**-6
    assert torch.equal(pk.dequantize_k(block).values, t.values)


def test_peak_element_maps_to_full_scale():  # test_keyquant.py:57-62
    vals = np.random.default_rng(0).normal(size=256).astype(np.float32)
    block = pk.quantize_k(scalar_tensor(vals))
    assert abs(int(host(block.codes).ravel()[np.abs(vals).argmax()])) == 127


def test_keys_match_scalar_reference():  # test_keyquant.py:64-69
    vals = np.random.default_rng(7).normal(0, 2.5, size=1000).astype(np.float32)
    t = scalar_tensor(vals)
    block = pk.quantize_k(t)
    assert host(block.codes).ravel().tolist() == scalar_reference(vals, block.scale)
    assert_k_matches_oracle(t, block)


def test_half_grid_points_round_away_from_zero():  # test_keyquant.py:71-78
    scale = 2.0**-6
    block = pk.quantize_k(scalar_tensor(np.array([127, 2.5, -2.5, 0.5, -0.5, 10.5]) * scale))
    assert block.scale == scale
    assert host(block.codes).ravel().tolist() == [127, 3, -3, 1, -1, 11]


def test_key_error_bound_random():  # test_keyquant.py:80-86
    vals = np.random.default_rng(123).normal(0, 1 / np.sqrt(128), size=100_000).astype(np.float32)
    t = scalar_tensor(vals)
    block = pk.quantize_k(t)
    err = float((pk.dequantize_k(block).values - t.values).abs().max())
    assert err <= (block.scale / 2) * (1 + 1e-6)
    assert_k_matches_oracle(t, block)


def test_key_requantization_is_stable():  # test_keyquant.py:88-94
    t = scalar_tensor(np.random.default_rng(9).normal(size=512).astype(np.float32))
    once = pk.quantize_k(t)
    twice = pk.quantize_k(pk.dequantize_k(once))
    assert twice.scale == once.scale
    assert torch.equal(twice.codes, once.codes)


def test_key_block_validation():  # test_keyquant.py:98-119
    g = pk.ModelGeometry(num_layers=1, kv_heads=1, head_dim=1, seq_len=2)
    with pytest.raises(pk.CorruptBlockError, match="int8"):
        pk.QuantizedKeyBlock(g, 1.0, np.zeros((1, 1, 2, 1), dtype=np.int16))
    with pytest.raises(pk.CorruptBlockError, match="zero scale"):
        pk.QuantizedKeyBlock(g, 0.0, np.array([1, 0], dtype=np.int8).reshape(1, 1, 2, 1))
    with pytest.raises(pk.CorruptBlockError):
        pk.QuantizedKeyBlock(g, -0.5, np.zeros((1, 1, 2, 1), dtype=np.int8))
    assert pk.quantize_k(scalar_tensor([1.0, -1.0, 0.5])).payload_nbytes == 3 + 4


# ---------------------------------------------------------------- values (test_valuequant.py)
def test_zero_value_tensor():  # test_valuequant.py:122-127
    t = value_tensor(np.zeros((4, 64), dtype=np.float32))
    block = pk.quantize_v(t)
    assert not bool(block.codes.any()) and not bool(block.scales.any())
    assert torch.equal(pk.dequantize_v(block).values, t.values)


def test_constant_rotated_coordinates_code_uniformly():  # test_valuequant.py:129-138
    for level, want in ((0.245, 5), (-0.245, 2)):
        x = rotate_inverse(np.full((1, 128), level)).astype(np.float32)
        t = value_tensor(x)
        block = pk.quantize_v(t)
        assert bool((block.codes == want).all())
        assert_v_matches_oracle(t, block)


def test_centroid_valued_rotation_roundtrips_nearly_exactly():  # test_valuequant.py:140-155
    rng = np.random.default_rng(4)
    mags = np.repeat([0.245, 0.756, 1.344, 2.152], [57, 35, 22, 14])
    y = (mags * rng.choice([-1.0, 1.0], size=128))[None, :]
    rng.shuffle(y[0])
    t = value_tensor(rotate_inverse(y).astype(np.float32))
    block = pk.quantize_v(t)
    assert float(block.scales.ravel()[0]) == pytest.approx(1.0, abs=1e-6)
    err = float((pk.dequantize_v(block).values - t.values).abs().max())
    assert err <= 1e-5 * float(t.values.abs().max())
    assert_v_matches_oracle(t, block)


def test_value_codes_are_scale_invariant():  # test_valuequant.py:157-163
    base = np.random.default_rng(3).normal(size=(6, 64)).astype(np.float32)
    a = pk.quantize_v(value_tensor(base))
    b = pk.quantize_v(value_tensor(7.3 * base))
    assert torch.equal(a.codes, b.codes)
    assert host(b.scales).ravel() == pytest.approx(7.3 * host(a.scales).ravel(), rel=1e-5)


def test_scales_are_rotated_rms():  # test_valuequant.py:165-171
    x = np.random.default_rng(8).normal(size=(5, 128)).astype(np.float32)
    t = value_tensor(x)
    block = pk.quantize_v(t)
    want = np.linalg.norm(x.astype(np.float64), axis=-1) / np.sqrt(128)
    assert host(block.scales).ravel() == pytest.approx(want, rel=1e-5)
    assert_v_matches_oracle(t, block)


BETA_CELL_PROBS_D128 = np.array([0.04021054, 0.10754843, 0.16155194, 0.19068909,
                                 0.19068909, 0.16155194, 0.10754843, 0.04021054])


def test_code_histogram_follows_the_sphere_marginal():  # test_valuequant.py:173-182
    g = pk.ModelGeometry(num_layers=1, kv_heads=8, head_dim=128, seq_len=1024)
    x = np.random.default_rng(12).normal(size=g.tensor_shape).astype(np.float32)
    t = pk.KvTensor(g, torch.from_numpy(x).cuda())
    block = pk.quantize_v(t)
    counts = torch.bincount(block.codes.reshape(-1).long(), minlength=8).cpu().numpy()
    n = g.elements_per_tensor
    sigma = np.sqrt(n * BETA_CELL_PROBS_D128 * (1 - BETA_CELL_PROBS_D128))
    assert (np.abs(counts - n * BETA_CELL_PROBS_D128) <= 3 * sigma).all()
    assert_v_matches_oracle(t, block)


def test_value_requantization_is_stable():  # test_valuequant.py:188-193
    t = value_tensor(np.random.default_rng(21).normal(size=(32, 128)).astype(np.float32) / np.sqrt(128))
    once = pk.quantize_v(t)
    twice = pk.quantize_v(pk.dequantize_v(once))
    assert torch.equal(once.codes, twice.codes)


def test_distortion_on_gaussian_input():  # test_valuequant.py:195-205
    g = pk.ModelGeometry(num_layers=1, kv_heads=8, head_dim=128, seq_len=1024)
    x = (np.random.default_rng(31).normal(size=g.tensor_shape) / np.sqrt(128)).astype(np.float32)
    t = pk.KvTensor(g, torch.from_numpy(x).cuda())
    back = host(pk.dequantize_v(pk.quantize_v(t)).values).astype(np.float64)
    ref = x.astype(np.float64)
    nmse = np.mean((back - ref) ** 2) / np.mean(ref ** 2)
    assert nmse <= pk.DistortionBound(3).bound
    assert nmse == pytest.approx(0.0345, abs=0.002)


def test_sign_diagonal_roundtrip_and_determinism():  # test_valuequant.py:206-217
    t = value_tensor(np.random.default_rng(17).normal(size=(16, 64)).astype(np.float32))
    a, b = pk.quantize_v(t, sign_seed=5), pk.quantize_v(t, sign_seed=5)
    assert torch.equal(a.codes, b.codes)
    assert not torch.equal(a.codes, pk.quantize_v(t, sign_seed=6).codes)
    back = host(pk.dequantize_v(a).values).astype(np.float64)
    ref = t.numpy().astype(np.float64)
    assert np.mean((back - ref) ** 2) / np.mean(ref ** 2) <= pk.DistortionBound(3).bound
    assert_v_matches_oracle(t, a, sign_seed=5)


def test_value_block_validation():  # test_valuequant.py:225-258
    g = pk.ModelGeometry(num_layers=1, kv_heads=1, head_dim=2, seq_len=1)
    ones = np.ones((1, 1, 1), dtype=np.float32)
    with pytest.raises(pk.CorruptBlockError, match="out of range"):
        pk.QuantizedValueBlock(g, pk.GAUSSIAN_3BIT.name, 3, codes=np.array([8, 0], np.uint8).reshape(1, 1, 1, 2),
                               scales=ones)
    with pytest.raises(pk.CorruptBlockError, match="zero-scale"):
        pk.QuantizedValueBlock(g, pk.GAUSSIAN_3BIT.name, 3, codes=np.array([1, 0], np.uint8).reshape(1, 1, 1, 2),
                               scales=np.zeros_like(ones))
    block = pk.quantize_v(value_tensor(np.ones((2, 8), dtype=np.float32)))
    other = pk.Codebook(bits=3, centroids=CENTROIDS * 2, name="other")
    with pytest.raises(pk.CorruptBlockError, match="coded with"):
        pk.dequantize_v(block, other)
    block = pk.quantize_v(value_tensor(np.ones((3, 8), dtype=np.float32)))
    assert block.payload_nbytes == 24 + 3 * 4
    assert block.packed_payload_nbytes == 3 * 3 + 3 * 4


@pytest.mark.parametrize("sign_seed", [None, 3])
@pytest.mark.parametrize("d", [1, 2, 4, 8, 16, 32, 64, 128, 256])
def test_every_power_of_two_head_dim_codes_like_the_oracle(d, sign_seed):
    # rotation identities across dimensions (test_acceptance.py:138-155): the
    # device codec, at every head_dim up to 256 (d < 8 through the
    # thread-per-word kernels), equals the oracle -- codes, scales, f32 and
    # bf16 decodes; 37 rows make the packed stream end mid-word for d < 8
    x = np.random.default_rng(d).normal(size=(1, 2, 37, d)).astype(np.float32)
    x[0, 1, 5] = 0.0  # a zero vector: scale 0, codes 0
    t = value_tensor(x)
    block = pk.quantize_v(t, sign_seed=sign_seed)
    assert_v_matches_oracle(t, block, sign_seed=sign_seed)
    codes, scales = O.quantize_v(x, sign_seed=sign_seed)
    want = O.dequantize_v(codes, scales, sign_seed=sign_seed)
    assert np.array_equal(host(pk.dequantize_v(block).values).view(np.uint32), want.view(np.uint32))
    bf = pk.dequantize_v(block, dtype=torch.bfloat16).values
    assert np.array_equal(host(bf.float()).view(np.uint32), O.round_to_bfloat16(want).view(np.uint32))
    assert bytes(host(block.packed)[:3 * ((x.size + 7) // 8)]) == O.pack3(codes)


# ---------------------------------------------------------------- pool (test_pool.py)
@pytest.fixture(scope="module")
def small_pool_and_dump():  # test_pool.py:28-32 (same geometry and seed)
    g = pk.ModelGeometry(num_layers=3, kv_heads=2, head_dim=32, seq_len=16)
    dump = pk.synth_gaussian_dump(g, seed=20)
    return pk.build_pool(dump), dump


def test_pool_is_sealed_with_stats(small_pool_and_dump):  # test_pool.py:36-42
    pool, _ = small_pool_and_dump
    assert pool.sealed
    assert len(pool.build_stats) == 3
    for s in pool.build_stats:
        assert s.k_mse > 0 and s.v_mse > 0
        assert s.k_max_err <= (s.k_scale / 2) * (1 + 1e-6)


def test_build_is_deterministic():  # test_pool.py:44-54
    g = pk.ModelGeometry(num_layers=2, kv_heads=2, head_dim=16, seq_len=8)
    dump = pk.synth_gaussian_dump(g, seed=1)
    a, b = pk.build_pool(dump), pk.build_pool(dump)
    for i in range(2):
        (ka, va), (kb, vb) = a.layer_blocks(i), b.layer_blocks(i)
        assert ka.scale == kb.scale and torch.equal(ka.codes, kb.codes)
        assert torch.equal(va.codes, vb.codes) and torch.equal(va.scales, vb.scales)


def test_attach_requires_sealed_and_valid_precision(small_pool_and_dump):  # test_pool.py:56-68
    pool, _ = small_pool_and_dump
    unsealed = pk.SharedPool(pool.geometry, [pool.layer_blocks(i) for i in range(pool.num_layers)])
    with pytest.raises(pk.UnsealedPoolError):
        unsealed.attach()
    unsealed.seal()
    assert unsealed.attach().agent_id == 0
    with pytest.raises(ValueError, match="decode_bits"):
        pool.attach(decode_bits=8)


def test_agent_ids_are_distinct_under_contention(small_pool_and_dump):  # test_pool.py:70-87
    import threading

    pool, _ = small_pool_and_dump
    views = [None] * 32
    barrier = threading.Barrier(32)

    def grab(i):
        barrier.wait()
        views[i] = pk.attach_agent(pool)

    threads = [threading.Thread(target=grab, args=(i,)) for i in range(32)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert len({v.agent_id for v in views}) == 32


def test_layer_out_of_range(small_pool_and_dump):  # test_pool.py:89-95
    view = small_pool_and_dump[0].attach()
    for bad in (3, -1):
        with pytest.raises(IndexError):
            view.get_kv_for_layer(bad)


def test_two_views_read_identical_bits_and_precisions_differ(small_pool_and_dump):  # test_pool.py:97-111
    pool, _ = small_pool_and_dump
    a, b = pool.attach(16), pool.attach(16)
    for i in range(pool.num_layers):
        (ka, va), (kb, vb) = a.get_kv_for_layer(i), b.get_kv_for_layer(i)
        assert torch.equal(ka.values, kb.values) and torch.equal(va.values, vb.values)
    k16, _ = pool.attach(16).get_kv_for_layer(0)
    k32, _ = pool.attach(32).get_kv_for_layer(0)
    assert k16.dtype == torch.bfloat16 and k32.dtype == torch.float32
    assert not torch.equal(k16.values.float(), k32.values)
    assert torch.equal(k16.values, k32.values.to(torch.bfloat16))  # RNE == round_to_bfloat16


def test_reads_do_not_grow_the_pool(small_pool_and_dump):  # test_pool.py:113-120
    pool, _ = small_pool_and_dump
    before = (pool.payload_nbytes(), pool.device_nbytes())
    for _ in range(15):
        view = pool.attach()
        for i in range(pool.num_layers):
            view.get_kv_for_layer(i)
    assert (pool.payload_nbytes(), pool.device_nbytes()) == before


def test_fidelity_against_source(small_pool_and_dump):  # test_pool.py:122-133
    pool, dump = small_pool_and_dump
    view = pool.attach(32)
    for i, (k, v) in enumerate(dump.layers):
        kq, _ = pool.layer_blocks(i)
        kd, vd = view.get_kv_for_layer(i)
        assert float((kd.values.cpu() - k.values.cpu().float()).abs().max()) <= (kq.scale / 2) * (1 + 1e-6)
        ref = v.values.cpu().double()
        nmse = float(((vd.values.cpu().double() - ref) ** 2).mean() / (ref ** 2).mean())
        assert nmse <= 0.0425109


def test_transcripts_agree_across_agents_and_fingerprint_tensors(small_pool_and_dump):  # test_pool.py:135-172
    pool, _ = small_pool_and_dump
    views = [pool.attach() for _ in range(4)]
    ts = [v.inject_all() for v in views]
    assert [e.layer for e in ts[0].entries] == list(range(pool.num_layers))
    assert all(t.checksums() == ts[0].checksums() for t in ts)
    k, v = views[0].get_kv_for_layer(1)
    assert ts[0].checksums()[1] == (pk.tensor_checksum(k.values), pk.tensor_checksum(v.values))


@pytest.mark.parametrize("d", [1, 2, 4])
def test_small_head_dim_pool_reads_like_the_oracle(d):
    # a whole pool at head_dim < 8 (keys through the warp kernels, values
    # through the thread-per-word kernels), read back at 16 and 32 bits
    g = pk.ModelGeometry(num_layers=3, kv_heads=3, head_dim=d, seq_len=13, batch=2)
    dump = pk.synth_gaussian_dump(g, seed=d)
    pool = pk.build_pool(dump, sign_seed=7)
    ref = O.synth_dump(3, 3, d, 13, batch=2, seed=d)
    for bits in (16, 32):
        view = pool.attach(bits)
        for i, (k_in, v_in) in enumerate(ref):
            s, kc = O.quantize_k_tensor(k_in)
            vc, vs = O.quantize_v(v_in, sign_seed=7)
            kw, vw = O.decode_layer(kc, s, vc, vs, decode_bits=bits, sign_seed=7)
            k, v = view.get_kv_for_layer(i)
            assert np.array_equal(k.numpy().view(np.uint32), kw.view(np.uint32))
            assert np.array_equal(v.numpy().view(np.uint32), vw.view(np.uint32))


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
@pytest.mark.parametrize("bad", [float("nan"), float("-inf"), -float("nan")])
def test_nonfinite_key_in_a_full_item_raises(dtype, bad):
    # model.py rejects NaN/Inf (GeometryError); on the device the key absmax
    # of a FULL streamed item (16384 elements here, two f32 / one bf16 item)
    # must carry a NaN or an infinity into the layer maximum
    g = pk.ModelGeometry(num_layers=2, kv_heads=2, head_dim=128, seq_len=64)
    dump = pk.synth_gaussian_dump(g, seed=3, device="cuda", dtype=dtype)
    dump.layers[1][0].values[0, 1, 40, 77] = bad
    with pytest.raises(pk.GeometryError, match="NaN or Inf"):
        pk.build_pool(dump)
    k = dump.layers[1][0]
    with pytest.raises(pk.GeometryError, match="NaN or Inf"):
        pk.quantize_k(k)


@pytest.mark.parametrize("dtype", [torch.float32, torch.bfloat16])
def test_more_layers_than_one_launch_holds(dtype):
    # Llama-70B has 80 layers: pkv_encode / pkv_decode split into launches of
    # PKV_MAX_LAYERS_PER_LAUNCH (64) layers; the per-tensor key maxima, the
    # layer-major arena and the decode must line up across the boundary
    g = pk.ModelGeometry(num_layers=80, kv_heads=2, head_dim=128, seq_len=24)
    dump = pk.synth_gaussian_dump(g, seed=80, device="cuda", dtype=dtype)
    pool = pk.build_pool(dump, sign_seed=2)
    assert len(pool.build_stats) == 80
    view = pool.attach(32)
    outs = view.materialize_all()
    for li in (0, 62, 63, 64, 65, 79):
        k_in, v_in = (t.values.float().cpu().numpy() for t in dump.layers[li])
        s, kc = O.quantize_k_tensor(k_in)
        vc, vs = O.quantize_v(v_in, sign_seed=2)
        kq, vq = pool.layer_blocks(li)
        assert np.float32(kq.scale) == np.float32(s) and np.array_equal(host(kq.codes), kc), li
        assert np.array_equal(host(vq.codes), vc) and np.array_equal(host(vq.scales).view(np.uint32), vs.view(np.uint32)), li
        kw, vw = O.decode_layer(kc, s, vc, vs, decode_bits=32, sign_seed=2)
        assert np.array_equal(host(outs[li][0]).view(np.uint32), kw.view(np.uint32)), li
        assert np.array_equal(host(outs[li][1]).view(np.uint32), vw.view(np.uint32)), li
        k1, v1 = view.get_kv_for_layer(li)
        assert torch.equal(k1.values, outs[li][0]) and torch.equal(v1.values, outs[li][1])


def test_non_contiguous_and_host_inputs_encode_like_contiguous_ones():
    # a KV cache laid out [B, T, H, D] (transformers' key_states before the
    # transpose) viewed as [B, H, T, D], and plain host numpy arrays: the
    # reference takes any array; the device path must give the same pool
    g = pk.ModelGeometry(num_layers=2, kv_heads=4, head_dim=64, seq_len=33)
    rng = np.random.default_rng(5)
    layers_np = [(rng.normal(size=g.tensor_shape).astype(np.float32),
                  rng.normal(size=g.tensor_shape).astype(np.float32)) for _ in range(2)]
    as_bthd = lambda a: torch.from_numpy(np.ascontiguousarray(a.transpose(0, 2, 1, 3))).cuda().transpose(1, 2)
    assert not as_bthd(layers_np[0][0]).is_contiguous()
    strided = pk.KvDump(g, tuple((pk.KvTensor(g, as_bthd(k)), pk.KvTensor(g, as_bthd(v))) for k, v in layers_np))
    host_dump = pk.KvDump(g, tuple((pk.KvTensor(g, k), pk.KvTensor(g, v)) for k, v in layers_np))
    a, b = pk.build_pool(strided), pk.build_pool(host_dump)
    for i, (k, v) in enumerate(layers_np):
        s, kc = O.quantize_k_tensor(k)
        vc, vs = O.quantize_v(v)
        for p in (a, b):
            kq, vq = p.layer_blocks(i)
            assert np.float32(kq.scale) == np.float32(s) and np.array_equal(host(kq.codes), kc)
            assert np.array_equal(host(vq.codes), vc) and np.array_equal(host(vq.scales).view(np.uint32), vs.view(np.uint32))


@pytest.mark.parametrize("scale", [1e-38, 1e-25, 1e-12, 1e12, 1e25, 1e30])
def test_extreme_magnitudes_code_like_the_oracle(scale):
    # per-vector norms far from 1 (sub-normal-ish and huge): the fast path
    # hands vectors with sum(x^2) outside [2^-200, 2^200] to the exact replay,
    # keys below a 1e-30 scale to the exact key path; everything must match
    # the f64 reference, decode included
    x = (np.random.default_rng(int(abs(np.log10(scale)))).normal(size=(1, 3, 21, 128)) * scale).astype(np.float32)
    k = (np.random.default_rng(7).normal(size=(1, 3, 21, 128)) * scale).astype(np.float32)
    t, tk = value_tensor(x), value_tensor(k)
    block = pk.quantize_v(t)
    assert_v_matches_oracle(t, block)
    codes, scales = O.quantize_v(x)
    want = O.dequantize_v(codes, scales)
    assert np.array_equal(host(pk.dequantize_v(block).values).view(np.uint32), want.view(np.uint32))
    kb = pk.quantize_k(tk)
    assert_k_matches_oracle(tk, kb)
    s, kc = O.quantize_k_tensor(k)
    assert np.array_equal(host(pk.dequantize_k(kb).values).view(np.uint32), O.dequantize_k_tensor(kc, s).view(np.uint32))


def _canary_views(nbytes_list, dtype_list, device, pad=256, fill=0xA5):
    """One buffer per request, each carved at a 256-byte aligned offset out of
    a larger canary-filled byte buffer; returns (views, checker)."""
    bufs, views = [], []
    for nbytes, dt in zip(nbytes_list, dtype_list):
        big = torch.full((pad + ((nbytes + 255) // 256) * 256 + pad,), fill, dtype=torch.uint8, device=device)
        view = big[pad:pad + nbytes].view(dt)
        bufs.append((big, nbytes))
        views.append(view)

    def intact():
        for big, nbytes in bufs:
            b = big.cpu().numpy()
            if (b[:pad] != fill).any() or (b[pad + nbytes:] != fill).any():
                return False
        return True
    return views, intact


@pytest.mark.parametrize("D,H,T,dtype", [(128, 3, 37, torch.float32), (64, 5, 23, torch.bfloat16),
                                          (2, 1, 7, torch.float32), (16, 2, 9, torch.bfloat16)])
def test_kernels_write_exactly_the_documented_bytes(D, H, T, dtype):
    # compute-sanitizer is not available on this GPU pool: instead every output
    # of pkv_encode / pkv_decode is a view at an aligned offset inside a larger
    # canary-filled buffer, sized exactly as include/polykv.h documents (n key
    # codes, 3*ceil(n/8) packed bytes, one f32 scale per head vector, n
    # outputs); nothing around them may change
    from paper_2604_24971_b200 import _codec
    from paper_2604_24971_b200.keyquant import K_MODES

    L, dev = 2, torch.device("cuda", torch.cuda.current_device())
    nvec, n = H * T, H * T * D
    rng = np.random.default_rng(D + T)
    ks = [torch.from_numpy(rng.normal(size=n).astype(np.float32)).to(dev, dtype) for _ in range(L)]
    vs = [torch.from_numpy(rng.normal(size=n).astype(np.float32)).to(dev, dtype) for _ in range(L)]
    pk_bytes = 3 * ((n + 7) // 8)
    views, intact = _canary_views([n] * L + [4] * L + [pk_bytes] * L + [4 * nvec] * L,
                                  [torch.int8] * L + [torch.float32] * L + [torch.uint8] * L + [torch.float32] * L, dev)
    k_codes, k_scale, v_packed, v_scales = views[:L], views[L:2 * L], views[2 * L:3 * L], views[3 * L:]
    status = torch.zeros(L, dtype=torch.int32, device=dev)
    _codec.encode(num_vectors=nvec, head_dim=D, k_in=ks, v_in=vs, k_mode=K_MODES["tensor"], k_codes=k_codes,
                  k_scale=k_scale, k_bscale=None, v_packed=v_packed, v_scales=v_scales,
                  centroids=pk.GAUSSIAN_3BIT.centroids, sign_seed=None, status=status, replay=None, device=dev)
    torch.cuda.synchronize()
    assert intact(), "pkv_encode wrote outside its documented outputs"
    for li in range(L):  # and the codes are the reference's
        s, kc = O.quantize_k_tensor(ks[li].float().cpu().numpy())
        vc, vsc = O.quantize_v(vs[li].float().cpu().numpy().reshape(1, H, T, D))
        assert np.array_equal(k_codes[li].cpu().numpy(), kc.reshape(-1))
        assert bytes(v_packed[li].cpu().numpy()) == O.pack3(vc)
    for out_dt, eb in ((torch.bfloat16, 2), (torch.float32, 4)):
        outs, intact_o = _canary_views([n * eb] * (2 * L), [out_dt] * (2 * L), dev)
        _codec.decode(num_vectors=nvec, head_dim=D, out_dtype=out_dt, k_mode=K_MODES["tensor"], k_codes=k_codes,
                      k_scale=k_scale, k_bscale=None, v_packed=v_packed, v_scales=v_scales,
                      centroids=pk.GAUSSIAN_3BIT.centroids, sign_seed=None, k_out=outs[:L], v_out=outs[L:],
                      device=dev)
        torch.cuda.synchronize()
        assert intact_o(), f"pkv_decode ({out_dt}) wrote outside its outputs"


@pytest.mark.parametrize("D,H,T", [(128, 3, 37), (64, 2, 5), (4, 3, 11)])
def test_block32_encode_writes_exactly_the_documented_bytes(D, H, T):
    from paper_2604_24971_b200 import _codec
    from paper_2604_24971_b200.keyquant import K_MODES

    dev = torch.device("cuda", torch.cuda.current_device())
    n = H * T * D
    ks = [torch.from_numpy(np.random.default_rng(T).normal(size=n).astype(np.float32)).to(dev)]
    nb = (n + 31) // 32
    (k_codes, k_bscale), intact = _canary_views([n, 2 * nb], [torch.int8, torch.int16], dev)
    status = torch.zeros(1, dtype=torch.int32, device=dev)
    _codec.encode(num_vectors=H * T, head_dim=D, k_in=ks, v_in=None, k_mode=K_MODES["block32"], k_codes=[k_codes],
                  k_scale=None, k_bscale=[k_bscale], v_packed=None, v_scales=None,
                  centroids=pk.GAUSSIAN_3BIT.centroids, sign_seed=None, status=status, replay=None, device=dev)
    torch.cuda.synchronize()
    assert intact(), "block32 pkv_encode wrote outside its documented outputs"
    s16, kc = O.quantize_k_block32(ks[0].cpu().numpy())
    assert np.array_equal(k_codes.cpu().numpy(), kc) and np.array_equal(k_bscale.cpu().numpy().view(np.uint16), s16.view(np.uint16))


@pytest.mark.parametrize("D,H,T,R,G,cap", [(128, 8, 1000, 15, 4, 16), (64, 4, 70, 3, 2, 0), (128, 2, 5, 1, 1, 3)])
def test_attention_writes_exactly_its_output_and_workspace(D, H, T, R, G, cap):
    from paper_2604_24971_b200 import _lib
    from paper_2604_24971_b200 import attention as A

    dev = torch.device("cuda", torch.cuda.current_device())
    g = pk.ModelGeometry(num_layers=1, kv_heads=H, head_dim=D, seq_len=T)
    pool = pk.build_pool(pk.synth_gaussian_dump(g, seed=T, device=dev), build_stats=False)
    need = _lib.load().pkv_attention_workspace_bytes(R, H, G, D, T)
    (out, ws), intact = _canary_views([R * H * G * D * 4, ((need + 3) // 4) * 4], [torch.float32, torch.float32], dev)
    gen = torch.Generator(device="cuda").manual_seed(T)
    q = torch.randn(R, H, G, D, device=dev, generator=gen)
    kw = {}
    if cap:
        kw = dict(tail_k=torch.randn(R, H, cap, D, device=dev, generator=gen).bfloat16(),
                  tail_v=torch.randn(R, H, cap, D, device=dev, generator=gen).bfloat16(),
                  tail_len=torch.randint(0, cap + 1, (R,), device=dev, dtype=torch.int32, generator=gen))
    res = A.decode_attention(pool, 0, q, out=out.view(R, H, G, D), workspace=ws, out_dtype=torch.float32, **kw)
    torch.cuda.synchronize()
    assert res.data_ptr() == out.data_ptr()
    assert intact(), "decode attention wrote outside its output / workspace"
    assert bool(torch.isfinite(res).all())
