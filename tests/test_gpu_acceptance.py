"""The reference's acceptance criteria (`/root/reference/pkg/tests/test_acceptance.py`)
run on the GPU path, each criterion additionally pinned to the oracle where
it has a numeric answer. Wall-clock budgets of the reference (one CPU core)
are kept as upper bounds; the device path is far inside them.
"""

from __future__ import annotations

import threading
import time

import numpy as np
import pytest
import torch

import paper_2604_24971_b200 as pk
from oracle import kvpool_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def serving_pool():  # test_acceptance.py:50-54
    g = pk.ModelGeometry(num_layers=32, kv_heads=8, head_dim=128, seq_len=1024)
    return pk.build_pool(pk.synth_gaussian_dump(g, seed=0))


def test_value_distortion_on_gaussian_dumps():  # test_acceptance.py:97-112
    g = pk.ModelGeometry(num_layers=4, kv_heads=8, head_dim=128, seq_len=256)
    dump = pk.synth_gaussian_dump(g, seed=11)
    num = den = 0.0
    for _, v in dump.layers:
        back = pk.dequantize_v(pk.quantize_v(v)).values.double().cpu()
        ref = v.values.double().cpu()
        num += float(((back - ref) ** 2).sum())
        den += float((ref ** 2).sum())
    nmse = num / den
    assert nmse <= 0.0425109 and abs(nmse - 0.0345) <= 0.002


def test_key_quantization_error_bound():  # test_acceptance.py:115-135
    rng = np.random.default_rng(100)
    g = pk.ModelGeometry(num_layers=1, kv_heads=2, head_dim=64, seq_len=32)
    worst = 0.0
    for _ in range(100):
        vals = rng.normal(0, rng.choice([0.01, 1.0, 100.0]), size=g.tensor_shape).astype(np.float32)
        t = pk.KvTensor(g, torch.from_numpy(vals).cuda())
        block = pk.quantize_k(t)
        err = float((pk.dequantize_k(block).values - t.values).abs().max())
        worst = max(worst, err / ((block.scale / 2) * (1 + 1e-6)))
        s, codes = O.quantize_k_tensor(vals)
        assert np.float32(block.scale) == np.float32(s)
        assert np.array_equal(block.codes.cpu().numpy(), codes)
    assert worst <= 1.0
    grid = np.arange(-127, 128, dtype=np.float64).reshape(1, 1, 255, 1) * 2.0**-6
    gg = pk.ModelGeometry(num_layers=1, kv_heads=1, head_dim=1, seq_len=255)
    t = pk.KvTensor(gg, torch.from_numpy(grid.astype(np.float32)).cuda())
    assert torch.equal(pk.dequantize_k(pk.quantize_k(t)).values, t.values)


def test_fifteen_concurrent_readers_are_bit_identical(serving_pool):  # test_acceptance.py:157-202
    t0 = time.perf_counter()
    pool = serving_pool
    reference = pool.attach(16).inject_all().checksums()
    # the transcript itself is the reference's: two layers against the oracle
    src = O.synth_dump(32, 8, 128, 1024, seed=0)
    for li in (0, 31):
        k_in, v_in = src[li]
        s, kc = O.quantize_k_tensor(k_in)
        vc, vs = O.quantize_v(v_in)
        kw, vw = O.decode_layer(kc, s, vc, vs, decode_bits=16)
        assert reference[li] == (O.tensor_checksum(kw), O.tensor_checksum(vw))
    mismatches, errors = [], []

    def reader(round_idx, slot, barrier):
        view = pool.attach(16)
        layers = np.random.default_rng(1000 * round_idx + slot).integers(0, pool.num_layers, size=2)
        barrier.wait()
        try:
            for layer in layers:
                k, v = view.get_kv_for_layer(int(layer))
                if (pk.tensor_checksum(k.values), pk.tensor_checksum(v.values)) != reference[int(layer)]:
                    mismatches.append((round_idx, slot, int(layer)))
        except Exception as e:  # a thread's exception would otherwise not fail the test
            errors.append(repr(e))

    for round_idx in range(20):
        barrier = threading.Barrier(15)
        threads = [threading.Thread(target=reader, args=(round_idx, s, barrier)) for s in range(15)]
        for t in threads:
            t.start()
        for t in threads:
            t.join()
    transcripts = [None] * 5
    barrier = threading.Barrier(5)

    def full(slot):
        view = pool.attach(16)
        barrier.wait()
        try:
            transcripts[slot] = view.inject_all().checksums()
        except Exception as e:
            errors.append(repr(e))

    threads = [threading.Thread(target=full, args=(i,)) for i in range(5)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    assert not errors, errors[:3]
    assert not mismatches
    assert all(tr == reference for tr in transcripts)
    assert time.perf_counter() - t0 < 60.0


def test_pool_bytes_do_not_scale_with_agents(serving_pool):  # test_acceptance.py:205-214
    pool = serving_pool
    torch.cuda.synchronize()
    sizes, resident = {}, {}
    for n in (3, 5, 10, 15):
        views = [pool.attach(16) for _ in range(n)]
        sizes[n] = pool.payload_nbytes()
        resident[n] = (pool.device_nbytes(), torch.cuda.memory_allocated())
        del views
    assert len(set(sizes.values())) == 1
    assert len(set(resident.values())) == 1


def test_packed_snapshots_decode_identically(tmp_path):  # test_acceptance.py:246-272
    rng = np.random.default_rng(55)
    for trial in range(50):
        g = pk.ModelGeometry(
            num_layers=int(rng.integers(1, 4)), kv_heads=int(rng.integers(1, 5)),
            head_dim=int(2 ** rng.integers(3, 8)), seq_len=int(rng.integers(1, 41)),
            batch=int(rng.integers(1, 3)))
        pool = pk.build_pool(pk.synth_gaussian_dump(g, seed=trial))
        u_path, p_path = tmp_path / f"u{trial}.pkvp", tmp_path / f"p{trial}.pkvp"
        pk.save_pool(pool, u_path, packed=False)
        pk.save_pool(pool, p_path, packed=True)
        a, b = pk.load_pool(u_path).attach(16), pk.load_pool(p_path).attach(16)
        for i in range(g.num_layers):
            (ka, va), (kb, vb) = a.get_kv_for_layer(i), b.get_kv_for_layer(i)
            assert torch.equal(ka.values, kb.values) and torch.equal(va.values, vb.values)
