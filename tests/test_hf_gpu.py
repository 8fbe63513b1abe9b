"""Injection of the pool into a transformers Llama (kvbridge/hfcache.py semantics).

Mirrors the reference's bridge tests (pkg/exporter/tests/test_evaluator.py
:64-124, test_exporter.py:82-92) on a deterministic random-init GQA Llama
(conftest.py:56-69 builds one with head_dim 16; the pool attention kernel
covers head_dim 64/128, so this fixture uses 64).
"""

from __future__ import annotations

import numpy as np
import pytest
import torch

import paper_2604_24971_b200 as pk
from oracle import kvpool_oracle as O

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tiny_llama():
    from transformers import LlamaConfig, LlamaForCausalLM

    torch.manual_seed(1234)
    cfg = LlamaConfig(vocab_size=256, hidden_size=256, intermediate_size=512, num_hidden_layers=3,
                      num_attention_heads=4, num_key_value_heads=2, head_dim=64, max_position_embeddings=512,
                      attn_implementation="sdpa")
    model = LlamaForCausalLM(cfg).cuda().eval()
    return model


def _prefill_pool(model, ids, prefix):
    from paper_2604_24971_b200 import hf

    with torch.no_grad():
        out = model(ids[:, :prefix], use_cache=True)
    layers = hf.cache_layers(out.past_key_values)
    geo = hf.model_kv_geometry(model)
    g = pk.ModelGeometry(num_layers=geo["num_layers"], kv_heads=geo["kv_heads"], head_dim=geo["head_dim"],
                         seq_len=prefix)
    dump = pk.KvDump(g, tuple((pk.KvTensor(g, k.float()), pk.KvTensor(g, v.float())) for k, v in layers))
    return pk.build_pool(dump), layers


def test_cache_layers_and_geometry(tiny_llama):
    from paper_2604_24971_b200 import hf

    ids = torch.randint(0, 256, (1, 20), device="cuda")
    with torch.no_grad():
        out = tiny_llama(ids, use_cache=True)
    layers = hf.cache_layers(out.past_key_values)
    assert len(layers) == 3 and layers[0][0].shape == (1, 2, 20, 64)
    assert hf.model_kv_geometry(tiny_llama) == {"num_layers": 3, "kv_heads": 2, "head_dim": 64}
    with pytest.raises(hf.CacheLayoutError):
        hf.cache_layers(None)


def test_materialized_injection_is_the_reference_cache(tiny_llama):
    """build_cache(mode="materialize") == DynamicCache built from the oracle's
    get_kv_for_layer output, so the continuation logits are identical."""
    from paper_2604_24971_b200 import hf

    torch.manual_seed(7)
    ids = torch.randint(0, 256, (1, 40), device="cuda")
    pool, _ = _prefill_pool(tiny_llama, ids, 32)
    for bits in (16, 32):
        ref_layers = []
        for li in range(pool.num_layers):
            kq, vq = pool.layer_blocks(li)
            kd, vd = O.decode_layer(kq.codes.cpu().numpy(), kq.scale, vq.codes.cpu().numpy(),
                                    vq.scales.cpu().numpy(), bits)
            ref_layers.append((torch.from_numpy(kd).cuda(), torch.from_numpy(vd).cuda()))
        ref = hf.build_dynamic_cache(ref_layers)
        ours = hf.build_cache(pool.attach(bits), "materialize", dtype=torch.float32)
        for (rk, rv), layer in zip(ref_layers, ours.layers):
            assert torch.equal(layer.keys, rk) and torch.equal(layer.values, rv)
        with torch.no_grad():
            a = tiny_llama(ids[:, 32:], past_key_values=ref).logits
            b = tiny_llama(ids[:, 32:], past_key_values=ours).logits
        assert torch.equal(a, b)


def test_materialized_cache_is_a_fresh_copy(tiny_llama):
    # test_exporter.py:82-92: the injected cache must not alias the pool
    from paper_2604_24971_b200 import hf

    ids = torch.randint(0, 256, (1, 24), device="cuda")
    pool, _ = _prefill_pool(tiny_llama, ids, 24)
    c1 = hf.build_cache(pool.attach(32), "materialize")
    c1.layers[0].keys.zero_()
    c2 = hf.build_cache(pool.attach(32), "materialize")
    assert c2.layers[0].keys.abs().sum() > 0


@pytest.mark.parametrize("agents", [1, 3])
def test_streamed_decode_matches_materialized_decode(tiny_llama, agents):
    """Greedy decode through the packed pool (pkv_decode_attention) follows the
    materialised-cache decode: same tokens, logits within bf16-tail error."""
    from paper_2604_24971_b200 import hf

    torch.manual_seed(11)
    ids = torch.randint(0, 256, (1, 40), device="cuda")
    pool, _ = _prefill_pool(tiny_llama, ids, 32)
    B = agents
    full = ids.expand(B, -1)
    # reference: materialised 32-bit cache, sdpa, manual greedy loop
    pool_bytes = pool.device_nbytes()
    ref_cache = hf.build_cache(pool.attach(32), "materialize", batch=B, dtype=torch.float32)
    st_cache = hf.build_cache(pool.attach(32), "stream", batch=B)
    tiny_llama.set_attn_implementation("sdpa")
    steps = 6
    ref_logits, st_logits = [], []
    with torch.no_grad():
        step = full[:, 32:]
        pos = 32
        for _ in range(steps):
            position_ids = torch.arange(pos, pos + step.shape[1], device="cuda").unsqueeze(0).expand(B, -1)
            ref_logits.append(tiny_llama(step, past_key_values=ref_cache, position_ids=position_ids).logits[:, -1])
            nxt = ref_logits[-1].argmax(-1, keepdim=True)
            pos += step.shape[1]
            step = nxt
        hf.use_pooled_attention(tiny_llama)
        step = full[:, 32:]
        pos = 32
        for i in range(steps):
            position_ids = torch.arange(pos, pos + step.shape[1], device="cuda").unsqueeze(0).expand(B, -1)
            st_logits.append(tiny_llama(step, past_key_values=st_cache, position_ids=position_ids).logits[:, -1])
            pos += step.shape[1]
            step = ref_logits[i].argmax(-1, keepdim=True)  # teacher-force the reference tokens
    tiny_llama.set_attn_implementation("sdpa")
    for r, s in zip(ref_logits, st_logits):
        rel = float((r - s).abs().max() / r.abs().max())
        assert rel < 5e-3, rel
        assert torch.equal(r.argmax(-1), s.argmax(-1))
    assert st_cache.get_seq_length() == 32 + 8 + steps - 1
    # pool memory is shared: the pool's HBM footprint did not change, and the
    # streaming agents hold only their private tails (no per-agent prefix copy)
    assert pool.device_nbytes() == pool_bytes

    # every streamed layer holds only its [B, H, capacity, D] bf16 tail buffers
    for layer in st_cache.layers:
        assert layer.keys.shape[2] == layer.capacity and layer.values.shape == layer.keys.shape
        assert layer.keys.dtype == torch.bfloat16 and layer.tail_len == 8 + steps - 1


def test_greedy_continuation_modes_agree(tiny_llama):
    from paper_2604_24971_b200 import hf

    torch.manual_seed(5)
    ids = torch.randint(0, 256, (1, 36), device="cuda")
    pool, _ = _prefill_pool(tiny_llama, ids, 32)
    a = hf.greedy_continuation(tiny_llama, ids, pool.attach(32), 5, mode="materialize", batch=2)
    tiny_llama.set_attn_implementation("sdpa")
    b = hf.greedy_continuation(tiny_llama, ids, pool.attach(32), 5, mode="stream", batch=2)
    tiny_llama.set_attn_implementation("sdpa")
    assert a.shape == (2, 5)
    # 32-bit decode: the streamed pool attention must pick the same tokens
    assert torch.equal(a, b), (a, b)
    assert torch.equal(a[0], a[1]) and torch.equal(b[0], b[1])
