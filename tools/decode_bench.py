"""Model-level shared-pool decode throughput (SURVEY §8(d) "Decode tok/s").

A random-init Llama of the config's shape prefills the shared context once;
the context K/V is compressed into a SharedPool on the GPU; then N agents
greedy-decode in lockstep:

  pooled_graph   PooledCache + "polykv" attention (pkv_decode_attention over
                 the packed pool), one decode step captured in a CUDA graph
  pooled_eager   the same, eager (HF Python loop)
  materialized   the reference semantics on the same GPU: every agent owns a
                 bf16 DynamicCache copy of the decoded prefix (kvbridge
                 hfcache.build_cache) and stock SDPA attention, eager

tok/s = agents x steps / elapsed (CUDA events around the decode loop).
"""

from __future__ import annotations

import argparse
import json
import sys
from pathlib import Path

import torch

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))

SHAPES = {
    # name: (layers, hidden, heads, kv_heads, head_dim, ffn, vocab, prefix, agents)
    "c2": (24, 2048, 32, 32, 64, 8192, 49152, 1851, 5),
    "c3": (32, 4096, 32, 8, 128, 14336, 128256, 4096, 15),
}


def build_model(shape):
    from transformers import LlamaConfig, LlamaForCausalLM

    L, hid, heads, kvh, hd, ffn, vocab, prefix, _ = shape
    cfg = LlamaConfig(vocab_size=vocab, hidden_size=hid, intermediate_size=ffn, num_hidden_layers=L,
                      num_attention_heads=heads, num_key_value_heads=kvh, head_dim=hd,
                      max_position_embeddings=prefix + 1024, attn_implementation="sdpa")
    torch.manual_seed(0)
    prev = torch.get_default_dtype()
    torch.set_default_dtype(torch.bfloat16)
    try:
        with torch.device("cuda"):
            model = LlamaForCausalLM(cfg).eval()
    finally:
        torch.set_default_dtype(prev)
    return model


def run(config: str = "c3", steps: int = 32, agents: int | None = None, modes=("pooled_graph", "pooled_eager",
                                                                              "materialized")) -> dict:
    import paper_2604_24971_b200 as pk
    from paper_2604_24971_b200 import hf

    shape = SHAPES[config]
    L, hid, heads, kvh, hd, ffn, vocab, prefix, A0 = shape
    A = agents or A0
    dev = torch.device("cuda")
    model = build_model(shape)
    ids = torch.randint(0, vocab, (1, prefix), device=dev)
    with torch.no_grad():
        out = model(ids, use_cache=True)
    layers = hf.cache_layers(out.past_key_values)
    first = out.logits[:, -1].argmax(-1, keepdim=True).expand(A, 1).contiguous()
    del out
    g = pk.ModelGeometry(num_layers=L, kv_heads=kvh, head_dim=hd, seq_len=prefix)
    pool = pk.build_pool(pk.KvDump(g, tuple((pk.KvTensor(g, k), pk.KvTensor(g, v)) for k, v in layers)))
    del layers
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    res = {"config": config, "agents": A, "steps": steps, "prefix": prefix, "layers": L,
           "pool_bytes": pool.device_nbytes(), "weights_bytes": sum(p.numel() * 2 for p in model.parameters())}

    def timed(fn, n):
        s, e = ev(), ev()
        torch.cuda.synchronize()
        s.record()
        fn(n)
        e.record()
        torch.cuda.synchronize()
        return s.elapsed_time(e)

    with torch.no_grad():
        if "pooled_graph" in modes or "pooled_eager" in modes:
            hf.use_pooled_attention(model)
            for mode in ("pooled_eager", "pooled_graph"):
                if mode not in modes:
                    continue
                cache = hf.build_cache(pool.attach(32), "stream", batch=A, tail_capacity=steps + 16)
                step_ids = first.clone()
                pos = torch.full((A, 1), prefix, dtype=torch.long, device=dev)

                def one():
                    logits = model(step_ids, past_key_values=cache, position_ids=pos, use_cache=True).logits
                    step_ids.copy_(logits[:, -1].argmax(-1, keepdim=True))
                    pos.add_(1)

                one()  # first decode step (allocations, lazy init)
                if mode == "pooled_graph":
                    side = torch.cuda.Stream()
                    side.wait_stream(torch.cuda.current_stream())
                    with torch.cuda.stream(side):
                        one()
                    torch.cuda.current_stream().wait_stream(side)
                    graph = torch.cuda.CUDAGraph()
                    with torch.cuda.graph(graph):
                        one()
                    graph.replay()

                    def loop(n):
                        for _ in range(n):
                            graph.replay()
                else:
                    def loop(n):
                        for _ in range(n):
                            one()
                ms = timed(loop, steps)
                cache.sync_lengths()
                res[mode] = {"tokens_per_s": A * steps / (ms / 1e3), "ms_per_step": ms / steps}
            model.set_attn_implementation("sdpa")
        if "materialized" in modes:
            cache = hf.build_cache(pool.attach(16), "materialize", batch=A, dtype=torch.bfloat16)
            step_ids = first.clone()
            pos = torch.full((A, 1), prefix, dtype=torch.long, device=dev)

            def loop(n):
                for _ in range(n):
                    logits = model(step_ids, past_key_values=cache, position_ids=pos, use_cache=True).logits
                    step_ids.copy_(logits[:, -1].argmax(-1, keepdim=True))
                    pos.add_(1)

            loop(1)
            ms = timed(loop, steps)
            res["materialized"] = {"tokens_per_s": A * steps / (ms / 1e3), "ms_per_step": ms / steps,
                                   "kv_bytes": sum(layer.keys.numel() * 4 for layer in cache.layers)}
    return res


if __name__ == "__main__":
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c3", choices=sorted(SHAPES))
    ap.add_argument("--steps", type=int, default=32)
    ap.add_argument("--agents", type=int, default=None)
    a = ap.parse_args()
    print(json.dumps(run(a.config, a.steps, a.agents)))
