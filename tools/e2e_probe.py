"""e2e breakdown: pinned-host build_pool (H2D + encode) and materialize_to_host (decode + D2H)."""
import sys, time
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch
import paper_2604_24971_b200 as pk

L, H, D, T = 32, 8, 128, 4096
g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
dev = torch.device("cuda")
dump = pk.synth_gaussian_dump(g, seed=0, device=dev, dtype=torch.bfloat16, generator="torch")
host = [(k.values.cpu().pin_memory(), v.values.cpu().pin_memory()) for k, v in dump.layers]
hd = pk.KvDump(g, tuple((pk.KvTensor(g, k), pk.KvTensor(g, v)) for k, v in host))
out = [(torch.empty(g.tensor_shape, dtype=torch.bfloat16).pin_memory(),
        torch.empty(g.tensor_shape, dtype=torch.bfloat16).pin_memory()) for _ in range(L)]
ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
def allocs():
    st = torch.cuda.memory_stats()
    return st.get("num_device_alloc", 0), st.get("num_device_free", 0), st.get("num_sync_all_streams", 0)


for chunk in (4, 8, 32):
    for _ in range(3):
        n0 = allocs()
        a, b, c = ev(), ev(), ev()
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        a.record()
        p = pk.build_pool(hd, build_stats=False, device=dev, check=False, pipeline_chunk=chunk)
        b.record()
        t1 = time.perf_counter()
        p.attach(16).materialize_to_host(out, chunk=chunk)
        c.record()
        t2 = time.perf_counter()
        torch.cuda.synchronize()
        t3 = time.perf_counter()
        print(f"chunk {chunk}: build {a.elapsed_time(b):.2f} ms, materialize {b.elapsed_time(c):.2f} ms "
              f"(host enqueue {1e3*(t1-t0):.2f} / {1e3*(t2-t1):.2f}, total wall {1e3*(t3-t0):.2f}) "
              f"device alloc/free/syncs {[x - y for x, y in zip(allocs(), n0)]}", flush=True)
