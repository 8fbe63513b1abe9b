"""Time decode attention (all layers, batched agents) with CUDA graphs; C3 shape."""
import sys, torch
from pathlib import Path
sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import paper_2604_24971_b200 as pk
from paper_2604_24971_b200.attention import decode_attention
L, H, D, T, A, G = 32, 8, 128, 4096, 15, 4
if len(sys.argv) > 1 and sys.argv[1] == "c2":
    L, H, D, T, A, G = 24, 32, 64, 1851, 5, 1
if len(sys.argv) > 2:  # agent count override (e.g. few agents: 16-row tiles)
    A = int(sys.argv[2])
dev = torch.device("cuda")
g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
pool = pk.build_pool(pk.synth_gaussian_dump(g, seed=0, device=dev, dtype=torch.bfloat16, generator="torch"))
q = torch.randn(A, H, G, D, device=dev, dtype=torch.bfloat16)
out = torch.empty_like(q)
need = pk._lib.load().pkv_attention_workspace_bytes(A, H, G, D, T)
ws = torch.empty((need + 3) // 4, dtype=torch.float32, device=dev)
def step():
    for li in range(L):
        decode_attention(pool, li, q, softmax_scale=D ** -0.5, out=out, workspace=ws)
step(); torch.cuda.synchronize()
gr = torch.cuda.CUDAGraph()
s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
with torch.cuda.stream(s):
    step()
torch.cuda.current_stream().wait_stream(s)
with torch.cuda.graph(gr):
    step()
for _ in range(3): gr.replay()
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
n = 50
e0.record()
for _ in range(n): gr.replay()
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / n
flops = 2 * 2 * A * G * T * D * H * L
print(f"attention step (all {L} layers, {A} agents): {ms:.3f} ms -> {A / ms * 1e3:.0f} tok/s, {flops / ms / 1e9:.1f} TFLOP/s")
