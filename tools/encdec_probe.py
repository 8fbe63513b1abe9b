import sys, torch
sys.path.insert(0, "/root/repo")
import paper_2604_24971_b200 as pk
from paper_2604_24971_b200 import _codec
from paper_2604_24971_b200.pool import _Arena, _encode_layers
L, H, D, T = 32, 8, 128, 4096
g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
dev = torch.device("cuda")
dump = pk.synth_gaussian_dump(g, seed=0, device=dev, dtype=torch.float32, generator="torch")
ks = [k for k, _ in dump.layers]; vs = [v for _, v in dump.layers]
arena = _Arena(g, L, "tensor", dev)
ok = [torch.empty(g.tensor_shape, dtype=torch.bfloat16, device=dev) for _ in range(L)]
ov = [torch.empty(g.tensor_shape, dtype=torch.bfloat16, device=dev) for _ in range(L)]
junk = torch.empty(256 << 20, dtype=torch.uint8, device=dev)
def enc(): _encode_layers(ks, vs, g, pk.GAUSSIAN_3BIT, None, "tensor", device=dev, arena=arena, check=False)
def dec():
    _codec.decode(num_vectors=g.vectors_per_tensor, head_dim=D, out_dtype=torch.bfloat16, k_mode=0,
                  k_codes=[arena.k_codes[i] for i in range(L)], k_scale=[arena.k_scale[i:i+1] for i in range(L)],
                  k_bscale=None, v_packed=[arena.v_packed[i] for i in range(L)],
                  v_scales=[arena.v_scales[i, :g.vectors_per_tensor] for i in range(L)],
                  centroids=pk.GAUSSIAN_3BIT.centroids, sign_seed=None, k_out=ok, v_out=ov, device=dev)
def graph(fn):
    s = torch.cuda.Stream(); s.wait_stream(torch.cuda.current_stream())
    with torch.cuda.stream(s): fn()
    torch.cuda.current_stream().wait_stream(s)
    gr = torch.cuda.CUDAGraph()
    with torch.cuda.graph(gr): fn()
    return gr.replay
E, Dd = graph(enc), graph(dec)
def run(seq, n=30):
    for _ in range(3):
        for f, _ in seq: f()
    torch.cuda.synchronize()
    ev = [[torch.cuda.Event(enable_timing=True) for _ in range(len(seq) + 1)] for _ in range(n)]
    for i in range(n):
        for j, (f, _) in enumerate(seq):
            ev[i][j].record(); f()
        ev[i][-1].record()
    torch.cuda.synchronize()
    return [round(sum(ev[i][j].elapsed_time(ev[i][j + 1]) for i in range(n)) / n * 1e3, 1) for j in range(len(seq))]
print("enc,enc", run([(E, "e"), (E, "e")]))
print("enc,dec", run([(E, "e"), (Dd, "d")]))
print("enc,junkwrite,dec", run([(E, "e"), (lambda: junk.fill_(1), "j"), (Dd, "d")]))
print("dec,junkread?,enc", run([(Dd, "d"), (lambda: junk.sum(), "r"), (E, "e")]))
ED = graph(lambda: (enc(), dec()))
print("one graph enc+dec", run([(ED, "ed")]))
print("two graphs enc,dec", run([(E, "e"), (Dd, "d")]))
def run_noev(seq, n=30):
    for _ in range(3):
        for f in seq: f()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        for f in seq: f()
    b.record(); torch.cuda.synchronize()
    return round(a.elapsed_time(b) / n * 1e3, 1)
print("no events: two graphs", run_noev([E, Dd]), "one graph", run_noev([ED]))
