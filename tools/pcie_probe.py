"""PCIe copy-engine probe: H2D alone, D2H alone, both concurrently (pinned)."""
import torch
dev = torch.device("cuda")
n = 8 * 4096 * 128  # one C3 layer tensor, bf16
L = 64
host = [torch.randn(n).to(torch.bfloat16).pin_memory() for _ in range(L)]
hout = [torch.empty(n, dtype=torch.bfloat16).pin_memory() for _ in range(L)]
devb = [torch.empty(n, dtype=torch.bfloat16, device=dev) for _ in range(L)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
def t(fn, reps=3):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.current_stream().wait_stream(s1); torch.cuda.current_stream().wait_stream(s2)
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps
def h2d():
    with torch.cuda.stream(s1):
        for h, d in zip(host, devb): d.copy_(h, non_blocking=True)
def d2h():
    with torch.cuda.stream(s2):
        for h, d in zip(hout, devb): h.copy_(d, non_blocking=True)
def both():
    h2d(); d2h()
B = L * n * 2
for name, fn in (("h2d", h2d), ("d2h", d2h), ("both", both)):
    ms = t(fn)
    print(f"{name}: {ms:.2f} ms  {B / ms / 1e6:.1f} GB/s per direction")
