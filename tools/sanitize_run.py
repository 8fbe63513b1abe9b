"""Small end-to-end run of every libpolykv kernel for compute-sanitizer
(memcheck / racecheck / synccheck): stream + warp-granular encode (both key
modes, both dtypes, sign diagonal), decode, pkv_k_absmax, head-sharded
encode, build stats, tensor-core and CUDA-core decode attention."""
import os
import sys
from pathlib import Path

sys.path.insert(0, str(Path(__file__).resolve().parents[1]))
import torch  # noqa: E402

import paper_2604_24971_b200 as pk  # noqa: E402
from paper_2604_24971_b200 import _lib, parallel  # noqa: E402
from paper_2604_24971_b200.attention import decode_attention  # noqa: E402

dev = torch.device("cuda")
for D, H, T, dt in ((128, 4, 300, torch.bfloat16), (64, 2, 129, torch.float32)):
    g = pk.ModelGeometry(num_layers=2, kv_heads=H, head_dim=D, seq_len=T)
    dump = pk.synth_gaussian_dump(g, seed=1, device=dev, dtype=dt, generator="torch")
    for mode in ("tensor", "block32"):
        pool = pk.build_pool(dump, k_scale_mode=mode, sign_seed=5 if mode == "tensor" else None, build_stats=True)
        _ = pool.build_stats
        for bits in (16, 32):
            pool.attach(bits).materialize_all()
        q = torch.randn(3, H, 4, D, device=dev)
        tl = torch.tensor([0, 2, 5], dtype=torch.int32, device=dev)
        tk = torch.randn(3, H, 8, D, device=dev).bfloat16()
        tv = torch.randn(3, H, 8, D, device=dev).bfloat16()
        for path in ("mma", "simt"):
            os.environ["PKV_ATTN_PATH"] = path
            _lib.reload_tuning()
            decode_attention(pool, 1, q, tail_k=tk, tail_v=tv, tail_len=tl, softmax_scale=D ** -0.5)
    hp = parallel.build_pool_head_sharded(dump, heads=range(0, H // 2 or 1))
    os.environ["PKV_CODEC_PATH"] = "warp"
    _lib.reload_tuning()
    pk.build_pool(dump, build_stats=False).attach(16).materialize_all()
    os.environ.pop("PKV_CODEC_PATH")
    _lib.reload_tuning()
torch.cuda.synchronize()
print("sanitize run ok")
