"""Generate golden vectors by running the reference `kvpool` itself.

Run in the build container (where /root/reference exists):

    NUMBA_CACHE_DIR=/tmp/numba python tests/golden/make_golden.py

Writes tests/golden/golden.npz. The reference is imported read-only from
/root/reference/pkg/src; nothing here is shipped or used at run time on the
GPU box — the committed .npz is what travels.
"""

from __future__ import annotations

import os
import sys
from pathlib import Path

import numpy as np

REF = Path("/root/reference/pkg/src")
OUT = Path(__file__).resolve().parent / "golden.npz"


def main() -> None:
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_golden")
    sys.path.insert(0, str(REF))
    import kvpool  # noqa: E402  (the reference)
    from kvpool import (  # noqa: E402
        KvTensor,
        ModelGeometry,
        build_pool,
        quantize_k,
        quantize_v,
        rotate_inverse,
        synth_gaussian_dump,
    )
    from kvpool.valuequant import pack_indices_3bit  # noqa: E402

    out: dict[str, np.ndarray] = {}
    cases = []

    def add_pool_case(name, L, H, d, T, seed, sign_seed=None, batch=1, transform=None):
        g = ModelGeometry(num_layers=L, kv_heads=H, head_dim=d, seq_len=T, batch=batch)
        dump = synth_gaussian_dump(g, seed=seed)
        if transform is not None:
            layers = []
            for li, (k, v) in enumerate(dump.layers):
                layers.append((KvTensor(g, transform(k.values, li, 0)), KvTensor(g, transform(v.values, li, 1))))
            dump = kvpool.KvDump(g, tuple(layers))
        pool = build_pool(dump, sign_seed=sign_seed)
        v16 = pool.attach(16)
        v32 = pool.attach(32)
        tr = v16.inject_all()
        out[f"{name}/geom"] = np.array([L, batch, H, T, d, -1 if sign_seed is None else sign_seed])
        for li in range(L):
            k, v = dump.layers[li]
            kq, vq = pool.layer_blocks(li)
            out[f"{name}/k_in/{li}"] = k.values
            out[f"{name}/v_in/{li}"] = v.values
            out[f"{name}/k_scale/{li}"] = np.array([kq.scale], dtype=np.float64)
            out[f"{name}/k_codes/{li}"] = kq.codes
            out[f"{name}/v_codes/{li}"] = vq.codes
            out[f"{name}/v_scales/{li}"] = vq.scales
            out[f"{name}/v_packed/{li}"] = np.frombuffer(pack_indices_3bit(vq.codes), dtype=np.uint8)
            k16, vv16 = v16.get_kv_for_layer(li)
            k32, vv32 = v32.get_kv_for_layer(li)
            out[f"{name}/k16/{li}"] = k16.values
            out[f"{name}/v16/{li}"] = vv16.values
            out[f"{name}/k32/{li}"] = k32.values
            out[f"{name}/v32/{li}"] = vv32.values
        out[f"{name}/checksums16"] = np.array(tr.checksums(), dtype=np.uint64)
        cases.append(name)

    # config-1 shape at reduced size (SmolLM2: d=64, 32 KV heads)
    add_pool_case("c1mini", L=2, H=32, d=64, T=12, seed=0)
    # Llama-3-8B head shape
    add_pool_case("d128", L=2, H=8, d=128, T=24, seed=3)
    add_pool_case("d128_sign", L=1, H=4, d=128, T=16, seed=4, sign_seed=9)
    add_pool_case("d64_batch2", L=1, H=2, d=64, T=10, seed=5, batch=2)
    for d in (8, 16, 32, 256):
        add_pool_case(f"d{d}", L=1, H=2, d=d, T=20, seed=10 + d)
    # bf16-valued inputs (the serving dtype), fed as f32
    def to_bf16(x, li, kv):
        u = np.ascontiguousarray(x, dtype=np.float32).view(np.uint32)
        r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
        return r.view(np.float32)
    add_pool_case("bf16in", L=2, H=4, d=128, T=16, seed=6, transform=to_bf16)

    # heavy tails + outliers + zero / tiny / huge rows
    def laplace(x, li, kv):
        rng = np.random.default_rng(100 + 2 * li + kv)
        y = rng.laplace(0.0, 0.1, size=x.shape).astype(np.float32)
        y[0, 0, 0, :] = 0.0                    # zero vector
        y[0, 0, 1, :] *= np.float32(1e-30)     # tiny vector
        y[0, 0, 2, :] *= np.float32(1e25)      # huge vector
        y[0, 1, 3, 5] = np.float32(40.0)       # outlier
        return y
    add_pool_case("laplace", L=2, H=2, d=128, T=8, seed=7, transform=laplace)

    # value tie adversaries: rotated images exactly on centroid midpoints
    mids = kvpool.GAUSSIAN_3BIT.midpoints
    rng = np.random.default_rng(42)
    rows = []
    for r in range(64):
        y = rng.choice(mids, size=128) * (1.0 + (r % 4) * 0.25)
        y[rng.integers(0, 128, 8)] = rng.choice([0.245, -0.756, 1.344], size=8)
        rows.append(y)
    y = np.stack(rows)[None, None]  # [1,1,64,128]
    x = rotate_inverse(y).astype(np.float32)
    g = ModelGeometry(num_layers=1, kv_heads=1, head_dim=128, seq_len=64)
    vq = quantize_v(KvTensor(g, x))
    out["tie/v_in"] = x
    out["tie/v_codes"] = vq.codes
    out["tie/v_scales"] = vq.scales

    # key known answers (pkg/tests/test_keyquant.py:41-78) + random adversaries
    def kscalar(vals):
        vals = np.asarray(vals, dtype=np.float32)
        gg = ModelGeometry(num_layers=1, kv_heads=1, head_dim=1, seq_len=vals.size)
        kq = quantize_k(KvTensor(gg, vals.reshape(1, 1, -1, 1)))
        return kq.scale, kq.codes.reshape(-1)
    kat = {
        "sym": [-2.54, 0.0, 2.54],
        "grid": list(np.array([-127, -3, 0, 64, 127], dtype=np.float64) * 2.0**-6),
        "half": list(np.array([127, 2.5, -2.5, 0.5, -0.5, 10.5]) * 2.0**-6),
    }
    half_grid = (np.arange(-127, 128) + 0.5) * 2.0**-6
    kat["halfgrid_all"] = list(np.concatenate([half_grid, [127 * 2.0**-6]]))
    for nm, vals in kat.items():
        s, c = kscalar(vals)
        out[f"kat/{nm}/in"] = np.asarray(vals, dtype=np.float32)
        out[f"kat/{nm}/scale"] = np.array([s])
        out[f"kat/{nm}/codes"] = c

    out["cases"] = np.array(cases)
    np.savez_compressed(OUT, **out)
    print(f"wrote {OUT} ({OUT.stat().st_size} bytes, {len(cases)} pool cases)")


if __name__ == "__main__":
    main()
