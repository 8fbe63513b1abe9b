"""Pool verification on the device (kvpool `verify`, cli.py:216-315).

The reference's `kvpool verify` rebuilds the pool from its source dump and
compares FNV checksums, runs N concurrent reader threads and checks their
injection transcripts agree, checks the fidelity bounds and that pool bytes do
not grow with attached agents. The same checks here run on the GPU: the
rebuild and the reader decodes are device launches; readers run in Python
threads on separate CUDA streams; bit-identity is checked on the device, and
the first reader's FNV-1a transcript is also compared with a fresh view's.
"""

from __future__ import annotations

import threading
from dataclasses import dataclass, field

import torch

from .metrics import distortion_report
from .model import KvDump
from .pool import SharedPool, build_pool


@dataclass
class VerifyReport:
    checks: list = field(default_factory=list)  # (name, ok, detail)

    def add(self, name: str, ok: bool, detail: str = "") -> None:
        self.checks.append((name, bool(ok), detail))

    @property
    def ok(self) -> bool:
        return all(ok for _, ok, _ in self.checks)

    def lines(self) -> list[str]:
        return [f"{'ok  ' if ok else 'FAIL'} - {name}" + (f": {d}" if d else "") for name, ok, d in self.checks]


def verify_pool(dump: KvDump, pool: SharedPool, *, agents=(1, 3, 15), decode_bits: int = 16) -> VerifyReport:
    """Run the reference's verify checks (cli.py:239-313) against `pool`."""
    rep = VerifyReport()
    if dump.geometry != pool.geometry:
        rep.add("geometry matches the dump", False, f"{dump.geometry} vs {pool.geometry}")
        return rep

    # payload bits: a fresh build from the dump reproduces the pool exactly
    fresh = build_pool(dump, pool.codebook, pool.sign_seed, k_scale_mode=pool.k_scale_mode, build_stats=False)
    bad = []
    for i in range(pool.num_layers):
        (kq, vq), (rk, rv) = pool.layer_blocks(i), fresh.layer_blocks(i)
        same = torch.equal(kq.codes, rk.codes) and torch.equal(vq.packed, rv.packed) and \
            torch.equal(vq.scales, rv.scales)
        if kq.mode == "tensor":
            same = same and kq.scale == rk.scale
        else:
            same = same and torch.equal(kq.block_scales, rk.block_scales)
        if not same:
            bad.append(i)
    rep.add("payload matches a fresh build", not bad, f"layers {bad}" if bad else "")

    # concurrent readers (threads, one CUDA stream each) hand out identical bits
    n = max(agents)
    ref = pool.attach(decode_bits).materialize_all()
    ref_sums = pool.attach(decode_bits).inject_all().checksums()
    results: list = [None] * n
    barrier = threading.Barrier(n)

    def reader(slot: int) -> None:
        view = pool.attach(decode_bits)
        stream = torch.cuda.Stream(pool.device)
        barrier.wait()
        with torch.cuda.stream(stream):
            out = view.materialize_all()
            ok = all(torch.equal(a, b) and torch.equal(c, d) for (a, c), (b, d) in zip(out, ref))
        stream.synchronize()
        results[slot] = ok

    threads = [threading.Thread(target=reader, args=(i,)) for i in range(n)]
    for t in threads:
        t.start()
    for t in threads:
        t.join()
    diverged = [i for i, ok in enumerate(results) if not ok]
    sums_ok = pool.attach(decode_bits).inject_all().checksums() == ref_sums
    rep.add(f"{n} concurrent readers agree bit-for-bit", not diverged and sums_ok,
            f"readers {diverged} diverged" if diverged else ("" if sums_ok else "FNV transcripts differ"))

    # fidelity bounds against the source dump
    report = distortion_report(dump, pool)
    k_bad = [s.layer for s in report.layer_stats if s.k_max_err > (s.k_scale / 2.0) * (1.0 + 1e-6)]
    if pool.k_scale_mode == "tensor":
        rep.add("key error within scale/2 on every layer", not k_bad, f"layers {k_bad}" if k_bad else "")
    rep.add(f"value distortion under the {report.v_bound:.4f} ceiling on every layer",
            not report.v_bound_violations,
            f"layers {list(report.v_bound_violations)}" if report.v_bound_violations else "")

    # pool memory must not scale with attached agents: the pool's own HBM
    # footprint and the device allocator's total both stay put while views
    # are attached (a view holds no tensor state, pool.py:217-222)
    torch.cuda.synchronize(pool.device)
    base_alloc = torch.cuda.memory_allocated(pool.device)
    base_pool = pool.device_nbytes()
    sizes = []
    views = []
    for count in agents:
        views.extend(pool.attach(decode_bits) for _ in range(count))
        torch.cuda.synchronize(pool.device)
        sizes.append((len(views), pool.device_nbytes(), torch.cuda.memory_allocated(pool.device) - base_alloc))
    invariant = all(p == base_pool and grown == 0 for _, p, grown in sizes)
    rep.add(f"pool HBM bytes invariant across agent counts {tuple(agents)}", invariant,
            "" if invariant else f"(agents, pool bytes, allocator growth): {sizes}")
    return rep


__all__ = ["VerifyReport", "verify_pool"]
