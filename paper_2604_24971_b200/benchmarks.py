"""Timing harness with the kvpool.bench API (bench.py:19-99), timed on the device.

run_bench builds a pool from a synthetic dump and has N agents decode every
layer `repetitions` times. The reference spins N host threads; here the
agents' decodes are enqueued on one stream and timed with CUDA events.
Bytes are counted like the reference: the decoded tensors as f32
(bench.py:88), independent of decode_bits.
"""

from __future__ import annotations

from dataclasses import dataclass

import torch

from .model import ModelGeometry, synth_gaussian_dump
from .pool import build_pool


@dataclass(frozen=True)
class BenchResult:
    geometry: ModelGeometry
    agents: int
    repetitions: int
    build_seconds: float
    decode_seconds_per_layer: float
    decoded_bytes: int
    wall_seconds: float
    aggregate_bytes_per_second: float


def _elapsed(fn) -> float:
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    s.record()
    fn()
    e.record()
    e.synchronize()
    return s.elapsed_time(e) / 1e3


def run_bench(geometry: ModelGeometry, agents: int = 1, repetitions: int = 3, seed: int = 0,
              decode_bits: int = 16) -> BenchResult:
    if agents < 1:
        raise ValueError(f"agents must be >= 1, got {agents}")
    if repetitions < 1:
        raise ValueError(f"repetitions must be >= 1, got {repetitions}")
    dump = synth_gaussian_dump(geometry, seed=seed, device="cuda")
    build_pool(dump, build_stats=False)  # warm-up (module load, allocator)
    holder = {}
    build_seconds = _elapsed(lambda: holder.setdefault("p", build_pool(dump, build_stats=False)))
    pool = holder["p"]
    view = pool.attach(decode_bits)
    view.get_kv_for_layer(0)
    per_layer = _elapsed(lambda: [view.get_kv_for_layer(i) for i in range(pool.num_layers)]) / pool.num_layers
    views = [pool.attach(decode_bits) for _ in range(agents)]

    def sweep():
        for _ in range(repetitions):
            for v in views:
                v.materialize_all()

    wall = _elapsed(sweep)
    decoded = agents * repetitions * pool.num_layers * 2 * geometry.elements_per_tensor * 4
    return BenchResult(geometry, agents, repetitions, build_seconds, per_layer, decoded, wall,
                       decoded / wall if wall > 0 else 0.0)
