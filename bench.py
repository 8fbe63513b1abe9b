#!/usr/bin/env python
"""Benchmark of the SharedKVPool compress/inject hot path on B200.

One step = compress every layer of a synthetic KV dump into the packed pool
(one pkv_encode launch: q8_0 keys + FWHT/RMS/3-bit Lloyd-Max packed values)
+ materialise every layer back to bf16 for one agent (one pkv_decode launch).
That is the reference's build_pool + inject_all round trip
(kvpool/pool.py:258-293, :239-255). metric = algorithmic bytes / time (GB/s).

Secondary: shared-pool decode attention over the packed pool for all agents
(pkv_decode_attention, one launch pair per layer), reported as tokens/s.

    python bench.py [--gpus N --steps K --warmup W --config c3 --dtype bf16]
    python bench.py --impl reference ...   # the reference algorithm on host cores
"""

from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time
from pathlib import Path

ROOT = Path(__file__).resolve().parent
sys.path.insert(0, str(ROOT))

CONFIGS = {
    # name: (layers, kv_heads, head_dim, seq_len, agents, group, description)
    "c1": (24, 32, 64, 600, 3, 1, "SmolLM2-1.7B-shape KV (L24 H32 d64), T=600, 3 agents"),
    "c2": (24, 32, 64, 1851, 5, 1, "SmolLM2-1.7B-shape KV (L24 H32 d64), T=1851, 5 agents"),
    "c3": (32, 8, 128, 4096, 15, 4, "Llama-3-8B-shape KV (L32 H8 d128 GQA g4), T=4096, 15 agents"),
    "c4": (32, 8, 128, 7194, 15, 4, "Llama-3-8B-shape KV (L32 H8 d128 GQA g4), T=7194, 15 agents"),
}
METRIC = "KV compress+dequant GB/s (HBM roofline); shared-pool decode tok/s"


def algorithmic_bytes(L, H, D, T, in_bytes, out_bytes, k_mode="tensor"):
    """per-element bytes of compress and materialise."""
    n = H * T * D
    vecs = H * T
    k_scale_b = 4 if k_mode == "tensor" else 2 * ((n + 31) // 32)
    comp = L * (n * in_bytes + n + k_scale_b + n * in_bytes + 3 * n / 8 + 4 * vecs)
    deq = L * (n + k_scale_b + n * out_bytes + 3 * n / 8 + 4 * vecs + n * out_bytes)
    return comp, deq


# ---------------------------------------------------------------------------
# clocks
# ---------------------------------------------------------------------------
class ClockSampler:
    """SM clocks and throttle reasons sampled every ~5 ms during the timed
    region (NVML via nvidia-ml-py; falls back to nvidia-smi)."""

    # NVML clocks-event reason bits
    REASONS = {0x8: "hw_slowdown", 0x40: "hw_thermal_slowdown", 0x20: "sw_thermal_slowdown", 0x4: "sw_power_cap"}

    def __init__(self, index: int):
        self.index = index
        self.samples = []
        self._stop = threading.Event()
        self._t = None
        self._nvml = None
        try:
            import pynvml

            pynvml.nvmlInit()
            self._nvml = pynvml
            self._h = pynvml.nvmlDeviceGetHandleByIndex(index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self._h, pynvml.NVML_CLOCK_SM)
        except Exception:
            self._nvml = None
            self.max_mhz = None

    def _sample(self):
        if self._nvml is not None:
            p = self._nvml
            sm = p.nvmlDeviceGetClockInfo(self._h, p.NVML_CLOCK_SM)
            try:
                r = p.nvmlDeviceGetCurrentClocksEventReasons(self._h)
            except Exception:
                r = p.nvmlDeviceGetCurrentClocksThrottleReasons(self._h)
            return sm, [n for bit, n in self.REASONS.items() if r & bit]
        out = subprocess.run(["nvidia-smi", f"--id={self.index}", "--query-gpu=clocks.sm,clocks.max.sm",
                              "--format=csv,noheader,nounits"], capture_output=True, text=True, timeout=5).stdout
        sm, mx = (float(x) for x in out.strip().split(",")[:2])
        self.max_mhz = mx
        return sm, []

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self._sample())
            except Exception:
                pass
            self._stop.wait(0.005)

    def __enter__(self):
        self._t = threading.Thread(target=self._run, daemon=True)
        self._t.start()
        return self

    def __exit__(self, *exc):
        self._stop.set()
        self._t.join(timeout=6)

    def summary(self):
        if not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": self.max_mhz, "reasons": ["unsampled"]}
        sm = [s for s, _ in self.samples]
        reasons = sorted({r for _, rs in self.samples for r in rs})
        return {"sm_mhz": statistics.median(sm), "sm_max_mhz": self.max_mhz, "reasons": reasons,
                "samples": len(self.samples), "source": "nvml" if self._nvml else "nvidia-smi"}


def measured_peaks():
    p = ROOT / "MEASURED_PEAKS.json"
    if p.exists():
        d = json.loads(p.read_text())
        return float(d.get("hbm_gbs", 6650.0)), "measured"
    return 6650.0, "fallback"


# ---------------------------------------------------------------------------
# CPU baseline: the UNMODIFIED reference (kvpool from baseline/_ref) on host cores
# ---------------------------------------------------------------------------
REF_DIR = ROOT / "baseline" / "_ref"
_REF = {}


def reference_available() -> bool:
    return (REF_DIR / "kvpool" / "__init__.py").exists()


def _ref_init(H, D, T, use_ref):
    """Worker initialiser: import the stock kvpool (or the labelled oracle
    port when baseline/_ref is absent) and draw one synthetic layer with the
    reference's own generator (model.py:250-273), reused by every task."""
    os.environ.setdefault("NUMBA_CACHE_DIR", "/tmp/numba_ref_bench")
    if use_ref:
        sys.path.insert(0, str(REF_DIR))
        import kvpool

        g = kvpool.ModelGeometry(num_layers=1, kv_heads=H, head_dim=D, seq_len=T)
        _REF["kv"] = kvpool
        _REF["dump"] = kvpool.synth_gaussian_dump(g, seed=0)
    else:
        import numpy as np

        rng = np.random.default_rng(0)
        std = float(np.sqrt(1.0 / D))
        _REF["kv"] = None
        _REF["k"] = rng.normal(0.0, std, size=(1, H, T, D)).astype(np.float32)
        _REF["v"] = rng.normal(0.0, std, size=(1, H, T, D)).astype(np.float32)


def _ref_layer(_i):
    """One layer of the compress/inject round trip through the reference's
    public API, stock code path: build_pool (quantize_k + quantize_v + build
    stats, pool.py:258-293) then attach(16).get_kv_for_layer (pool.py:229-237)."""
    kv = _REF["kv"]
    t0 = time.perf_counter()
    if kv is not None:
        pool = kv.build_pool(_REF["dump"])
        pool.attach(16).get_kv_for_layer(0)
    else:  # labelled fallback: the oracle port (oracle/kvpool_oracle.py)
        from oracle import kvpool_oracle as O

        s, kc = O.quantize_k_tensor(_REF["k"])
        vc, vs = O.quantize_v(_REF["v"])
        O.decode_layer(kc, s, vc, vs, 16)
    return time.perf_counter() - t0


def cpu_info() -> dict:
    import platform

    import numpy as np

    model = platform.processor() or ""
    try:
        for line in Path("/proc/cpuinfo").read_text().splitlines():
            if line.startswith("model name"):
                model = line.split(":", 1)[1].strip()
                break
    except OSError:
        pass
    return {"cpu_model": model, "os_cpu_count": os.cpu_count(), "numpy": np.__version__,
            "python": platform.python_version()}


class ReferenceCPU:
    """A pool of `procs` spawn-started worker processes, each running the
    unmodified reference on whole layers (the reference's build_pool is a
    single-threaded loop over layers, pool.py:271, so layers are the unit of
    parallelism: BASELINE.md §4 step 3)."""

    def __init__(self, H, D, T, procs=None):
        import multiprocessing as mp
        from concurrent.futures import ProcessPoolExecutor

        self.use_ref = reference_available()
        self.procs = procs or os.cpu_count() or 1
        self.ex = ProcessPoolExecutor(max_workers=self.procs, mp_context=mp.get_context("spawn"),
                                      initializer=_ref_init, initargs=(H, D, T, self.use_ref))
        list(self.ex.map(_ref_layer, range(self.procs)))  # start + warm every worker

    @property
    def kind(self):
        return "reference" if self.use_ref else "port"

    def step(self, layers):
        """Wall seconds for `layers` layers spread over the workers."""
        t0 = time.perf_counter()
        list(self.ex.map(_ref_layer, range(layers)))
        return time.perf_counter() - t0

    def close(self):
        self.ex.shutdown()


def run_reference(args, cfg):
    """`--impl reference`: the reference's own CPU implementation of the path
    (stock kvpool from baseline/_ref; the oracle port only if it is missing,
    labelled kind=port) on all host cores, same config, metric and unit as our
    arm. A step is the full config (all layers) unless warmup + steps would
    exceed ~3 minutes, in which case each step is a bounded sample of whole
    layers (stated in config.sample, same_config false)."""
    L, H, D, T, agents, group, desc = cfg
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return 0
    ref = ReferenceCPU(H, D, T)
    try:
        t_full = ref.step(L)  # first warmup step: the whole config
        n_rest = args.steps + max(0, args.warmup - 1)
        budget_s = 180.0
        layers = L
        if n_rest * t_full > budget_s:
            layers = max(ref.procs, min(L, int(L * budget_s / (n_rest * t_full))))
            layers = max(1, layers // ref.procs) * ref.procs if layers >= ref.procs else layers
        for _ in range(args.warmup - 1):
            ref.step(layers)
        times = [ref.step(layers) for _ in range(args.steps)]
    finally:
        ref.close()
    sec = sum(times) / len(times)
    comp, deq = algorithmic_bytes(layers, H, D, T, 4, 2)  # the reference computes on f32 input
    value = (comp + deq) / sec / 1e9
    same = layers == L
    sample = (f"{layers} of {L} layers [1,{H},{T},{D}] f32 per step over {ref.procs} processes: stock "
              f"kvpool build_pool + attach(16).get_kv_for_layer per layer")
    line = {
        "metric": METRIC, "impl": "reference", "value": value, "unit": "GB/s", "n_gpus": args.gpus,
        "steps": args.steps, "warmup": args.warmup, "ms_per_step": sec * 1e3, "higher_is_better": True,
        "scaling": "weak", "vs_baseline": None, "dtype": "f32 in (numpy f64 internal)", "data": "synthetic",
        "config": {"workload": desc, "sample": sample, "same_config": same, "layers_per_step": layers},
        "cpu_baseline": {"value": value, "unit": "GB/s", "cores": ref.procs, "kind": ref.kind, "sample": sample,
                         **cpu_info()},
        "e2e": {"value": value, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
    }
    print(json.dumps(line), flush=True)
    return 0


# ---------------------------------------------------------------------------
# our implementation
# ---------------------------------------------------------------------------
def run_ours(args, cfg):
    """Our arm. At N GPUs (one process per GPU, torchrun) the step is the
    north_star pipeline with the config split over the GPUs: each rank
    compresses its contiguous layer shard (one pkv_encode launch), ONE NCCL
    all_gather_into_tensor replicates the packed pool (layer-major arena, so
    the collective moves exactly the pool bytes), and each rank materialises
    its shard to bf16 (one pkv_decode launch). Total work is fixed (strong
    scaling); at N=1 the gather is absent. Decode attention: the config's
    agents are partitioned over the ranks, each attending over its replica of
    the whole pool (no per-step collective)."""
    import torch
    import torch.distributed as dist

    import paper_2604_24971_b200 as pk
    from paper_2604_24971_b200 import _codec, parallel
    from paper_2604_24971_b200.attention import decode_attention
    from paper_2604_24971_b200.pool import _Arena, _encode_layers, pool_from_arena, raise_for_status

    L, H, D, T, agents, group, desc = cfg
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    plumbing = args.dist_backend == "gloo"  # N>1 code path on fewer GPUs: exercises, does not measure
    if torch.cuda.device_count() <= local and not plumbing:
        raise SystemExit(f"bench.py: rank {rank} needs cuda:{local}, {torch.cuda.device_count()} visible")
    if plumbing:
        local = local % torch.cuda.device_count()
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        if plumbing:
            dist.init_process_group("gloo")
        else:
            os.environ.setdefault("NCCL_DEBUG", "INFO")  # communicator size in the log (nRanks)
            os.environ.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
            dist.init_process_group("nccl", device_id=dev)
    g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
    mine = list(parallel.layer_shard(L, world, rank))
    my_agents = parallel.partition_agents(agents, world, rank)
    rows_max = len(parallel.layer_shard(L, world, 0))
    even = all(len(parallel.layer_shard(L, world, r)) == rows_max for r in range(world))
    stream = torch.cuda.current_stream(dev)
    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    n, vecs = g.elements_per_tensor, g.vectors_per_tensor
    cb = pk.GAUSSIAN_3BIT

    def max_over_ranks(ms):
        if world == 1:
            return ms
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    def barrier():
        if world > 1:
            dist.barrier()

    def capture(fn):
        """CUDA-graph a launch sequence (the timed loop then measures the GPU,
        not the Python/ctypes enqueue path); None if capture is unavailable."""
        if args.no_graph:
            return None
        try:
            side = torch.cuda.Stream(dev)
            side.wait_stream(torch.cuda.current_stream(dev))
            with torch.cuda.stream(side):
                fn()
            torch.cuda.current_stream(dev).wait_stream(side)
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr):
                fn()
            torch.cuda.synchronize(dev)
            return gr.replay
        except Exception as exc:  # noqa: BLE001
            print(f"[bench] graph capture unavailable ({exc}); eager launches", file=sys.stderr)
            return None

    def shard_inputs(dtype):
        """This rank's layers of a synthetic dump, drawn on the device."""
        gen = torch.Generator(device=dev)
        out = []
        for li in mine:
            gen.manual_seed(1000 + li)
            k = torch.randn(g.tensor_shape, generator=gen, device=dev, dtype=torch.float32) * D ** -0.5
            v = torch.randn(g.tensor_shape, generator=gen, device=dev, dtype=torch.float32) * D ** -0.5
            out.append((pk.KvTensor(g, k.to(dtype)), pk.KvTensor(g, v.to(dtype))))
        return out

    def measure(dtype, steps, with_clocks=False, k_mode=None):
        """Time `steps` steps of encode(shard) [+ all-gather] + decode(shard)."""
        km = k_mode or args.k_mode
        in_b = 2 if dtype == torch.bfloat16 else 4
        layers = shard_inputs(dtype)
        ks = [k for k, _ in layers]
        vs = [v for _, v in layers]
        arena = _Arena(g, len(mine), km, dev)
        full_flat = (torch.empty((world * rows_max, arena.layer_bytes), dtype=torch.uint8, device=dev)
                     if world > 1 else None)
        out_k = [torch.empty(g.tensor_shape, dtype=torch.bfloat16, device=dev) for _ in mine]
        out_v = [torch.empty(g.tensor_shape, dtype=torch.bfloat16, device=dev) for _ in mine]
        kmode = pk.keyquant.K_MODES[km]

        def encode():
            _encode_layers(ks, vs, g, cb, None, km, device=dev, arena=arena, check=False)

        def gather():
            if world > 1:
                arena.status_row.copy_(arena.status)
                if even and not plumbing:
                    dist.all_gather_into_tensor(full_flat, arena.flat)
                elif even:
                    full_flat.copy_(parallel.gather_arena(arena, L).flat)
                else:
                    parallel.gather_arena(arena, L)

        def decode():
            _codec.decode(num_vectors=vecs, head_dim=D, out_dtype=torch.bfloat16, k_mode=kmode,
                          k_codes=[arena.k_codes[i] for i in range(len(mine))],
                          k_scale=[arena.k_scale[i:i + 1] for i in range(len(mine))] if km == "tensor" else None,
                          k_bscale=[arena.k_bscale[i] for i in range(len(mine))] if km == "block32" else None,
                          v_packed=[arena.v_packed[i] for i in range(len(mine))],
                          v_scales=[arena.v_scales[i, :vecs] for i in range(len(mine))],
                          centroids=cb.centroids, sign_seed=None, k_out=out_k, v_out=out_v, device=dev)

        for _ in range(args.warmup):
            encode()
            gather()
            decode()
        raise_for_status(arena.status)
        torch.cuda.synchronize(dev)
        # (the all-gather runs eager: one NCCL call per step; capturing a
        # collective is not needed to time it and a failed capture must not
        # disturb the encode / decode graphs)
        run_enc, run_gat, run_dec = capture(encode) or encode, gather, capture(decode) or decode
        graphed = not args.no_graph and run_enc is not encode
        for _ in range(args.warmup):
            run_enc()
            run_gat()
            run_dec()
        torch.cuda.synchronize(dev)
        barrier()
        marks = [(ev(), ev(), ev(), ev()) for _ in range(steps)]
        start, end = ev(), ev()
        clocks = ClockSampler(local) if with_clocks else None
        if clocks:
            clocks.__enter__()
        torch.cuda.synchronize(dev)
        start.record(stream)
        for a_, b_, c_, d_ in marks:
            a_.record(stream)
            run_enc()
            b_.record(stream)
            run_gat()
            c_.record(stream)
            run_dec()
            d_.record(stream)
        end.record(stream)
        torch.cuda.synchronize(dev)
        if clocks:
            clocks.__exit__(None, None, None)
        res = {
            "ms_step": max_over_ranks(start.elapsed_time(end) / steps),
            "encode_ms": sum(a_.elapsed_time(b_) for a_, b_, _, _ in marks) / steps,
            "gather_ms": sum(b_.elapsed_time(c_) for _, b_, c_, _ in marks) / steps,
            "decode_ms": sum(c_.elapsed_time(d_) for _, _, c_, d_ in marks) / steps,
            "graphed": graphed, "in_b": in_b, "clocks": clocks.summary() if clocks else None,
            "replays": int(arena.replay.item()), "arena": arena, "full_flat": full_flat,
        }
        comp_b, deq_b = algorithmic_bytes(L, H, D, T, in_b, 2, km)
        res["comp_b"], res["deq_b"] = comp_b, deq_b
        res["value"] = (comp_b + deq_b) / (res["ms_step"] / 1e3) / 1e9
        if world == 1:
            none = [None] * len(mine)

            def time_it(fn, k):
                s_, e_ = ev(), ev()
                fn()
                torch.cuda.synchronize(dev)
                s_.record(stream)
                for _ in range(k):
                    fn()
                e_.record(stream)
                torch.cuda.synchronize(dev)
                return s_.elapsed_time(e_) / k

            enc_k = capture(lambda: _encode_layers(ks, none, g, cb, None, km, device=dev, arena=arena,
                                                   check=False))
            enc_v = capture(lambda: _encode_layers(none, vs, g, cb, None, km, device=dev, arena=arena,
                                                   check=False))
            if enc_k and enc_v:
                res["encode_keys_ms"] = time_it(enc_k, steps)
                res["encode_values_ms"] = time_it(enc_v, steps)
        return res

    main_dt = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    other_dt = torch.float32 if main_dt == torch.bfloat16 else torch.bfloat16
    r = measure(main_dt, args.steps, with_clocks=True)
    variant = None if args.skip_variant else measure(other_dt, max(5, min(args.steps, 50)))
    # the north star's key format (q8_0 per 32 elements, fp16 scales), same input dtype:
    # reported beside the headline, which keeps the reference's per-tensor keys
    other_km = "block32" if args.k_mode == "tensor" else "tensor"
    kvariant = None if args.skip_variant else measure(main_dt, max(5, min(args.steps, 50)), k_mode=other_km)
    ms_step, value, comp_b, deq_b, in_b = r["ms_step"], r["value"], r["comp_b"], r["deq_b"], r["in_b"]

    # the pool every rank now holds (gathered), for attention
    arena = r["arena"]
    if world > 1:
        full = _Arena.like(arena, r["full_flat"][:L]) if even else parallel.gather_arena(arena, L)
        raise_for_status(full.status)  # every rank's status words travelled inside the rows
        pool = pool_from_arena(full, g, cb, None, args.k_mode)
    else:
        pool = pool_from_arena(arena, g, cb, None, args.k_mode)

    # ---- e2e through the public API with host buffers ----
    e2e = None
    if not args.skip_e2e:
        host = [(k.values.cpu().pin_memory(), v.values.cpu().pin_memory()) for k, v in shard_inputs(main_dt)]
        placeholder = host[0]
        by_layer = dict(zip(mine, host))
        host_dump = pk.KvDump(g, tuple((pk.KvTensor(g, by_layer.get(i, placeholder)[0]),
                                        pk.KvTensor(g, by_layer.get(i, placeholder)[1])) for i in range(L)))
        host_out = [(torch.empty(g.tensor_shape, dtype=torch.bfloat16).pin_memory(),
                     torch.empty(g.tensor_shape, dtype=torch.bfloat16).pin_memory()) for _ in mine]
        inflight = []

        def e2e_step():
            # build uploads the pinned inputs (chunk-wise, overlapped with the
            # encode), materialize_to_host overlaps decode with the D2H copies.
            # The host may run one step ahead but no further (unbounded
            # run-ahead grows the caching allocator: cudaMalloc stalls).
            if world == 1:
                p = pk.build_pool(host_dump, build_stats=False, device=dev, check=False)
            else:
                p = parallel.build_pool_sharded(host_dump, device=dev, check=False)
            p.attach(16).materialize_to_host(host_out, layers=mine)
            done = torch.cuda.Event()
            done.record(stream)
            inflight.append(done)
            if len(inflight) > 1:
                inflight.pop(0).synchronize()

        for _ in range(max(3, args.warmup)):
            e2e_step()
        torch.cuda.synchronize(dev)
        es, ee = ev(), ev()
        n_e2e = max(3, min(args.steps, 20))
        barrier()
        es.record(stream)
        for _ in range(n_e2e):
            e2e_step()
        ee.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = max_over_ranks(es.elapsed_time(ee) / n_e2e)
        e2e = {"value": (comp_b + deq_b) / (e2e_ms / 1e3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": 2 * L * n * in_b, "d2h_bytes_per_step": 2 * L * n * 2,
               "ms_per_step": e2e_ms, "api": "build_pool / parallel.build_pool_sharded + "
                                             "attach(16).materialize_to_host (pinned host in and out)",
               "bytes_note": "h2d/d2h summed over all ranks (each rank moves its layer shard)"}

    # ---- shared-pool decode attention: agents partitioned over ranks ----
    attn = None
    if not args.skip_attention and D in (64, 128):
        a_ms = 0.0
        if my_agents:
            q = torch.randn(len(my_agents), H, group, D, device=dev, dtype=torch.bfloat16)
            outa = torch.empty_like(q)
            need = pk._lib.load().pkv_attention_workspace_bytes(len(my_agents), H, group, D, T)
            ws = torch.empty((need + 3) // 4, dtype=torch.float32, device=dev)

            def attn_step():
                for li in range(L):
                    decode_attention(pool, li, q, softmax_scale=D ** -0.5, out=outa, workspace=ws)

            run_attn = capture(attn_step) or attn_step
            for _ in range(3):
                run_attn()
            torch.cuda.synchronize(dev)
        barrier()
        if my_agents:
            s2, e2 = ev(), ev()
            s2.record(stream)
            for _ in range(args.steps):
                run_attn()
            e2.record(stream)
            torch.cuda.synchronize(dev)
            a_ms = s2.elapsed_time(e2) / args.steps
        a_ms = max_over_ranks(a_ms)
        pool_bytes = L * (n * (1 + 3 / 8) + 4 * vecs + 4)
        flops = 4.0 * L * agents * H * group * T * D  # q.k and p.v for every query row of every head and layer
        attn = {"tokens_per_s": agents / (a_ms / 1e3), "ms_per_token_step": a_ms, "agents": agents,
                "agents_per_rank": len(my_agents), "layers": L,
                "scope": "attention only (all layers), each rank batches its agents over its pool replica",
                "pool_gbs_per_rank": pool_bytes / (a_ms / 1e3) / 1e9,
                "tflops": flops / (a_ms / 1e3) / 1e12 if world == 1 else None,
                "kernel": "prefix (mma.sync f16 / f32 acc, split-f16 Q and centroids) + combine"}

    # ---- model-level shared-pool decode (random-init model of the config's shape) ----
    dec_e2e = None
    if not args.skip_decode_e2e and args.config in ("c2", "c3") and rank == 0 and world == 1:
        try:
            sys.path.insert(0, str(ROOT / "tools"))
            import decode_bench

            dec_e2e = decode_bench.run(args.config, steps=32)
            dec_e2e["scope"] = ("greedy decode, agents in lockstep, random-init model; pooled = PooledCache + "
                                "pkv_decode_attention, materialized = per-agent bf16 DynamicCache + SDPA "
                                "(reference semantics) on the same GPU")
        except Exception as exc:  # noqa: BLE001
            dec_e2e = {"error": repr(exc)[:300]}

    peak, peak_kind = measured_peaks()
    kscale_b = 4 if args.k_mode == "tensor" else 2 * ((n + 31) // 32)
    Lr = len(mine)
    enc_bytes = Lr * (2 * n * in_b + n + kscale_b + 3 * n / 8 + 4 * vecs)   # this rank's shard
    dec_bytes = Lr * (n + kscale_b + 3 * n / 8 + 4 * vecs + 2 * n * 2)
    kernels = {"encode": (r["encode_ms"], enc_bytes), "decode": (r["decode_ms"], dec_bytes)}
    dom_name = max(kernels, key=lambda k: kernels[k][0])
    dom_ms, dom_bytes = kernels[dom_name]
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    traffic = None
    prof = ROOT / "profiles" / "traffic.json"
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(f"{args.config}/{args.dtype}/{dom_name}")
        except Exception:
            traffic = None

    def kernel_block(res, label):
        d = {"dtype_in": label, "step_ms": res["ms_step"], "value_gbs": res["value"],
             "encode_ms": res["encode_ms"], "decode_ms": res["decode_ms"],
             "encode_gbs_per_gpu": Lr * (2 * n * res["in_b"] + n + kscale_b + 3 * n / 8 + 4 * vecs)
             / (res["encode_ms"] / 1e3) / 1e9,
             "decode_gbs_per_gpu": dec_bytes / (res["decode_ms"] / 1e3) / 1e9,
             "cuda_graph": res["graphed"], "replayed_vectors": res["replays"]}
        if world > 1:
            d["gather_ms"] = res["gather_ms"]
        if "encode_keys_ms" in res:
            d["encode_keys_ms"] = res["encode_keys_ms"]
            d["encode_values_ms"] = res["encode_values_ms"]
        d["encode_frac_of_peak"] = d["encode_gbs_per_gpu"] / peak
        return d

    cpu = None
    if rank == 0 and not args.skip_cpu:
        # one step of the whole config through the stock reference on all host
        # cores (~15-30 s of CPU work), same bytes accounting (f32 input)
        ref = ReferenceCPU(H, D, T)
        try:
            sec = ref.step(L)
        finally:
            ref.close()
        cbb, dbb = algorithmic_bytes(L, H, D, T, 4, 2)
        cpu = {"value": (cbb + dbb) / sec / 1e9, "unit": "GB/s", "cores": ref.procs, "kind": ref.kind,
               "sample": f"all {L} layers [1,{H},{T},{D}] f32, one step: stock kvpool build_pool + "
                         f"attach(16).get_kv_for_layer per layer, {ref.procs} processes",
               **cpu_info()}

    if rank == 0:
        dtn = "f32" if main_dt == torch.float32 else "bf16"
        par = ("1 GPU: the whole pool" if world == 1 else
               f"layer-sharded build ({rows_max} layers/GPU) + one NCCL all-gather of the packed pool "
               f"(replicated on every GPU) + materialise of each GPU's layers; decode agents partitioned "
               f"{[len(parallel.partition_agents(agents, world, x)) for x in range(world)]}")
        line = {
            **({"plumbing_test": "gloo backend, ranks share GPUs: a code-path check, not a measurement"}
               if plumbing else {}),
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": f"{dtn} in / u8+int8 pool / bf16 out",
            "data": "synthetic (torch.randn, var 1/head_dim, random-init)",
            "config": {"workload": desc, "layers": L, "kv_heads": H, "head_dim": D, "seq_len": T,
                       "agents": agents, "k_scale_mode": args.k_mode, "input_dtype": dtn,
                       "step": "build_pool (pkv_encode) + inject to bf16 (pkv_decode) of every layer; "
                               "at N>1 + the pool all-gather",
                       "l2": "inputs larger than L2 (no flush needed)", "parallelism": par},
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": peak,
                         "algorithmic_bytes": dom_bytes, "kernel_ms": dom_ms, "peak_kind": peak_kind,
                         "unit": "GB/s", "frac": achieved / peak, "traffic": traffic},
            "kernels": kernel_block(r, dtn),
            "variant": kernel_block(variant, "bf16" if dtn == "f32" else "f32") if variant else None,
            "k_mode_variant": ({"k_scale_mode": other_km, "step_ms": kvariant["ms_step"],
                                "value_gbs": kvariant["value"], "encode_ms": kvariant["encode_ms"],
                                "decode_ms": kvariant["decode_ms"]} if kvariant else None),
            # per step: encode + decode (+ the all-gather at N>1; + one workspace memset)
            "gpu_launches": (2 + (1 if world > 1 else 0)) * args.steps,
            "clocks": r["clocks"],
            "e2e": e2e,
            "decode_attention": attn,
            "decode_e2e": dec_e2e,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def print_plan(args, cfg) -> int:
    """The sharding plan every rank computes, gathered to rank 0 over gloo
    (exercises the self-launch, rendezvous and partitioning without a GPU)."""
    import torch.distributed as dist

    from paper_2604_24971_b200 import parallel

    L, H, D, T, agents, group, desc = cfg
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    if world != args.gpus:
        raise SystemExit(f"bench.py: --gpus {args.gpus} but WORLD_SIZE={world}")
    mine = {"rank": rank, "layers": list(parallel.layer_shard(L, world, rank)),
            "agents": parallel.partition_agents(agents, world, rank)}
    plans = [mine]
    if world > 1:
        dist.init_process_group("gloo")
        plans = [None] * world
        dist.all_gather_object(plans, mine)
        dist.destroy_process_group()
    if rank == 0:
        print(json.dumps({"config": args.config, "world": world, "plan": plans}), flush=True)
    return 0


def launch_ranks(args) -> int:
    """`--gpus N` without torchrun: re-run this script as N ranks (one process
    per GPU) through torch.distributed.run on 127.0.0.1, NCCL_DEBUG=INFO."""
    import socket

    with socket.socket() as s_:
        s_.bind(("127.0.0.1", 0))
        port = s_.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={args.gpus}",
           "--master-addr", "127.0.0.1", f"--master-port={port}", str(Path(__file__).resolve()), *sys.argv[1:]]
    env = dict(os.environ)
    env.setdefault("NCCL_DEBUG", "INFO")
    env.setdefault("NCCL_DEBUG_SUBSYS", "INIT")
    return subprocess.call(cmd, env=env)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--dtype", default="f32", choices=["bf16", "f32"],
                    help="input dtype of the headline (f32: the reference's dtype, SURVEY 8(d)); "
                         "the other one is measured as the variant")
    ap.add_argument("--k-mode", default="tensor", choices=["tensor", "block32"])
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-attention", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of CUDA graphs")
    ap.add_argument("--skip-decode-e2e", action="store_true", help="skip the model-level decode measurement")
    ap.add_argument("--skip-variant", action="store_true", help="skip the other input dtype's measurement")
    ap.add_argument("--dist-backend", default="nccl", choices=["nccl", "gloo"],
                    help="gloo: run the N>1 path with ranks sharing the visible GPUs (plumbing check only)")
    ap.add_argument("--plan-only", action="store_true",
                    help="print each rank's layer / agent shard (gloo; no GPU work) and exit")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.gpus > 1 and "WORLD_SIZE" not in os.environ:
        return launch_ranks(args)
    if args.plan_only:
        return print_plan(args, cfg)
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
