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
    import torch
    import torch.distributed as dist

    import paper_2604_24971_b200 as pk
    from paper_2604_24971_b200 import _codec
    from paper_2604_24971_b200.attention import decode_attention
    from paper_2604_24971_b200.pool import _Arena, _encode_layers, raise_for_status

    L, H, D, T, agents, group, desc = cfg
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    dtype = torch.bfloat16 if args.dtype == "bf16" else torch.float32
    in_b = 2 if dtype == torch.bfloat16 else 4
    g = pk.ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T)
    dump = pk.synth_gaussian_dump(g, seed=rank, device=dev, dtype=dtype, generator="torch")
    ks = [k for k, _ in dump.layers]
    vs = [v for _, v in dump.layers]
    arena = _Arena(g, L, args.k_mode, dev)
    kb, vb, _ = _encode_layers(ks, vs, g, pk.GAUSSIAN_3BIT, None, args.k_mode, device=dev, arena=arena)
    pool = pk.SharedPool(g, list(zip(kb, vb))).seal()
    out_k = [torch.empty(g.tensor_shape, dtype=torch.bfloat16, device=dev) for _ in range(L)]
    out_v = [torch.empty(g.tensor_shape, dtype=torch.bfloat16, device=dev) for _ in range(L)]
    stream = torch.cuda.current_stream(dev)

    def encode():
        _encode_layers(ks, vs, g, pk.GAUSSIAN_3BIT, None, args.k_mode, device=dev, arena=arena, check=False)

    def decode():
        _codec.decode(num_vectors=g.vectors_per_tensor, head_dim=D, out_dtype=torch.bfloat16,
                      k_mode=pk.keyquant.K_MODES[args.k_mode], k_codes=pool.k_codes, k_scale=pool.k_scale,
                      k_bscale=pool.k_bscale, v_packed=pool.v_packed, v_scales=pool.v_scales,
                      centroids=pk.GAUSSIAN_3BIT.centroids, sign_seed=None, k_out=out_k, v_out=out_v,
                      device=dev)

    ev = lambda: torch.cuda.Event(enable_timing=True)  # noqa: E731
    none = [None] * L

    def encode_k():
        _encode_layers(ks, none, g, pk.GAUSSIAN_3BIT, None, args.k_mode, device=dev, arena=arena, check=False)

    def encode_v():
        _encode_layers(none, vs, g, pk.GAUSSIAN_3BIT, None, args.k_mode, device=dev, arena=arena, check=False)

    def capture(fn):
        """CUDA-graph a launch sequence so the timed loop measures the GPU, not
        the Python/ctypes enqueue path; None if capture is unavailable."""
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
            print(f"[bench] graph capture unavailable ({exc}); timing eager launches", file=sys.stderr)
            return None

    for _ in range(args.warmup):
        encode()
        decode()
    raise_for_status(arena.status)
    torch.cuda.synchronize(dev)
    run_enc = capture(encode) or encode
    run_dec = capture(decode) or decode
    run_enc_k = capture(encode_k) or encode_k
    run_enc_v = capture(encode_v) or encode_v
    graphed = not args.no_graph and run_enc is not encode
    for _ in range(args.warmup):
        run_enc()
        run_dec()
    torch.cuda.synchronize(dev)
    if world > 1:
        dist.barrier()
    marks = [(ev(), ev(), ev()) for _ in range(args.steps)]
    start, end = ev(), ev()
    with ClockSampler(local) as clocks:
        torch.cuda.synchronize(dev)
        start.record(stream)
        for a_, b_, c_ in marks:
            a_.record(stream)
            run_enc()
            b_.record(stream)
            run_dec()
            c_.record(stream)
        end.record(stream)
        torch.cuda.synchronize(dev)
    total_ms = start.elapsed_time(end)
    enc_ms = sum(a_.elapsed_time(b_) for a_, b_, _ in marks) / args.steps
    dec_ms = sum(b_.elapsed_time(c_) for _, b_, c_ in marks) / args.steps

    def time_it(fn, n):
        s_, e_ = ev(), ev()
        fn()
        torch.cuda.synchronize(dev)
        s_.record(stream)
        for _ in range(n):
            fn()
        e_.record(stream)
        torch.cuda.synchronize(dev)
        return s_.elapsed_time(e_) / n

    enc_k_ms = time_it(run_enc_k, args.steps)
    enc_v_ms = time_it(run_enc_v, args.steps)
    def max_over_ranks(ms):
        if world == 1:
            return ms
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        return float(t.item())

    total_ms = max_over_ranks(total_ms)
    ms_step = total_ms / args.steps
    comp_b, deq_b = algorithmic_bytes(L, H, D, T, in_b, 2, args.k_mode)
    value = world * (comp_b + deq_b) / (ms_step / 1e3) / 1e9

    # ---- e2e through the public API with host buffers ----
    e2e = None
    if not args.skip_e2e:
        host_layers = [(k.values.cpu().pin_memory(), v.values.cpu().pin_memory()) for k, v in dump.layers]
        host_dump = pk.KvDump(g, tuple((pk.KvTensor(g, k), pk.KvTensor(g, v)) for k, v in host_layers))
        host_out = [(torch.empty(g.tensor_shape, dtype=torch.bfloat16).pin_memory(),
                     torch.empty(g.tensor_shape, dtype=torch.bfloat16).pin_memory()) for _ in range(L)]

        inflight = []

        def e2e_step():
            # build_pool uploads the pinned dump chunk by chunk, overlapped with
            # the encode; materialize_to_host overlaps decode with the D2H copies.
            # The host may run one step ahead (step n+1 uploads while step n
            # downloads) but no further: unbounded run-ahead makes the caching
            # allocator grow (cudaMalloc stalls the host for 100s of ms).
            p = pk.build_pool(host_dump, build_stats=False, device=dev, check=False)
            p.attach(16).materialize_to_host(host_out)
            done = torch.cuda.Event()
            done.record(stream)
            inflight.append(done)
            if len(inflight) > 1:
                inflight.pop(0).synchronize()

        # warm the caching allocator (each step allocates a fresh pool and
        # staging buffers; the first steps pay cudaMalloc) before timing
        for _ in range(max(3, args.warmup)):
            e2e_step()
        torch.cuda.synchronize(dev)
        es, ee = ev(), ev()
        n_e2e = max(3, min(args.steps, 20))
        if world > 1:
            dist.barrier()
        es.record(stream)
        for _ in range(n_e2e):
            e2e_step()
        ee.record(stream)
        torch.cuda.synchronize(dev)
        e2e_ms = max_over_ranks(es.elapsed_time(ee) / n_e2e)
        h2d = 2 * L * g.elements_per_tensor * in_b
        d2h = 2 * L * g.elements_per_tensor * 2
        e2e = {"value": world * (comp_b + deq_b) / (e2e_ms / 1e3) / 1e9, "unit": "GB/s",
               "h2d_bytes_per_step": h2d, "d2h_bytes_per_step": d2h, "ms_per_step": e2e_ms}

    # ---- shared-pool decode attention (all agents, all layers) ----
    attn = None
    if not args.skip_attention and D in (64, 128):
        q = torch.randn(agents, H, group, D, device=dev, dtype=torch.bfloat16)
        outa = torch.empty_like(q)
        need = pk._lib.load().pkv_attention_workspace_bytes(agents, H, group, D, T)
        ws = torch.empty((need + 3) // 4, dtype=torch.float32, device=dev)

        def attn_step():
            for li in range(L):
                decode_attention(pool, li, q, softmax_scale=D ** -0.5, out=outa, workspace=ws)

        for _ in range(2):
            attn_step()
        torch.cuda.synchronize(dev)
        s2, e2 = ev(), ev()
        if world > 1:
            dist.barrier()
        s2.record(stream)
        for _ in range(args.steps):
            attn_step()
        e2.record(stream)
        torch.cuda.synchronize(dev)
        a_ms = max_over_ranks(s2.elapsed_time(e2) / args.steps)
        pool_bytes = L * (g.elements_per_tensor * (1 + 3 / 8) + 4 * g.vectors_per_tensor + 4)
        attn = {"tokens_per_s": world * agents / (a_ms / 1e3), "ms_per_token_step": a_ms,
                "agents": agents, "layers": L, "scope": "attention only (all layers), batched agents",
                "pool_gbs": pool_bytes / (a_ms / 1e3) / 1e9}

    # ---- model-level shared-pool decode (random-init model of the config's shape) ----
    dec_e2e = None
    if not args.skip_decode_e2e and args.config in ("c2", "c3") and rank == 0:
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
    n = g.elements_per_tensor
    vecs = g.vectors_per_tensor
    kb = 4 if args.k_mode == "tensor" else 2 * ((n + 31) // 32)
    bytes_k = L * (n * in_b + n + kb)                      # key encode (absmax pass + codes)
    bytes_v = L * (n * in_b + 3 * n / 8 + 4 * vecs)        # value encode
    # the step's two launches: the fused encode (value + key roles) and the decode
    kernels = {"encode": (enc_ms, comp_b), "decode": (dec_ms, deq_b)}
    dom_name = max(kernels, key=lambda k: kernels[k][0])
    dom_ms, dom_bytes = kernels[dom_name]
    achieved = dom_bytes / (dom_ms / 1e3) / 1e9
    prof = ROOT / "profiles" / "traffic.json"
    traffic = None
    if prof.exists():
        try:
            traffic = json.loads(prof.read_text()).get(f"{args.config}/{args.dtype}/{dom_name}")
        except Exception:
            traffic = None

    cpu = None
    if rank == 0 and not args.skip_cpu:
        # one step of the whole config through the stock reference on all host
        # cores (~15-30 s of CPU work), same bytes accounting (f32 input)
        ref = ReferenceCPU(H, D, T)
        try:
            sec = ref.step(L)
        finally:
            ref.close()
        cb, dbb = algorithmic_bytes(L, H, D, T, 4, 2)
        cpu = {"value": (cb + dbb) / sec / 1e9, "unit": "GB/s", "cores": ref.procs, "kind": ref.kind,
               "sample": f"all {L} layers [1,{H},{T},{D}] f32, one step: stock kvpool build_pool + "
                         f"attach(16).get_kv_for_layer per layer, {ref.procs} processes",
               **cpu_info()}

    if rank == 0:
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
            "vs_baseline": None, "dtype": "bf16 in / u8+int8 pool / bf16 out" if in_b == 2 else "f32 in / u8+int8 pool / bf16 out",
            "data": "synthetic (torch.randn, var 1/head_dim, random-init)",
            "config": {"workload": desc, "layers": L, "kv_heads": H, "head_dim": D, "seq_len": T,
                       "agents": agents, "k_scale_mode": args.k_mode,
                       "step": "build_pool (pkv_encode, all layers) + inject_all to bf16 (pkv_decode, all layers)",
                       "l2": "inputs larger than L2 (no flush needed)",
                       "parallelism": f"replica x{world} (independent pools per GPU)"},
            "roofline": {"bound": "hbm", "kernel": dom_name, "achieved": achieved, "peak": peak,
                         "algorithmic_bytes": dom_bytes, "kernel_ms": dom_ms,
                         "peak_kind": peak_kind, "unit": "GB/s", "frac": achieved / peak, "traffic": traffic},
            "kernels": {"encode_ms": enc_ms, "encode_gbs": comp_b / (enc_ms / 1e3) / 1e9,
                        "decode_ms": dec_ms, "decode_gbs": deq_b / (dec_ms / 1e3) / 1e9,
                        "encode_values_ms": enc_v_ms, "encode_values_gbs": bytes_v / (enc_v_ms / 1e3) / 1e9,
                        "encode_keys_ms": enc_k_ms, "encode_keys_gbs": bytes_k / (enc_k_ms / 1e3) / 1e9,
                        "encode_bytes": comp_b, "decode_bytes": deq_b, "cuda_graph": graphed},
            # per step: one encode launch (value + key roles) and one decode launch (+ one memset)
            "gpu_launches": 2 * args.steps,
            "clocks": clocks.summary(),
            "e2e": e2e,
            "decode_attention": attn,
            "decode_e2e": dec_e2e,
            "replayed_vectors_per_build": pool.replay_count,
            "cpu_baseline": cpu,
        }
        print(json.dumps(line), flush=True)
    if world > 1:
        dist.destroy_process_group()
    return 0


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=400)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--config", default="c3", choices=sorted(CONFIGS))
    ap.add_argument("--dtype", default="bf16", choices=["bf16", "f32"])
    ap.add_argument("--k-mode", default="tensor", choices=["tensor", "block32"])
    ap.add_argument("--skip-e2e", action="store_true")
    ap.add_argument("--skip-attention", action="store_true")
    ap.add_argument("--skip-cpu", action="store_true")
    ap.add_argument("--no-graph", action="store_true", help="time eager launches instead of CUDA graphs")
    ap.add_argument("--skip-decode-e2e", action="store_true", help="skip the model-level decode measurement")
    args = ap.parse_args()
    if args.warmup < 3:
        args.warmup = 3
    cfg = CONFIGS[args.config]
    if args.impl == "reference":
        return run_reference(args, cfg)
    return run_ours(args, cfg)


if __name__ == "__main__":
    sys.exit(main())
