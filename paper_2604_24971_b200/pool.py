"""Write-once shared pool of compressed KV layers in HBM, read by many agents.

API-compatible with kvpool.pool (/root/reference/pkg/src/kvpool/pool.py):
build_pool -> sealed SharedPool -> attach(decode_bits) -> AgentCacheView
.get_kv_for_layer / .inject_all, plus PKVP v1 snapshots.

B200 layout: one allocation per field for all layers (so every kernel
launch covers the whole pool through per-layer pointer tables):
    k_codes  int8   [L, pad16(n)]           q8_0 codes
    k_scale  f32    [L]        (tensor)     or  k_bscale f16 [L, pad8(n/32)]
    v_packed uint8  [L, pad16(3*ceil(n/8))] 3-bit codes, PKVP packed layout
    v_scales f32    [L, B*H*T]              per-vector RMS
n = B*H*T*D. Pool bytes are independent of the number of attached agents.
"""

from __future__ import annotations

import struct
import threading
from dataclasses import dataclass
from pathlib import Path

import numpy as np
import torch

from . import _codec
from ._lib import (
    PKV_FLAG_BAD_CODE,
    PKV_FLAG_K_NONFINITE,
    PKV_FLAG_K_SCALE_OVERFLOW,
    PKV_FLAG_V_NONFINITE,
)
from .errors import (
    BadMagicError,
    CorruptBlockError,
    GeometryError,
    KvPoolError,
    PayloadSizeError,
    TruncatedFileError,
    UnsealedPoolError,
    UnsupportedVersionError,
)
from .keyquant import K_MODES, QuantizedKeyBlock, block32_count
from .model import KvDump, KvTensor, ModelGeometry
from .valuequant import GAUSSIAN_3BIT, Codebook, QuantizedValueBlock, _require_3bit, packed_nbytes

PKVP_MAGIC = b"PKVP"
PKVP_VERSION = 1
FLAG_PACKED_VALUES = 0x0001
FLAG_SIGN_DIAGONAL = 0x0002
_POOL_HEADER = struct.Struct("<4sHHIIIIIHQ6x")  # pool.py:62-63
POOL_HEADER_SIZE = _POOL_HEADER.size  # 44


def _pad(x: int, m: int) -> int:
    return (x + m - 1) // m * m


def round_to_bfloat16(values):
    """RNE to bf16 precision, returned as f32 (pool.py:66-76).

    numpy in -> numpy out (host utility); torch in -> torch (device cast,
    bit-identical to the reference's integer rounding).
    """
    if isinstance(values, torch.Tensor):
        return values.to(torch.bfloat16).to(torch.float32)
    u = np.ascontiguousarray(values, dtype=np.float32).view(np.uint32)
    r = (u + np.uint32(0x7FFF) + ((u >> np.uint32(16)) & np.uint32(1))) & np.uint32(0xFFFF0000)
    return r.view(np.float32)


@dataclass(frozen=True)
class LayerStats:
    """Quantization error of one layer at 32-bit decode (pool.py:79-88)."""

    layer: int
    k_scale: float
    k_mse: float
    k_max_err: float
    v_mse: float
    v_nmse: float


@dataclass(frozen=True)
class TranscriptEntry:
    layer: int
    k_checksum: int
    v_checksum: int
    k_elements: int
    v_elements: int


@dataclass(frozen=True)
class InjectionTranscript:
    """Ordered record of one agent handing every layer to its serving stack."""

    agent_id: int
    decode_bits: int
    entries: tuple

    def __post_init__(self):
        object.__setattr__(self, "entries", tuple(self.entries))
        layers = [e.layer for e in self.entries]
        if layers != list(range(len(layers))):
            raise ValueError(f"transcript layers must be 0..L-1 in order, got {layers}")

    @property
    def total_elements(self) -> int:
        return sum(e.k_elements + e.v_elements for e in self.entries)

    def checksums(self) -> tuple:
        return tuple((e.k_checksum, e.v_checksum) for e in self.entries)


# ---------------------------------------------------------------------------
# encode (shared by quantize_k / quantize_v / build_pool)
# ---------------------------------------------------------------------------

class _Arena:
    """Device storage for L layers of one pool, layer-major.

    ONE uint8 allocation `flat` [L, layer_bytes]; each layer row holds that
    layer's fields back to back, every section 256-byte aligned (TMA needs 16):
        k_codes int8 [pad16(n)] | v_packed u8 [pad16(3 ceil(n/8))] |
        v_scales f32 [pad4(vecs)] | k_bscale f16 [pad8(n/32)] (block32) |
        k_scale f32 (tensor) | status i32 (gather copy)
    The per-field attributes are strided [L, ...] views into `flat` (kernels
    take per-layer pointers, so the row stride is invisible to them). A
    layer-sharded pool is therefore ONE contiguous block per rank and the
    multi-GPU assembly is ONE all_gather_into_tensor (parallel.gather_arena).
    `status` (the per-launch contiguous status words the encoder ORs into)
    and `replay` are small separate tensors.
    """

    ALIGN = 256

    def __init__(self, g: ModelGeometry, L: int, k_mode: str, device, with_k=True, with_v=True):
        n, vecs = g.elements_per_tensor, g.vectors_per_tensor
        secs = []
        if with_k:
            secs.append(("k_codes", _pad(n, 16), torch.int8))
        if with_v:
            secs.append(("v_packed", _pad(packed_nbytes(n), 16), torch.uint8))
            # rows padded to 4 floats so every layer's scales start 16-byte aligned (TMA)
            secs.append(("v_scales", 4 * _pad(vecs, 4), torch.float32))
        if with_k and k_mode == "block32":
            secs.append(("k_bscale", 2 * _pad(block32_count(n), 8), torch.float16))
        if with_k and k_mode == "tensor":
            secs.append(("k_scale", 16, torch.float32))
        secs.append(("status_row", 16, torch.int32))
        offs, off = {}, 0
        for name, nbytes, _ in secs:
            offs[name] = off
            off = _pad(off + nbytes, self.ALIGN)
        self.layer_bytes = off
        self.num_layers = L
        self.k_mode = k_mode
        self.flat = torch.empty((L, off), dtype=torch.uint8, device=device)
        self._sections = [(name, offs[name], nbytes, dt) for name, nbytes, dt in secs]
        self._bind()
        if self.k_scale is not None:
            self.k_scale.zero_()
        self.status = torch.zeros(L, dtype=torch.int32, device=device)
        self.replay = torch.zeros(1, dtype=torch.int32, device=device)

    def _bind(self):
        for name in ("k_codes", "v_packed", "v_scales", "k_bscale", "k_scale", "status_row"):
            setattr(self, name, None)
        for name, off, nbytes, dt in self._sections:
            v = self.flat[:, off:off + nbytes].view(dt)
            if name in ("k_scale", "status_row"):
                v = v[:, 0]
            setattr(self, name, v)

    @classmethod
    def like(cls, other: "_Arena", flat: torch.Tensor) -> "_Arena":
        """An arena with `other`'s layout around a given [L', layer_bytes] buffer
        (e.g. the all-gathered pool)."""
        a = object.__new__(cls)
        a.layer_bytes, a.k_mode, a._sections = other.layer_bytes, other.k_mode, other._sections
        a.num_layers = flat.shape[0]
        a.flat = flat
        a._bind()
        a.status = a.status_row.contiguous()
        a.replay = torch.zeros(1, dtype=torch.int32, device=flat.device)
        return a

    def nbytes(self) -> int:
        return self.flat.numel() + 4 * self.status.numel()


def _device_inputs(tensors, device):
    out = []
    for t in tensors:
        v = t.values
        if v.device != device:
            v = v.to(device, non_blocking=True)
        out.append(v.contiguous())
    return out


def raise_for_status(status: torch.Tensor) -> None:
    """Map device status bits to the reference's exceptions (one sync)."""
    flags = status.cpu().numpy()
    bad = np.bitwise_or.reduce(flags) if flags.size else 0
    if bad & (PKV_FLAG_K_NONFINITE | PKV_FLAG_V_NONFINITE):
        layer = int(np.flatnonzero(flags & (PKV_FLAG_K_NONFINITE | PKV_FLAG_V_NONFINITE))[0])
        raise GeometryError(f"tensor contains NaN or Inf (layer {layer})")
    if bad & PKV_FLAG_K_SCALE_OVERFLOW:
        raise KvPoolError("a block32 key scale overflows float16 (|K| > 8.3e6)")
    if bad & PKV_FLAG_BAD_CODE:
        raise CorruptBlockError("corrupt block: code out of range for 3-bit codebook")


def _rows(t: torch.Tensor, idx: list) -> torch.Tensor:
    """t[idx] without a host index tensor when idx is a contiguous range (so the
    call stays CUDA-graph capturable)."""
    if idx == list(range(idx[0], idx[0] + len(idx))):
        return t[idx[0]:idx[0] + len(idx)].contiguous()
    return t[torch.tensor(idx, device=t.device)].contiguous()


def _encode_layers(ks, vs, geometry: ModelGeometry, codebook: Codebook | None, sign_seed,
                   k_scale_mode: str, *, device=None, check: bool = True, arena: _Arena | None = None,
                   k_layer_max: torch.Tensor | None = None):
    """Encode parallel lists of K / V KvTensors (entries may be None) with one
    pkv_encode launch per input dtype. Returns (key blocks, value blocks, arena).
    k_layer_max: optional int32 [L] device tensor of per-layer max|K| bit
    patterns (head-sharded pools) replacing the encoder's own absmax pass."""
    if k_scale_mode not in K_MODES:
        raise ValueError(f"k_scale_mode must be one of {tuple(K_MODES)}, got {k_scale_mode!r}")
    ref = next(t for t in list(ks) + list(vs) if t is not None)
    if device is None:
        device = ref.values.device if ref.values.is_cuda else None
    device = _codec.require_device(device)
    L = len(ks)
    with_k = any(k is not None for k in ks)
    with_v = any(v is not None for v in vs)
    if with_v:
        _require_3bit(codebook)
    g = geometry
    a = arena or _Arena(g, L, k_scale_mode, device, with_k, with_v)
    n = g.elements_per_tensor
    kidx = [i for i, k in enumerate(ks) if k is not None]
    vidx = [i for i, v in enumerate(vs) if v is not None]
    kin = dict(zip(kidx, _device_inputs([ks[i] for i in kidx], device)))
    vin = dict(zip(vidx, _device_inputs([vs[i] for i in vidx], device)))
    # one launch per (dtype) group; K and V of a layer share a launch when possible
    dtypes = {t.dtype for t in list(kin.values()) + list(vin.values())}
    for dt in sorted(dtypes, key=str):
        kl = [i for i in kidx if kin[i].dtype == dt]
        vl = [i for i in vidx if vin[i].dtype == dt]
        if kl == vl and kl:
            groups = [(kl, vl)]
        else:
            groups = [(kl, []), ([], vl)]
        for kg, vg in groups:
            if not kg and not vg:
                continue
            layers = kg or vg
            if kg and vg and kg != vg:
                raise AssertionError
            st = a.status[layers[0]:layers[0] + 1] if len(layers) == 1 else None
            # status words must be contiguous per launch: use a scratch when scattered
            contiguous = layers == list(range(layers[0], layers[0] + len(layers)))
            status = a.status[layers[0]:layers[0] + len(layers)] if contiguous else \
                torch.zeros(len(layers), dtype=torch.int32, device=device)
            _codec.encode(
                num_vectors=g.vectors_per_tensor, head_dim=g.head_dim,
                k_in=[kin[i] for i in kg] if kg else None,
                v_in=[vin[i] for i in vg] if vg else None,
                k_mode=K_MODES[k_scale_mode],
                k_codes=[a.k_codes[i] for i in kg] if kg else None,
                k_scale=[a.k_scale[i:i + 1] for i in kg] if (kg and k_scale_mode == "tensor") else None,
                k_bscale=[a.k_bscale[i] for i in kg] if (kg and k_scale_mode == "block32") else None,
                v_packed=[a.v_packed[i] for i in vg] if vg else None,
                v_scales=[a.v_scales[i, :g.vectors_per_tensor] for i in vg] if vg else None,
                centroids=(codebook.centroids if codebook is not None else np.zeros(8)),
                sign_seed=sign_seed, status=status, replay=a.replay, device=device,
                k_layer_max=(_rows(k_layer_max, kg) if (k_layer_max is not None and kg
                                                         and k_scale_mode == "tensor") else None))
            if not contiguous:
                for j, i in enumerate(layers):
                    a.status[i] |= status[j]
            del st
    if check:
        raise_for_status(a.status)
    kblocks, vblocks = _blocks_from_arena(a, g, codebook, sign_seed, k_scale_mode,
                                          [k is not None for k in ks], [v is not None for v in vs])
    return kblocks, vblocks, a


def _blocks_from_arena(a: "_Arena", g: ModelGeometry, codebook, sign_seed, k_scale_mode: str, has_k, has_v):
    """Per-layer key/value blocks viewing an arena's rows (no copies)."""
    n = g.elements_per_tensor
    kblocks, vblocks = [], []
    nb = block32_count(n)
    for i in range(len(has_k)):
        if has_k[i]:
            kblocks.append(QuantizedKeyBlock(
                g, a.k_scale[i:i + 1] if k_scale_mode == "tensor" else 0.0,
                a.k_codes[i, :n].view(g.tensor_shape), mode=k_scale_mode,
                block_scales=a.k_bscale[i, :nb] if k_scale_mode == "block32" else None,
                _trusted=True))
        else:
            kblocks.append(None)
        if has_v[i]:
            vblocks.append(QuantizedValueBlock(
                g, codebook.name, codebook.bits, None, a.v_scales[i, :g.vectors_per_tensor].view(g.tensor_shape[:-1]),
                sign_seed, packed=a.v_packed[i, :packed_nbytes(n)], _trusted=True))
        else:
            vblocks.append(None)
    return kblocks, vblocks


def pool_from_arena(a: "_Arena", g: ModelGeometry, codebook: Codebook = GAUSSIAN_3BIT, sign_seed=None,
                    k_scale_mode: str = "tensor") -> "SharedPool":
    """Seal a pool around a fully populated arena (e.g. one gathered from other GPUs)."""
    L = g.num_layers
    kb, vb = _blocks_from_arena(a, g, codebook, sign_seed, k_scale_mode, [True] * L, [True] * L)
    pool = SharedPool(g, list(zip(kb, vb)), (), codebook=codebook, sign_seed=sign_seed)
    pool._arena = a
    pool._replay = a.replay
    pool.status = a.status
    return pool.seal()


# ---------------------------------------------------------------------------
# pool
# ---------------------------------------------------------------------------

class SharedPool:
    """Compressed KV layers shared by every agent serving the same prefix (pool.py:128-214)."""

    def __init__(self, geometry: ModelGeometry, layers, build_stats=(), codebook: Codebook = GAUSSIAN_3BIT,
                 sign_seed: int | None = None):
        layers = [tuple(p) for p in layers]
        if len(layers) != geometry.num_layers:
            raise GeometryError(f"pool has {len(layers)} layers, geometry says {geometry.num_layers}")
        modes = set()
        for i, (kq, vq) in enumerate(layers):
            if kq.geometry != geometry or vq.geometry != geometry:
                raise GeometryError(f"layer {i} block does not match pool geometry")
            if vq.codebook_name != codebook.name or vq.sign_seed != sign_seed:
                raise GeometryError(f"layer {i} value block coded with different settings")
            modes.add(kq.mode)
        if len(modes) != 1:
            raise GeometryError("all key blocks of a pool must share one k_scale_mode")
        self.geometry = geometry
        self.codebook = codebook
        self.sign_seed = sign_seed
        self.k_scale_mode = modes.pop()
        self._layers = tuple(layers)
        self._build_stats = tuple(build_stats)
        self._stats_source: KvDump | None = None
        self._sealed = False
        self._attach_lock = threading.Lock()
        self._num_agents = 0
        self._replay: torch.Tensor | None = None
        self._arena: _Arena | None = None
        self.device = layers[0][0].device
        # per-layer device tensors for whole-pool launches
        self.k_codes = [kq.codes for kq, _ in layers]
        self.k_scale = [kq.scale_t for kq, _ in layers] if self.k_scale_mode == "tensor" else None
        self.k_bscale = [kq.block_scales for kq, _ in layers] if self.k_scale_mode == "block32" else None
        self.v_packed = [vq.packed for _, vq in layers]
        self.v_scales = [vq.scales for _, vq in layers]

    @property
    def sealed(self) -> bool:
        return self._sealed

    @property
    def num_layers(self) -> int:
        return self.geometry.num_layers

    @property
    def num_agents(self) -> int:
        return self._num_agents

    @property
    def build_stats(self) -> tuple:
        """Per-layer LayerStats; computed on the GPU on first access when the
        pool was built with build_stats='lazy' (the default)."""
        if not self._build_stats and self._stats_source is not None:
            self._build_stats = compute_layer_stats(self._stats_source, self)
            self._stats_source = None
        return self._build_stats

    @property
    def replay_count(self) -> int:
        """Head vectors re-coded on the exact fp64 path (threshold ties) at build."""
        return 0 if self._replay is None else int(self._replay.item())

    def seal(self) -> "SharedPool":
        self._sealed = True
        return self

    def layer_blocks(self, layer_idx: int):
        if not 0 <= layer_idx < len(self._layers):
            raise IndexError(f"layer {layer_idx} out of range for {len(self._layers)}-layer pool")
        return self._layers[layer_idx]

    def attach(self, decode_bits: int = 16) -> "AgentCacheView":
        if not self._sealed:
            raise UnsealedPoolError("cannot attach to an unsealed pool")
        if decode_bits not in (16, 32):
            raise ValueError(f"decode_bits must be 16 or 32, got {decode_bits!r}")
        with self._attach_lock:
            agent_id = self._num_agents
            self._num_agents += 1
        return AgentCacheView(self, agent_id, decode_bits)

    def payload_nbytes(self) -> int:
        """Canonical byte-per-code bytes (pool.py:197-202); independent of agents."""
        return sum(kq.payload_nbytes + vq.payload_nbytes for kq, vq in self._layers)

    def packed_payload_nbytes(self) -> int:
        """Bytes with values packed 8-per-3 (pool.py:204-208) — the HBM footprint."""
        return sum(kq.payload_nbytes + vq.packed_payload_nbytes for kq, vq in self._layers)

    def logical_payload_bits(self) -> int:
        e = self.geometry.elements_per_tensor
        return (8 * e + self._layers[0][1].bits * e) * self.geometry.num_layers

    def decode_layers(self, layers=None, dtype=torch.bfloat16, *, keys=True, values=True, out=None):
        """Materialise the given layers (default: all) in ONE kernel launch.

        Returns a list of (K, V) tensors [B,H,T,D] of `dtype` (bf16 == the
        reference's decode_bits=16 values; f32 == decode_bits=32). `out`: an
        optional list of preallocated (K, V) device tensors to decode into.
        """
        g = self.geometry
        idx = list(range(self.num_layers)) if layers is None else list(layers)
        for i in idx:
            self.layer_blocks(i)
        if not idx:
            return []
        if out is not None:
            ko = [k for k, _ in out] if keys else None
            vo = [v for _, v in out] if values else None
        else:
            ko = [torch.empty(g.tensor_shape, dtype=dtype, device=self.device) for _ in idx] if keys else None
            vo = [torch.empty(g.tensor_shape, dtype=dtype, device=self.device) for _ in idx] if values else None
        _codec.decode(
            num_vectors=g.vectors_per_tensor, head_dim=g.head_dim, out_dtype=dtype,
            k_mode=K_MODES[self.k_scale_mode],
            k_codes=[self.k_codes[i] for i in idx] if keys else None,
            k_scale=[self.k_scale[i] for i in idx] if (keys and self.k_scale) else None,
            k_bscale=[self.k_bscale[i] for i in idx] if (keys and self.k_bscale) else None,
            v_packed=[self.v_packed[i] for i in idx] if values else None,
            v_scales=[self.v_scales[i] for i in idx] if values else None,
            centroids=self.codebook.centroids, sign_seed=self.sign_seed,
            k_out=ko, v_out=vo, device=self.device)
        return [(ko[j] if keys else None, vo[j] if values else None) for j in range(len(idx))]

    def device_nbytes(self) -> int:
        """Bytes the pool actually occupies in HBM (packed codes, scales, padding)."""
        if self._arena is not None:
            return self._arena.nbytes()
        tensors = self.k_codes + self.v_packed + self.v_scales + (self.k_scale or []) + (self.k_bscale or [])
        return sum(t.numel() * t.element_size() for t in tensors)


class AgentCacheView:
    """One agent's read handle over a sealed pool (pool.py:217-255).

    Views hold no tensor state; every read decodes fresh device buffers.
    """

    def __init__(self, pool: SharedPool, agent_id: int, decode_bits: int):
        self.pool = pool
        self.agent_id = agent_id
        self.decode_bits = decode_bits

    @property
    def out_dtype(self) -> torch.dtype:
        return torch.bfloat16 if self.decode_bits == 16 else torch.float32

    def get_kv_for_layer(self, layer_idx: int):
        """Decompress one layer's (K, V) at this view's precision (one launch)."""
        g = self.pool.geometry
        (k, v), = self.pool.decode_layers([layer_idx], self.out_dtype)
        return KvTensor(g, k), KvTensor(g, v)

    def materialize_all(self):
        """All layers in one launch: list of (K, V) device tensors."""
        return self.pool.decode_layers(None, self.out_dtype)

    def materialize_to_host(self, host_layers, chunk: int = 4, layers=None) -> None:
        """Decode every layer (or the given `layers`) into caller-provided
        pinned host (K, V) tensors, one pair per decoded layer.

        Layers are decoded `chunk` at a time into two alternating device
        buffers; each chunk's device->host copy runs on a side stream while
        the next chunk decodes. Enqueued work only: the current stream waits
        for the last copy, so a sync of it covers everything.
        """
        pool, g, dt = self.pool, self.pool.geometry, self.out_dtype
        order = list(range(pool.num_layers)) if layers is None else list(layers)
        L = len(order)
        if len(host_layers) != L:
            raise ValueError(f"need {L} host (K, V) pairs, got {len(host_layers)}")
        comp = torch.cuda.current_stream(pool.device)
        copy = _side_stream(pool.device, "d2h")
        copy.wait_stream(comp)
        nb = min(chunk, L)
        bufs = [[(torch.empty(g.tensor_shape, dtype=dt, device=pool.device),
                  torch.empty(g.tensor_shape, dtype=dt, device=pool.device)) for _ in range(nb)] for _ in range(2)]
        copied = [None, None]
        for c, c0 in enumerate(range(0, L, chunk)):
            pos = list(range(c0, min(L, c0 + chunk)))
            idx = [order[j] for j in pos]
            buf = bufs[c % 2][:len(idx)]
            if copied[c % 2] is not None:
                comp.wait_event(copied[c % 2])  # the buffer's previous D2H has finished
            pool.decode_layers(idx, dt, out=buf)
            decoded = torch.cuda.Event()
            decoded.record(comp)
            copy.wait_event(decoded)
            with torch.cuda.stream(copy):
                for (hk, hv), (dk, dv) in zip((host_layers[j] for j in pos), buf):
                    hk.copy_(dk, non_blocking=True)
                    hv.copy_(dv, non_blocking=True)
                done = torch.cuda.Event()
                done.record(copy)
            copied[c % 2] = done
        comp.wait_stream(copy)
        for pair in bufs:
            for k, v in pair:
                k.record_stream(copy)
                v.record_stream(copy)

    def inject_all(self) -> InjectionTranscript:
        """Decode every layer and fingerprint what is handed over (pool.py:239-255).

        Checksums are FNV-1a over the f32 image of the decoded values, exactly
        the reference's tensor_checksum; hashing runs on the host.
        """
        layers = self.materialize_all()
        entries = []
        for idx, (k, v) in enumerate(layers):
            kh, vh = k.cpu(), v.cpu()
            entries.append(TranscriptEntry(
                layer=idx,
                k_checksum=_codec.fnv1a64_tensor_f32_image(kh),
                v_checksum=_codec.fnv1a64_tensor_f32_image(vh),
                k_elements=kh.numel(), v_elements=vh.numel()))
        return InjectionTranscript(agent_id=self.agent_id, decode_bits=self.decode_bits,
                                   entries=tuple(entries))


def build_pool(dump: KvDump, codebook: Codebook = GAUSSIAN_3BIT, sign_seed: int | None = None, *,
               k_scale_mode: str = "tensor", build_stats: str | bool = "lazy", device=None,
               check: bool = True, pipeline_chunk: int = 4) -> SharedPool:
    """Quantize every layer of a dump on the GPU in one launch and seal it (pool.py:258-293).

    build_stats: "lazy" (default) keeps a reference to the dump and computes
    LayerStats on first access of pool.build_stats; True computes them now;
    False skips them. check=False skips the post-build status sync (call
    raise_for_status(pool.status) later). A dump held in pinned host memory
    is uploaded `pipeline_chunk` layers at a time on a side stream, overlapped
    with the encoding of the previous chunk.
    """
    g = dump.geometry
    ks = [k for k, _ in dump.layers]
    vs = [v for _, v in dump.layers]
    if _pinned_host(ks + vs) and g.num_layers > pipeline_chunk:
        kb, vb, arena = _encode_from_host(ks, vs, g, codebook, sign_seed, k_scale_mode, device, check,
                                          pipeline_chunk)
    else:
        kb, vb, arena = _encode_layers(ks, vs, g, codebook, sign_seed, k_scale_mode, device=device, check=check)
    pool = SharedPool(g, list(zip(kb, vb)), (), codebook=codebook, sign_seed=sign_seed)
    pool._replay = arena.replay
    pool._arena = arena
    pool.status = arena.status
    if build_stats == "lazy":
        pool._stats_source = dump
    elif build_stats:
        pool._build_stats = compute_layer_stats(dump, pool)
    return pool.seal()


_SIDE_STREAMS: dict = {}


def _side_stream(device, role: str = "d2h") -> torch.cuda.Stream:
    """One upload ("h2d") and one download ("d2h") stream per device, so both
    PCIe directions run concurrently (e.g. pool n+1 uploading while pool n's
    decoded layers download)."""
    key = (torch.device(device).index, role)
    if key not in _SIDE_STREAMS:
        _SIDE_STREAMS[key] = torch.cuda.Stream(device)
    return _SIDE_STREAMS[key]


def _pinned_host(tensors) -> bool:
    return all(t is not None and t.values.device.type == "cpu" and t.values.is_pinned() for t in tensors)


def _encode_from_host(ks, vs, g: ModelGeometry, codebook, sign_seed, k_scale_mode, device, check, chunk):
    """Upload chunk c+1 (side stream) while chunk c encodes (current stream)."""
    dev = _codec.require_device(device)
    L = len(ks)
    arena = _Arena(g, L, k_scale_mode, dev)
    comp = torch.cuda.current_stream(dev)
    copy = _side_stream(dev, "h2d")  # host inputs need no device-side ordering
    for c0 in range(0, L, chunk):
        idx = range(c0, min(L, c0 + chunk))
        with torch.cuda.stream(copy):
            dk = [ks[i].values.to(dev, non_blocking=True) for i in idx]
            dv = [vs[i].values.to(dev, non_blocking=True) for i in idx]
            landed = torch.cuda.Event()
            landed.record(copy)
        comp.wait_event(landed)
        for t in dk + dv:
            t.record_stream(comp)
        kc, vc = [None] * L, [None] * L
        for j, i in enumerate(idx):
            kc[i] = KvTensor(g, dk[j])
            vc[i] = KvTensor(g, dv[j])
        _encode_layers(kc, vc, g, codebook, sign_seed, k_scale_mode, device=dev, check=False, arena=arena)
    if check:
        raise_for_status(arena.status)
    kb, vb = _blocks_from_arena(arena, g, codebook, sign_seed, k_scale_mode, [True] * L, [True] * L)
    return kb, vb, arena


def attach_agent(pool: SharedPool, decode_bits: int = 16) -> AgentCacheView:
    return pool.attach(decode_bits)


def compute_layer_stats(dump: KvDump, pool: SharedPool, chunk: int = 8) -> tuple:
    """LayerStats (pool.py:274-288): the f32 decode of the pool (pkv_decode,
    == the reference's 32-bit dequantize_k / dequantize_v) and one fused f64
    error reduction (pkv_layer_stats), `chunk` layers at a time."""
    from ._lib import check, load, ptr_array

    g = pool.geometry
    n = g.elements_per_tensor
    dev = pool.device
    L = pool.num_layers
    lib = load()
    sums = torch.empty((L, 4), dtype=torch.float64, device=dev)
    ws_bytes = lib.pkv_layer_stats_workspace_bytes(min(L, chunk), n)
    ws = torch.empty((ws_bytes + 7) // 8, dtype=torch.float64, device=dev)
    for c0 in range(0, L, chunk):
        idx = list(range(c0, min(L, c0 + chunk)))
        decoded = pool.decode_layers(idx, torch.float32)
        ks = _device_inputs([dump.layers[i][0] for i in idx], dev)
        vs = _device_inputs([dump.layers[i][1] for i in idx], dev)
        dt = {t.dtype for t in ks + vs}
        if len(dt) != 1 or dt.pop() not in (torch.float32, torch.bfloat16):
            ks = [t.float() for t in ks]
            vs = [t.float() for t in vs]
        with torch.cuda.device(dev):
            rc = lib.pkv_layer_stats(
                len(idx), n, _codec.dtype_code(ks[0]), ptr_array([t.data_ptr() for t in ks]),
                ptr_array([t.data_ptr() for t in vs]), ptr_array([k.data_ptr() for k, _ in decoded]),
                ptr_array([v.data_ptr() for _, v in decoded]), sums[c0].data_ptr(), ws.data_ptr(),
                ws.numel() * 8, _codec.stream_ptr(dev))
        check(rc, "pkv_layer_stats")
    host = sums.cpu().numpy()
    stats = []
    for idx in range(L):
        sk, kmax, sv, sp = (float(x) for x in host[idx])
        kq, _ = pool.layer_blocks(idx)
        v_mse = sv / n
        v_power = sp / n
        stats.append(LayerStats(layer=idx, k_scale=kq.scale, k_mse=sk / n, k_max_err=kmax, v_mse=v_mse,
                                v_nmse=v_mse / v_power if v_power > 0.0 else 0.0))
    return tuple(stats)


# ---------------------------------------------------------------------------
# PKVP v1 snapshots (pool.py:14-25, 301-432)
# ---------------------------------------------------------------------------

def save_pool(pool: SharedPool, path: str | Path, packed: bool = False) -> None:
    """Serialise a sealed pool to PKVP v1, bit-compatible with the reference.

    The device layout already is the packed payload, so packed snapshots are
    plain device->host copies.
    """
    if not pool.sealed:
        raise UnsealedPoolError("cannot snapshot an unsealed pool")
    if pool.codebook.name != GAUSSIAN_3BIT.name:
        raise ValueError(f"PKVP v1 stores only the canonical codebook, pool uses {pool.codebook.name!r}")
    if pool.k_scale_mode != "tensor":
        raise ValueError("PKVP v1 stores one key scale per layer; block32 pools cannot be saved")
    g = pool.geometry
    flags, seed = 0, 0
    if packed:
        flags |= FLAG_PACKED_VALUES
    if pool.sign_seed is not None:
        if not 0 <= pool.sign_seed < 1 << 64:
            raise ValueError(f"sign seed must fit in u64, got {pool.sign_seed}")
        flags |= FLAG_SIGN_DIAGONAL
        seed = pool.sign_seed
    header = _POOL_HEADER.pack(PKVP_MAGIC, PKVP_VERSION, flags, g.num_layers, g.batch, g.kv_heads,
                               g.seq_len, g.head_dim, g.baseline_bits, seed)
    with open(path, "wb") as f:
        f.write(header)
        for i in range(pool.num_layers):
            kq, vq = pool.layer_blocks(i)
            f.write(kq.scale_t.cpu().numpy().astype("<f4").tobytes())
            f.write(kq.codes.cpu().numpy().tobytes())
            f.write(vq.scales.cpu().numpy().astype("<f4").tobytes())
            if packed:
                f.write(vq.packed.cpu().numpy().tobytes())
            else:
                f.write(vq.codes.cpu().numpy().tobytes())


def load_pool(path: str | Path, device=None) -> SharedPool:
    """Parse a PKVP v1 snapshot into a sealed pool on the GPU (pool.py:348-432)."""
    data = Path(path).read_bytes()
    if len(data) < POOL_HEADER_SIZE:
        raise TruncatedFileError(f"file too short for header: {len(data)} < {POOL_HEADER_SIZE} bytes",
                                 offset=len(data))
    magic, version, flags, L, B, H, T, D, bits, seed = _POOL_HEADER.unpack_from(data, 0)
    if magic != PKVP_MAGIC:
        raise BadMagicError(f"bad magic {magic!r}, expected {PKVP_MAGIC!r}", offset=0)
    if version != PKVP_VERSION:
        raise UnsupportedVersionError(f"unsupported version {version}, expected {PKVP_VERSION}", offset=4)
    if flags & ~(FLAG_PACKED_VALUES | FLAG_SIGN_DIAGONAL):
        raise UnsupportedVersionError(f"unknown flags 0x{flags:04x}", offset=6)
    packed = bool(flags & FLAG_PACKED_VALUES)
    sign_seed = int(seed) if flags & FLAG_SIGN_DIAGONAL else None
    g = ModelGeometry(num_layers=L, kv_heads=H, head_dim=D, seq_len=T, batch=B, baseline_bits=bits)
    e, vecs = g.elements_per_tensor, g.vectors_per_tensor
    v_payload = packed_nbytes(e) if packed else e
    per_layer = 4 + e + 4 * vecs + v_payload
    expected = POOL_HEADER_SIZE + L * per_layer
    if len(data) < expected:
        raise TruncatedFileError(f"payload truncated: expected {expected} bytes total, got {len(data)}",
                                 offset=len(data))
    if len(data) > expected:
        raise PayloadSizeError(f"{len(data) - expected} trailing bytes after payload", offset=expected)
    dev = _codec.require_device(device)
    layers = []
    off = POOL_HEADER_SIZE
    for _ in range(L):
        (k_scale,) = struct.unpack_from("<f", data, off)
        off += 4
        k_codes = np.frombuffer(data, dtype=np.int8, count=e, offset=off).reshape(g.tensor_shape)
        off += e
        v_scales = np.frombuffer(data, dtype="<f4", count=vecs, offset=off).reshape(g.tensor_shape[:-1])
        off += 4 * vecs
        raw = np.frombuffer(data, dtype=np.uint8, count=v_payload, offset=off)
        off += v_payload
        kq = QuantizedKeyBlock(g, float(k_scale), torch.from_numpy(k_codes.copy()).to(dev))
        sc = torch.from_numpy(v_scales.astype(np.float32)).to(dev)
        if packed:
            vq = QuantizedValueBlock(g, GAUSSIAN_3BIT.name, GAUSSIAN_3BIT.bits, None, sc, sign_seed,
                                     packed=torch.from_numpy(raw.copy()).to(dev))
        else:
            vq = QuantizedValueBlock(g, GAUSSIAN_3BIT.name, GAUSSIAN_3BIT.bits,
                                     torch.from_numpy(raw.copy()).to(dev).view(g.tensor_shape), sc, sign_seed)
        layers.append((kq, vq))
    return SharedPool(g, layers, (), codebook=GAUSSIAN_3BIT, sign_seed=sign_seed).seal()
