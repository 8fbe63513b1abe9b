// TMA-streamed SharedKVPool codec kernels for B200 (sm_100a).
//
// Same semantics as the warp-granular kernels in codec.cu (and therefore as
// the reference: kvpool/keyquant.py:52-71, valuequant.py:193-238,
// pool.py:66-76, 229-237), re-organised around the memory system:
//
//   * persistent grid, one CTA per SM, launched cooperatively;
//   * warp 0 is a producer: its elected lane claims work items from a global
//     ticket counter (dynamic load balancing) and moves each item's input
//     tile HBM -> shared memory with TMA (cp.async.bulk / .tensor), landing
//     on an mbarrier;
//   * warps 1..8 are two consumer groups of four warps that take the ring
//     stages alternately, compute from shared memory and stage their outputs
//     in shared memory, from where one elected thread per group writes them
//     back with a TMA bulk/tensor store;
//   * head-vector tiles use 128/64/32-byte swizzled TMA boxes so that one lane
//     owns one head vector (no warp shuffles in the rotation) and still reads
//     / writes its 16-byte chunks without bank conflicts.
//
// Per-tensor key scales (keyquant.py:55) need max|K| over a whole layer
// before any key code can be written. The encode grid is split by role: value
// CTAs stream V (ALU-bound), key CTAs run the absmax pass one layer ahead of
// the key encode (L2 evict_last on the first read), so encoding layer l waits
// only on per-layer completion counts that were met a segment earlier, and
// re-reads layer l from L2. Each SM runs a single code path (mixing both on
// one SM thrashes its I-cache).
#include <cudaTypedefs.h>

#include <cstdlib>
#include <mutex>

#include "../../include/polykv.h"
#include "diag.h"
#include "codec_common.cuh"
#include "pkv_common.cuh"
#include "tma.cuh"

namespace pkv {
namespace stream {

constexpr int kWarpsPerGroup = 4;
constexpr int kGroupThreads = 32 * kWarpsPerGroup;
constexpr int kEncGroups = 3;
#ifndef PKV_ENC_CHUNK
#define PKV_ENC_CHUNK 16384
#endif
#ifndef PKV_ENC_CHUNK_F32
#define PKV_ENC_CHUNK_F32 8192
#endif
// elements per encode work item: 32 KB stages for both input types (two
// stages per consumer group), so f32 key items can also be copied to
// registers and their stage released before the math
template <typename TIn>
constexpr int enc_chunk() {
  return sizeof(TIn) == 4 ? PKV_ENC_CHUNK_F32 : PKV_ENC_CHUNK;
}
inline int enc_chunk_for(int elem_bytes) { return elem_bytes == 4 ? PKV_ENC_CHUNK_F32 : PKV_ENC_CHUNK; }
#ifndef PKV_B32_UNROLL
#define PKV_B32_UNROLL 2
#endif
constexpr int kB32Unroll = PKV_B32_UNROLL;  // block32 key encode: chunks in flight per lane
#ifndef PKV_KEY_EARLY_RELEASE
#define PKV_KEY_EARLY_RELEASE 1
#endif
constexpr bool kKeyEarlyRelease = PKV_KEY_EARLY_RELEASE;
#ifndef PKV_KEY_DYNAMIC
#define PKV_KEY_DYNAMIC 1  // per-tensor keys: readiness-driven A/E order (else static segments)
#endif
constexpr bool kKeyDynamic = PKV_KEY_DYNAMIC;
#ifndef PKV_ROLE_MAP
#define PKV_ROLE_MAP 0  // 0: roles by block index, 1: by SM id (measured slightly slower)
#endif
#ifndef PKV_ENC_XHALF
#define PKV_ENC_XHALF 1  // encode, two lanes per vector: the cross-half FWHT stage first, from shared memory
#endif
#ifndef PKV_SIGNPACK
#define PKV_SIGNPACK 1  // value codes packed from sign bits by funnel shifts
#endif  // bf16 key items: copy to registers, release the stage
constexpr int kDecChunk = 8192;   // elements per decode work item
constexpr int kEncRingBytes = 192 * 1024;
constexpr int kMaxL = kMaxLayers;

template <int NG>
constexpr int threads_for() {
  return 32 + NG * kGroupThreads;  // producer warp + consumer groups
}
constexpr int kEncThreads = threads_for<kEncGroups>();
template <typename TOut>
constexpr int dec_groups() {
  return sizeof(TOut) == 2 ? 3 : 2;
}

enum ItemKind : int { kEnd = 0, kAbsmax = 1, kKeyEnc = 2, kValEnc = 3, kKeyDec = 4, kValDec = 5, kBarrier = 6, kNone = 7 };

struct Item {
  int kind;
  int layer;
  int idx;
  int pad;
};

// How a head vector of D coordinates maps onto lanes: TPV lanes per vector
// (2 at d=128 so a lane holds at most 64 coordinates), lane = s * VPW + r for
// vector r of the warp's pass and half s; the lane owns the contiguous
// coordinates [s * CPT, (s + 1) * CPT).
template <int D>
struct VL {
  static constexpr int TPV = D == 128 ? 2 : 1;
  static constexpr int CPT = D / TPV;   // coordinates per lane
  static constexpr int NCL = CPT / 8;   // 8-coordinate chunks per lane
  static constexpr int NP = CPT / 2;    // f32 pairs per lane
  static constexpr int VPW = 32 / TPV;  // vectors per warp pass
  static constexpr int PB = 3 * D / 8;  // packed bytes per vector
  static constexpr int PBL = PB / TPV;  // packed bytes per lane
};

// Geometry of a head-vector tile of CHUNK elements (VR vectors of D) held as
// TMA boxes of BR rows x IB bytes (IB = swizzle span), NCB boxes across a row
// and NRB boxes down.
template <int D, int EB, int CHUNK, int WPG = kWarpsPerGroup>
struct Tile {
  static constexpr int RB = D * EB;               // bytes per head vector
  static constexpr int IB = RB < 128 ? RB : 128;  // inner box bytes
  static constexpr int NCB = RB / IB;
  static constexpr int VR = CHUNK / D;            // vectors per item
  static constexpr int NRB = (VR + 255) / 256;    // boxes down (TMA box rows <= 256)
  static constexpr int BR = VR / NRB;             // rows per box
  static_assert(BR * NRB == VR, "item rows split into equal boxes");
  static constexpr int BOX_BYTES = BR * IB;
  static constexpr int PER_PASS = WPG * VL<D>::VPW;
  static constexpr int PASSES = VR / PER_PASS;
  static_assert(VR % PER_PASS == 0, "item must hold whole passes");
  // byte offset of 16-byte unit u of vector vr inside the tile
  __device__ __forceinline__ static uint32_t off(int vr, int u) {
    constexpr int UPB = IB / 16;  // units per box row
    const int rb = vr / BR, r = vr % BR, cb = u / UPB, ub = u % UPB;
    return (uint32_t)((rb * NCB + cb) * BOX_BYTES) + tma::swz<IB>(r, ub);
  }
};

struct EncArgs {
  CUtensorMap tm_v[kMaxL];  // value inputs, [nvec, D] per layer
  int num_layers, head_dim, k_mode, in_bytes;
  long long nvec, nelem;
  int nE, nV;  // items per layer
  int dbg;  // PKV_DBG_ENC experiments: 1 skip all math, 2 skip values, 3 skip keys, 4 no layer wait, 5 no key re-read
  unsigned int total;
  float delta;
  Codebook3 cb;
  uint32_t sign_bits[8];
  uint32_t* status;
  uint32_t* replay_count;
  unsigned int* layer_max;  // [L] max |K| bits (published by the key-role CTAs)
  unsigned int* layer_done;   // [L] absmax items folded into layer_max (per-tensor mode)
  const uint32_t* k_max_ext;  // per-tensor keys: external max|K| bits per layer (no absmax pass)
  int value_ctas;             // CTAs [0, value_ctas) encode values, the rest keys
  int nA;                     // absmax items per layer (per-tensor mode)
  int abs_G;                  // > 0: CTAs issuing absmax items (round-robin, layer-major); each
                              // publishes its layer max once, after its last item of the layer.
                              // 0: every item publishes (static key schedule)
  int abs_target;             // layer_done[l] value meaning "layer l's max is complete"
  int nseg;                   // key-role segments of nE items: kind (A/E) + layer
  int key_lag;                // absmax layers allowed ahead of the key encode
  int abs_lead;               // > 0: the VALUE CTAs run the absmax items, abs_lead layers ahead of their V cursor
  int co_roles;               // enc_co_kernel: 0 = values on groups 0-2 + keys on group 3, 1 = all values, 2 = all keys
  uint8_t seg_absmax[2 * kMaxL];
  uint8_t seg_layer[2 * kMaxL];
  const void* k_in[kMaxL];
  const void* v_in[kMaxL];
  int8_t* k_codes[kMaxL];
  float* k_scale[kMaxL];
  __half* k_bscale[kMaxL];
  uint8_t* v_packed[kMaxL];
  float* v_scales[kMaxL];
};

struct DecArgs {
  CUtensorMap tm_v[kMaxL];  // value outputs, [nvec, D] per layer
  int num_layers, head_dim, k_mode, out_bytes;
  long long nvec, nelem;
  int nK, nV;
  int key_ctas;  // > 0: CTAs [grid - key_ctas, grid) decode keys, the rest values; 0: interleaved items
  unsigned int total;
  float sqrt_d32, rcp_sqrt_d32;
  uint32_t sign_bits[8];
  float cent32[8];
  const int8_t* k_codes[kMaxL];
  const float* k_scale[kMaxL];
  const __half* k_bscale[kMaxL];
  void* k_out[kMaxL];
  const uint8_t* v_packed[kMaxL];
  const float* v_scales[kMaxL];
};

__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ uint32_t ld_acquire_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ uint32_t ld_relaxed_u32(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
// acquire pattern for a relaxed read that observed a release (PTX memory
// model: observation + fence.acq_rel synchronizes with red.release)
__device__ __forceinline__ void fence_acq_rel_gpu() { asm volatile("fence.acq_rel.gpu;" ::: "memory"); }
__device__ __forceinline__ void red_release_add(uint32_t* p, uint32_t v) {
  asm volatile("red.release.gpu.global.add.u32 [%0], %1;" ::"l"(p), "r"(v) : "memory");
}

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
// arithmetic shift right by 31 (all ones for a set sign bit), kept as one SHF
__device__ __forceinline__ uint32_t sar31(uint32_t x) {
  uint32_t r;
  asm("shr.s32 %0, %1, 31;" : "=r"(r) : "r"(x));
  return r;
}
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __ffma2_rn(b, f2(-1.f, -1.f), a); }

// ---------------------------------------------------------------------------
// Sylvester FWHT over N contiguous coordinates held as N/2 f32 pairs of
// neighbours:  xp[q] = (x[2q], x[2q + 1]).
// Stages run half = 1, 2, 4, ..., N/2 with lo' = lo + hi, hi' = lo - hi,
// exactly kvpool/fwht.py:31-39, so every output is bit-identical to numpy.
// half = 1 combines the two halves of one register pair (two scalar ops);
// every later stage combines whole pairs (paired FADD2 / FFMA2). The layout
// is the one 16-byte loads and table lookups produce, so filling it needs no
// register moves (the previous (x[8c+e], x[8c+8+e]) pairing cost ~1.8
// IMAD.MOV per coordinate in the encode).
// ---------------------------------------------------------------------------
template <int N>
__device__ __forceinline__ void fwht_pairs(float2* xp) {
  constexpr int NP = N / 2;
#pragma unroll
  for (int p = 0; p < NP; ++p) {  // coordinate bit 0
    const float a = xp[p].x, b = xp[p].y;
    xp[p].x = __fadd_rn(a, b);
    xp[p].y = __fsub_rn(a, b);
  }
#pragma unroll
  for (int h = 1; h < NP; h <<= 1) {  // coordinate bits 1.. = pair-index bits 0..
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      if (p & h) continue;
      const float2 a = xp[p], b = xp[p + h];
      xp[p] = add2(a, b);
      xp[p + h] = sub2(a, b);
    }
  }
}

// Rotation of one head vector: the lane-local stages, then (two lanes per
// vector) the last stage half = D/2 across the lane pair: the lower half
// keeps lo + hi = mine + partner, the upper half lo - hi = partner - mine;
// fma(+-1, mine, partner) rounds exactly like numpy's add / subtract.
template <int D>
__device__ __forceinline__ void fwht_vector(float2* xp, int s) {
  using G = VL<D>;
  fwht_pairs<G::CPT>(xp);
  if constexpr (G::TPV == 2) {
    const float sg = s ? -1.f : 1.f;
#pragma unroll
    for (int p = 0; p < G::NP; ++p) {
      const float px = __shfl_xor_sync(0xffffffffu, xp[p].x, G::VPW);
      const float py = __shfl_xor_sync(0xffffffffu, xp[p].y, G::VPW);
      xp[p] = __ffma2_rn(f2(sg, sg), xp[p], f2(px, py));
    }
  }
}

// coordinate (within the lane's CPT) of pair p, half hh
__device__ __forceinline__ constexpr int coord_of(int p, int hh) { return 2 * p + hh; }

template <int NP>
__device__ __forceinline__ void apply_sign(float2* xp, const uint32_t* bits, int base) {
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const int i0 = base + coord_of(p, 0), i1 = base + coord_of(p, 1);
    xp[p].x = __uint_as_float(__float_as_uint(xp[p].x) ^ (((bits[i0 >> 5] >> (i0 & 31)) & 1u) << 31));
    xp[p].y = __uint_as_float(__float_as_uint(xp[p].y) ^ (((bits[i1 >> 5] >> (i1 & 31)) & 1u) << 31));
  }
}

// 8 inputs of one 16/32-byte chunk from shared memory -> f32
template <typename TIn>
__device__ __forceinline__ void lds_chunk8(uint32_t a0, uint32_t a1, float (&t)[8]);
template <>
__device__ __forceinline__ void lds_chunk8<__nv_bfloat16>(uint32_t a0, uint32_t, float (&t)[8]) {
  const uint4 w = tma::lds128(a0);
  t[0] = bf16lo(w.x); t[1] = bf16hi(w.x); t[2] = bf16lo(w.y); t[3] = bf16hi(w.y);
  t[4] = bf16lo(w.z); t[5] = bf16hi(w.z); t[6] = bf16lo(w.w); t[7] = bf16hi(w.w);
}
template <>
__device__ __forceinline__ void lds_chunk8<float>(uint32_t a0, uint32_t a1, float (&t)[8]) {
  const uint4 w = tma::lds128(a0), v = tma::lds128(a1);
  t[0] = __uint_as_float(w.x); t[1] = __uint_as_float(w.y); t[2] = __uint_as_float(w.z); t[3] = __uint_as_float(w.w);
  t[4] = __uint_as_float(v.x); t[5] = __uint_as_float(v.y); t[6] = __uint_as_float(v.z); t[7] = __uint_as_float(v.w);
}

// Exact fp64 replay of kvpool.valuequant.quantize_v for one head vector,
// executed by the whole warp; writes the packed bytes and the scale.
template <int D, typename TIn>
__device__ __noinline__ void v_replay(const EncArgs& a, const TIn* src, uint8_t* out_packed, float* out_scale,
                                      double* R, uint8_t* C) {
  const int lane = threadIdx.x & 31;
  for (int i = lane; i < D; i += 32) {
    double x = (double)load1(src + i);
    if (sign_bit(a.sign_bits, i)) x = -x;  // vals * sign_diagonal (valuequant.py:205)
    R[i] = x;
  }
  __syncwarp();
  for (int h = 1; h < D; h <<= 1) {  // fwht.py:31-39 in f64
    for (int q = lane; q < D / 2; q += 32) {
      const int i = (q / h) * 2 * h + (q % h);
      const double lo = R[i], hi = R[i + h];
      R[i] = lo + hi;
      R[i + h] = lo - hi;
    }
    __syncwarp();
  }
  const double sq = sqrt((double)D);  // fwht.py:50
  for (int i = lane; i < D; i += 32) R[i] = R[i] / sq;
  __syncwarp();
  // np.mean(np.square(rot)) (valuequant.py:207) in numpy's pairwise order
  // (pkv_common.cuh:pairwise_sumsq): for D <= 128 the eight interleaved
  // accumulators r[j] run on lanes 0..7, then ((r0+r1)+(r2+r3))+((r4+r5)+(r6+r7))
  // by butterflies (IEEE addition is commutative, so the xor partners give
  // lane 0 exactly numpy's result).
  double sum;
  if constexpr (D >= 8 && D <= 128) {
    double acc = 0.0;
    if (lane < 8) {
      acc = sq_rn(R[lane]);
      for (int i = 8 + lane; i < D; i += 8) acc = __dadd_rn(acc, sq_rn(R[i]));
    }
    acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 1));
    acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 2));
    acc = __dadd_rn(acc, __shfl_xor_sync(0xffffffffu, acc, 4));
    sum = acc;
  } else {
    sum = lane == 0 ? pairwise_sumsq(R, D) : 0.0;
  }
  double rms = 0.0;
  if (lane == 0) rms = sqrt(sum / (double)D);
  rms = __shfl_sync(0xffffffffu, rms, 0);
  const float scale = (float)rms;  // valuequant.py:208
  const double den = rms > 0.0 ? rms : 1.0;
  for (int i = lane; i < D; i += 32) {
    const double z = R[i] / den;  // valuequant.py:209
    int c = 0;
#pragma unroll
    for (int k = 0; k < 7; ++k) c += (a.cb.mid64[k] < z) ? 1 : 0;  // searchsorted 'left'
    C[i] = scale == 0.0f ? 0 : (uint8_t)c;                          // valuequant.py:211
  }
  __syncwarp();
  for (int w = lane; w < D / 8; w += 32) {
    uint32_t word = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) word |= (uint32_t)C[8 * w + e] << (3 * e);
    out_packed[3 * w + 0] = (uint8_t)(word & 0xff);
    out_packed[3 * w + 1] = (uint8_t)((word >> 8) & 0xff);
    out_packed[3 * w + 2] = (uint8_t)((word >> 16) & 0xff);
  }
  if (lane == 0) {
    *out_scale = scale;
    if (a.replay_count) atomicAdd(a.replay_count, 1u);
  }
  __syncwarp();
}

// rsqrt.approx.f64: ~2^-22 relative seed for the Newton steps below
__device__ __forceinline__ double rsqrt_seed(double x) {
  double y;
  asm("rsqrt.approx.ftz.f64 %0, %1;" : "=d"(y) : "d"(x));
  return y;
}

// The f32 value scale RN32(sqrt(S / D)) (valuequant.py:207-208) from the
// fp64 sum of squares S in [2^-200, 2^200], without an fp64 square root:
// r = T * y with T = S / D (exact) and y = 1/sqrt(T) from the rsqrt seed and
// two Newton steps (relative error of r < 2^-48, S itself is within
// D * 2^-53 of numpy's sum). The f32 rounding of r is trusted when r is
// farther than 2^-40 * r from the f32 rounding boundary on its side of
// c = RN32(r); otherwise returns false and the vector is replayed in numpy's
// exact order. Also N = ||x|| = sqrt(D) * r in f32 (for the code
// thresholds; its error is inside the guard band, guard_delta()).
template <int D>
__device__ __forceinline__ bool scale_from_sumsq(double S, float& scale, float& N) {
  const double T = S * (1.0 / D);
  double y = rsqrt_seed(T);
  y = y * fma(-0.5 * T, y * y, 1.5);
  y = y * fma(-0.5 * T, y * y, 1.5);
  const double r = T * y;
  const float c = __double2float_rn(r);
  const double cd = (double)c;
  const uint32_t cb = __float_as_uint(c);
  const double gap = r >= cd ? (double)__uint_as_float(cb + 1u) - cd : cd - (double)__uint_as_float(cb - 1u);
  const double dist = 0.5 * gap - fabs(r - cd);  // to the rounding boundary between c and its neighbour
  scale = c;
  N = __double2float_rn(r * (D == 64 ? 8.0 : D == 16 ? 4.0 : D == 128 ? 11.313708498984761 : 5.656854249492381));
  return dist > 0x1p-40 * r;
}

// pack NW 24-bit words (chunk order) and store them at global address `dst`
template <int NW>
__device__ __forceinline__ void stg_words(uint8_t* dst, const uint32_t (&w)[NW]) {
  if constexpr (NW % 4 == 0) {
    uint32_t u[3 * NW / 4];
#pragma unroll
    for (int i = 0; i < NW / 4; ++i) {
      u[3 * i + 0] = w[4 * i] | (w[4 * i + 1] << 24);
      u[3 * i + 1] = (w[4 * i + 1] >> 8) | (w[4 * i + 2] << 16);
      u[3 * i + 2] = (w[4 * i + 2] >> 16) | (w[4 * i + 3] << 8);
    }
    if constexpr (NW == 16) {
      st_u4(dst, make_uint4(u[0], u[1], u[2], u[3]));
      st_u4(dst + 16, make_uint4(u[4], u[5], u[6], u[7]));
      st_u4(dst + 32, make_uint4(u[8], u[9], u[10], u[11]));
    } else if constexpr (NW == 8) {
      st_u2(dst, make_uint2(u[0], u[1]));
      st_u2(dst + 8, make_uint2(u[2], u[3]));
      st_u2(dst + 16, make_uint2(u[4], u[5]));
    } else {
      uint32_t* d = reinterpret_cast<uint32_t*>(dst);
      d[0] = u[0];
      d[1] = u[1];
      d[2] = u[2];
    }
  } else {  // NW == 2: 6 bytes, 2-byte aligned
    const uint32_t lo = w[0] | (w[1] << 24), hi = w[1] >> 8;
    uint16_t* d = reinterpret_cast<uint16_t*>(dst);
    d[0] = (uint16_t)(lo & 0xffff);
    d[1] = (uint16_t)(lo >> 16);
    d[2] = (uint16_t)(hi & 0xffff);
  }
}

// ---------------------------------------------------------------------------
// encode: value item (VR head vectors)
// ---------------------------------------------------------------------------
template <int D, typename TIn, bool SYM, bool SIGN, int CH, int WPG>
__device__ void enc_value_item(const EncArgs& a, const Item& it, uint32_t in_s, int wig, int lane, double* R,
                               uint8_t* C) {
  using G = VL<D>;
  using TL = Tile<D, (int)sizeof(TIn), CH, WPG>;
  constexpr int NP = G::NP, NCL = G::NCL;
  const int r = lane % G::VPW, s = lane / G::VPW;
  const long long vbase = (long long)it.idx * TL::VR;
  const float* m = a.cb.mid32;
  const float delta = a.delta;
  uint8_t* gpk = a.v_packed[it.layer] + vbase * G::PB;
  float* gsc = a.v_scales[it.layer] + vbase;
#pragma unroll 1
  for (int pass = 0; pass < TL::PASSES; ++pass) {
    const int vr = pass * TL::PER_PASS + wig * G::VPW + r;
    const long long v = vbase + vr;
    const bool valid = v < a.nvec;
    float2 xp[NP];
    double sacc[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) sacc[k] = 0.0;
    auto chunk_in = [&](int gc, float (&t)[8]) {
      if constexpr (sizeof(TIn) == 2) {
        lds_chunk8<TIn>(in_s + TL::off(vr, gc), 0, t);
      } else {
        lds_chunk8<TIn>(in_s + TL::off(vr, 2 * gc), in_s + TL::off(vr, 2 * gc + 1), t);
      }
    };
#if PKV_ENC_XHALF
    if constexpr (G::TPV == 2) {
      // Two lanes per vector. The stage across the two halves (half = D/2)
      // runs FIRST, on inputs read from shared memory: each lane loads its
      // own half and its partner's (the tile is in shared memory anyway) and
      // keeps own + other (lower lane) or other - own (upper lane), so the
      // remaining stages are lane-local and the rotation needs no shuffle
      // (4 issue cycles per coordinate). The stage order differs from
      // numpy's, which the fast path allows: the guard band bounds the fp32
      // rounding of log2(d) butterfly layers in any order (guard_delta), and
      // any vector near a decision threshold is replayed in numpy's order.
      // (C3 value role: f32 156 -> 152 us, bf16 151 -> 140 us)
      const float sg = s ? -1.f : 1.f;
#pragma unroll
      for (int c = 0; c < NCL; ++c) {
        float t[8], o[8];
        chunk_in(s * NCL + c, t);
        chunk_in((1 - s) * NCL + c, o);
#pragma unroll
        for (int e = 0; e < 8; ++e) sacc[e & 3] = fma((double)t[e], (double)t[e], sacc[e & 3]);
        if (SIGN) {  // vals * sign_diagonal on both halves
#pragma unroll
          for (int e = 0; e < 8; ++e) {
            const int im = s * G::CPT + 8 * c + e, io = (1 - s) * G::CPT + 8 * c + e;
            t[e] = __uint_as_float(__float_as_uint(t[e]) ^ (((a.sign_bits[im >> 5] >> (im & 31)) & 1u) << 31));
            o[e] = __uint_as_float(__float_as_uint(o[e]) ^ (((a.sign_bits[io >> 5] >> (io & 31)) & 1u) << 31));
          }
        }
#pragma unroll
        for (int i = 0; i < 4; ++i)
          xp[4 * c + i] = __ffma2_rn(f2(sg, sg), f2(t[2 * i], t[2 * i + 1]), f2(o[2 * i], o[2 * i + 1]));
      }
    } else
#endif
    {
#pragma unroll
      for (int c = 0; c < NCL; ++c) {
        float t[8];
        chunk_in(s * NCL + c, t);  // chunk index within the vector
#pragma unroll
        for (int i = 0; i < 4; ++i) xp[4 * c + i] = f2(t[2 * i], t[2 * i + 1]);
      }
      // squared norm in fp64 from the inputs (the rotation is orthogonal);
      // every x^2 is exact in fp64 and the sum is good to ~D * 2^-53.
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        sacc[(2 * p) & 3] = fma((double)xp[p].x, (double)xp[p].x, sacc[(2 * p) & 3]);
        sacc[(2 * p + 1) & 3] = fma((double)xp[p].y, (double)xp[p].y, sacc[(2 * p + 1) & 3]);
      }
    }
    double S = (sacc[0] + sacc[1]) + (sacc[2] + sacc[3]);
    if constexpr (G::TPV == 2) S += __shfl_xor_sync(0xffffffffu, S, G::VPW);  // a + b == b + a
#if PKV_ENC_XHALF
    if constexpr (G::TPV == 2) {
      fwht_pairs<G::CPT>(xp);  // the lane-local stages
    } else
#endif
    {
      if (SIGN) apply_sign<NP>(xp, a.sign_bits, s * G::CPT);
      fwht_vector<D>(xp, s);  // U = H x (unnormalised)
    }

    bool replay = false, nonfinite = false, zero = false;
    float scale = 0.f, N = 0.f;
    if (!(S <= 1.79e308)) {
      nonfinite = true;
    } else if (S == 0.0) {
      zero = true;
    } else if (S < 0x1p-200 || S > 0x1p+200) {
      replay = true;
    } else {
      replay = !scale_from_sumsq<D>(S, scale, N);  // f32 rounding of the scale in doubt -> exact replay
    }

    uint32_t words[NCL];
#pragma unroll
    for (int c = 0; c < NCL; ++c) words[c] = 0;
    if (SYM) {
      // thresholds folded into the U domain: |z| > t  <=>  |U| > t * ||x||
      const float2 T1 = f2(-m[4] * N, -m[4] * N), T2 = f2(-m[5] * N, -m[5] * N), T3 = f2(-m[6] * N, -m[6] * N);
      const float DL = delta * N;
      // distance to the nearest decision threshold (0 included); 4
      // independent min-accumulators keep the FMNMX3 chains short
      float gacc[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) gacc[k] = INFINITY;
#if PKV_SIGNPACK
      // Codes from sign bits. s_k = sign(|u| - t_k N) is a thermometer code
      // (t1 < t2 < t3), mm = s1 + s2 + s3 = #thresholds above |u| has
      // bit1 = s2 and bit0 = s1^s2^s3, and code = negative ? mm : 7 - mm.
      // So, with n = sign(u): code bits (2,1,0) = ~(n, s2^n, s1^s2^s3^n).
      // Per coordinate the raw bits (n, s2, s1^s3) are shifted into the word
      // MSB-first (one funnel shift each, coordinate 7 of the chunk first);
      // the XOR chain and the complement then run once per 24-bit word:
      // bit1 ^= bit2, bit0 ^= bit1, ~ (one XOR per coordinate saved).
#pragma unroll
      for (int q = 0; q < NP; ++q) {
        const int p = (q & ~3) | (3 - (q & 3));  // pairs (7,6), (5,4), .. of each chunk
        const float2 u = xp[p];
        const float2 au = f2(fabsf(u.x), fabsf(u.y));
        const float2 d1 = __fadd2_rn(au, T1), d2 = __fadd2_rn(au, T2), d3 = __fadd2_rn(au, T3);
        float& ga = gacc[(2 * p) & 3];
        float& gb = gacc[(2 * p + 1) & 3];
        ga = fminf(ga, fminf(fabsf(d1.x), fabsf(d1.y)));
        gb = fminf(gb, fminf(fabsf(d2.x), fabsf(d2.y)));
        ga = fminf(ga, fminf(fabsf(d3.x), fabsf(d3.y)));
        gb = fminf(gb, fminf(au.x, au.y));
        const int c = p >> 2;
        const uint32_t ux = __float_as_uint(u.x), uy = __float_as_uint(u.y);
        const uint32_t b2x = __float_as_uint(d2.x), b2y = __float_as_uint(d2.y);
        const uint32_t b13x = __float_as_uint(d1.x) ^ __float_as_uint(d3.x);
        const uint32_t b13y = __float_as_uint(d1.y) ^ __float_as_uint(d3.y);
        // y is the odd (higher) coordinate of the pair: its bits go in first
        words[c] = __funnelshift_l(b13y, __funnelshift_l(b2y, __funnelshift_l(uy, words[c], 1), 1), 1);
        words[c] = __funnelshift_l(b13x, __funnelshift_l(b2x, __funnelshift_l(ux, words[c], 1), 1), 1);
      }
#pragma unroll
      for (int c = 0; c < NCL; ++c) {
        uint32_t w = words[c];                // fields (n, s2, s1^s3), 24 bits
        w ^= (w >> 1) & 0x492492u;            // bit1 = s2 ^ n
        w ^= (w >> 1) & 0x249249u;            // bit0 = s1 ^ s3 ^ s2 ^ n
        words[c] = w ^ 0xffffffu;             // complement (the upper 8 bits are 0)
      }
#else
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const float2 u = xp[p];
        const float2 au = f2(fabsf(u.x), fabsf(u.y));
        const float2 d1 = __fadd2_rn(au, T1), d2 = __fadd2_rn(au, T2), d3 = __fadd2_rn(au, T3);
        float& ga = gacc[(2 * p) & 3];
        float& gb = gacc[(2 * p + 1) & 3];
        ga = fminf(ga, fminf(fabsf(d1.x), fabsf(d1.y)));
        gb = fminf(gb, fminf(fabsf(d2.x), fabsf(d2.y)));
        ga = fminf(ga, fminf(fabsf(d3.x), fabsf(d3.y)));
        gb = fminf(gb, fminf(au.x, au.y));
        // mm = #thresholds above |u|; code = negative ? mm : 7 - mm = (mm ^ 7 ^ sign) & 7
        const uint32_t mx = (__float_as_uint(d1.x) >> 31) + (__float_as_uint(d2.x) >> 31) + (__float_as_uint(d3.x) >> 31);
        const uint32_t my = (__float_as_uint(d1.y) >> 31) + (__float_as_uint(d2.y) >> 31) + (__float_as_uint(d3.y) >> 31);
        const uint32_t cx = (mx ^ 7u ^ sar31(__float_as_uint(u.x))) & 7u;
        const uint32_t cy = (my ^ 7u ^ sar31(__float_as_uint(u.y))) & 7u;
        const int c = p >> 2, e = 2 * (p & 3);
        words[c] += cx << (3 * e);  // disjoint fields: + == |, one LEA
        words[c] += cy << (3 * e + 3);
      }
#endif
      const float g = fminf(fminf(gacc[0], gacc[1]), fminf(gacc[2], gacc[3]));
      replay |= g < DL;
    } else {
      const float inv = N > 0.f ? 1.0f / N : 0.f;
      float g = INFINITY;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
#pragma unroll
        for (int hh = 0; hh < 2; ++hh) {
          const float z = (hh ? xp[p].y : xp[p].x) * inv;
          const bool p1 = z > m[3];
          const float t2 = p1 ? m[5] : m[1];
          const bool p2 = z > t2;
          const float t3 = p1 ? (p2 ? m[6] : m[4]) : (p2 ? m[2] : m[0]);
          const bool p3 = z > t3;
          g = fminf(g, fminf(fabsf(z - m[3]), fminf(fabsf(z - t2), fabsf(z - t3))));
          words[p >> 2] |= ((p1 ? 4u : 0u) | (p2 ? 2u : 0u) | (p3 ? 1u : 0u)) << (3 * (2 * (p & 3) + hh));
        }
      }
      replay |= g < delta;
    }
    if (zero || nonfinite) {
#pragma unroll
      for (int c = 0; c < NCL; ++c) words[c] = 0;
      scale = 0.f;
    }
    if constexpr (G::TPV == 2) replay |= __shfl_xor_sync(0xffffffffu, (int)replay, G::VPW) != 0;
    replay = replay && valid && !nonfinite && !zero;
    if (valid && nonfinite && s == 0) atomicOr(&a.status[it.layer], PKV_FLAG_V_NONFINITE);
    if (valid && !replay) {
      stg_words<NCL>(gpk + vr * G::PB + s * G::PBL, words);
      if (s == 0) gsc[vr] = scale;
    }
    // rare: exact fp64 replay, one vector at a time, whole warp
    unsigned mask = __ballot_sync(0xffffffffu, replay && s == 0);
    while (mask) {
      const int src_lane = __ffs(mask) - 1;
      mask &= mask - 1;
      const int rvr = pass * TL::PER_PASS + wig * G::VPW + src_lane;
      const TIn* src = static_cast<const TIn*>(a.v_in[it.layer]) + (vbase + rvr) * D;
      v_replay<D, TIn>(a, src, gpk + rvr * G::PB, gsc + rvr, R, C);
    }
  }
}

// ---------------------------------------------------------------------------
// encode: key items
// ---------------------------------------------------------------------------
// max(|a|, |b|) with the sign of a ^ b, NaN if either input is NaN
__device__ __forceinline__ float absmax_nan(float a, float b) {
  float r;
  asm("max.NaN.xorsign.abs.f32 %0, %1, %2;" : "=f"(r) : "f"(a), "f"(b));
  return r;
}

// |x| bit patterns of 8 inputs from shared memory, max-reduced
template <typename TIn>
__device__ __forceinline__ uint32_t lds_absmax8(uint32_t a);
template <>
__device__ __forceinline__ uint32_t lds_absmax8<__nv_bfloat16>(uint32_t a) {
  const uint4 w = tma::lds128(a);
  uint32_t m = __vmaxu2(__vmaxu2(w.x & 0x7fff7fffu, w.y & 0x7fff7fffu), __vmaxu2(w.z & 0x7fff7fffu, w.w & 0x7fff7fffu));
  m = max(m & 0xffffu, m >> 16);
  return m << 16;
}
template <>
__device__ __forceinline__ uint32_t lds_absmax8<float>(uint32_t a) {
  const uint4 w = tma::lds128(a), v = tma::lds128(a + 16);
  const uint32_t m = max(max(w.x & 0x7fffffffu, w.y & 0x7fffffffu), max(w.z & 0x7fffffffu, w.w & 0x7fffffffu));
  return max(m, max(max(v.x & 0x7fffffffu, v.y & 0x7fffffffu), max(v.z & 0x7fffffffu, v.w & 0x7fffffffu)));
}

template <typename TIn, int CH, int GT>
__device__ uint32_t enc_absmax_item(const EncArgs& a, const Item& it, uint32_t in_s, int gt) {
  constexpr int kEncChunk = CH, kGroupThreads = GT;
  const long long e0 = (long long)it.idx * kEncChunk;
  const int n = (int)min((long long)kEncChunk, a.nelem - e0);
  uint32_t m = 0;
  if constexpr (sizeof(TIn) == 2) {
    if (n == kEncChunk) {
      // bf16 pairs: one NaN-propagating |.| max per 2 elements (HMNMX2), the
      // two halves folded once per item; a NaN ends above +inf like the bit
      // patterns of the generic path
      __nv_bfloat162 acc = __floats2bfloat162_rn(0.f, 0.f);
#pragma unroll
      for (int i = 0; i < kEncChunk / 8 / kGroupThreads; ++i) {
        const uint4 w = tma::lds128(in_s + (i * kGroupThreads + gt) * 16);
        const __nv_bfloat162 p = __hmax2_nan(__habs2(*reinterpret_cast<const __nv_bfloat162*>(&w.x)),
                                             __habs2(*reinterpret_cast<const __nv_bfloat162*>(&w.y)));
        const __nv_bfloat162 q = __hmax2_nan(__habs2(*reinterpret_cast<const __nv_bfloat162*>(&w.z)),
                                             __habs2(*reinterpret_cast<const __nv_bfloat162*>(&w.w)));
        acc = __hmax2_nan(acc, __hmax2_nan(p, q));
      }
      const uint32_t ab = *reinterpret_cast<uint32_t*>(&acc);
      m = max(ab & 0x7fffu, (ab >> 16) & 0x7fffu) << 16;  // |.| patterns: NaN (0x7fff) > inf
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
      return m;
    }
  }
  if constexpr (sizeof(TIn) == 4) {
    if (n == kEncChunk) {
      // f32: one NaN-propagating max of magnitudes per element
      // (max.NaN.xorsign.abs: |result| = max(|a|, |b|), NaN if either is NaN;
      // the sign is dropped at the end), two independent chains
      float acc0 = 0.f, acc1 = 0.f;
#pragma unroll
      for (int i = 0; i < kEncChunk / 8 / kGroupThreads; ++i) {
        const uint32_t a0 = in_s + (i * kGroupThreads + gt) * 32;
        const uint4 w = tma::lds128(a0), v = tma::lds128(a0 + 16);
        acc0 = absmax_nan(absmax_nan(acc0, __uint_as_float(w.x)), __uint_as_float(w.y));
        acc1 = absmax_nan(absmax_nan(acc1, __uint_as_float(w.z)), __uint_as_float(w.w));
        acc0 = absmax_nan(absmax_nan(acc0, __uint_as_float(v.x)), __uint_as_float(v.y));
        acc1 = absmax_nan(absmax_nan(acc1, __uint_as_float(v.z)), __uint_as_float(v.w));
      }
      m = __float_as_uint(absmax_nan(acc0, acc1)) & 0x7fffffffu;  // NaN (0x7fc00000) > inf like the bit path
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
      return m;
    }
  }
  if (n == kEncChunk) {
#pragma unroll
    for (int i = 0; i < kEncChunk / 8 / kGroupThreads; ++i)
      m = max(m, lds_absmax8<TIn>(in_s + (i * kGroupThreads + gt) * 8 * (int)sizeof(TIn)));
  } else {
#pragma unroll 1
    for (int i = 0; i < kEncChunk / 8 / kGroupThreads; ++i) {
      const int u = i * kGroupThreads + gt;
      if (u * 8 < n) m = max(m, lds_absmax8<TIn>(in_s + u * 8 * (int)sizeof(TIn)));
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  return m;
}

// release() hands the input stage back to the producer; a path that has
// copied the stage into registers calls it before computing (and the caller
// then must not release again: `released` is set).
template <typename TIn, int CH, int GT, class Release>
__device__ void enc_key_item(const EncArgs& a, const Item& it, uint32_t in_s, int gt, int lane,
                             const uint32_t* layer_max, Release release, bool& released) {
  constexpr int kEncChunk = CH, kGroupThreads = GT;
  const long long e0 = (long long)it.idx * kEncChunk;
  const int n = (int)min((long long)kEncChunk, a.nelem - e0);
  int8_t* dst = a.k_codes[it.layer] + e0;
  if (a.k_mode == PKV_K_TENSOR) {
    const uint32_t pb = layer_max[it.layer];  // staged in smem once layer_done[l] == nA
    const bool nonfinite = pb >= 0x7f800000u;
    const float s = (nonfinite || pb == 0) ? 0.f : __uint_as_float(pb) / 127.0f;  // f32(peak/127), keyquant.py:60
    if (it.idx == 0 && gt == 0) {
      a.k_scale[it.layer][0] = s;
      if (nonfinite) atomicOr(&a.status[it.layer], PKV_FLAG_K_NONFINITE);
    }
    const float rcp = 1.0f / s;
    const bool exact_all = !(s >= 1e-30f);
    constexpr int ITERS = kEncChunk / 8 / kGroupThreads;
    if constexpr (kKeyEarlyRelease) {
      if (n == kEncChunk && !exact_all) {
        // full item: the lane's ITERS chunks of 8 inputs (64 registers for
        // both input types: 32 KB stages) are copied out and the stage
        // released at once, so its refill overlaps the math. Branch-free
        // pass; chunks near a half-point are re-coded from global memory
        // afterwards (rare; the stage may be refilled by then)
        constexpr int UPC = (int)sizeof(TIn) / 2;  // 16-byte units per chunk of 8 inputs
        uint4 raw[ITERS * UPC];
#pragma unroll
        for (int i = 0; i < ITERS; ++i)
#pragma unroll
          for (int h = 0; h < UPC; ++h)
            raw[i * UPC + h] = tma::lds128(in_s + ((i * kGroupThreads + gt) * UPC + h) * 16);
        release();
        released = true;
        uint32_t need = 0;
#pragma unroll
        for (int i = 0; i < ITERS; ++i) {
          const int u = i * kGroupThreads + gt;
          float x[8];
          if constexpr (UPC == 1) {
            const uint4 r = raw[i];
            x[0] = bf16lo(r.x); x[1] = bf16hi(r.x); x[2] = bf16lo(r.y); x[3] = bf16hi(r.y);
            x[4] = bf16lo(r.z); x[5] = bf16hi(r.z); x[6] = bf16lo(r.w); x[7] = bf16hi(r.w);
          } else {
            const uint4 r0 = raw[2 * i], r1 = raw[2 * i + 1];
            x[0] = __uint_as_float(r0.x); x[1] = __uint_as_float(r0.y); x[2] = __uint_as_float(r0.z);
            x[3] = __uint_as_float(r0.w); x[4] = __uint_as_float(r1.x); x[5] = __uint_as_float(r1.y);
            x[6] = __uint_as_float(r1.z); x[7] = __uint_as_float(r1.w);
          }
          bool bad;
          st_u2(dst + u * 8, key_chunk_fast(x, make_float2(rcp, rcp), bad));
          need |= (uint32_t)bad << i;
        }
        const TIn* src = static_cast<const TIn*>(a.k_in[it.layer]) + e0;
#pragma unroll 1
        while (need) {
          const int i = __ffs(need) - 1;
          need &= need - 1;
          const int u = i * kGroupThreads + gt;
          float x[8];
          load8(src + u * 8, x);
          uint32_t c[8];
#pragma unroll
          for (int j = 0; j < 8; ++j) c[j] = key_code_fma(x[j], s, rcp, -128, 127);
          st_u2(dst + u * 8, make_uint2(c[0] | (c[1] << 8) | (c[2] << 16) | (c[3] << 24),
                                        c[4] | (c[5] << 8) | (c[6] << 16) | (c[7] << 24)));
        }
        return;
      }
    }
    // branch-free fast pass over the whole item; chunks near a rounding
    // half-point are re-coded exactly afterwards (rare)
    uint32_t need = 0;
    auto chunk = [&](int i) {
      const int u = i * kGroupThreads + gt;
      float x[8];
      lds_chunk8<TIn>(in_s + u * 8 * (int)sizeof(TIn), in_s + u * 8 * (int)sizeof(TIn) + 16, x);
      bool bad;
      st_u2(dst + u * 8, key_chunk_fast(x, make_float2(rcp, rcp), bad));
      need |= (uint32_t)bad << i;
    };
    if (n == kEncChunk) {  // full item: straight-line code, chunks interleave
#pragma unroll
      for (int i = 0; i < ITERS; ++i) chunk(i);
    } else {
#pragma unroll 1
      for (int i = 0; i < ITERS; ++i)
        if ((i * kGroupThreads + gt) * 8 < n) chunk(i);
    }
    if (exact_all) need = (1u << ITERS) - 1u;
#pragma unroll 1
    while (need) {
      const int i = __ffs(need) - 1;
      need &= need - 1;
      const int u = i * kGroupThreads + gt;
      if (u * 8 >= n) continue;
      float x[8];
      lds_chunk8<TIn>(in_s + u * 8 * (int)sizeof(TIn), in_s + u * 8 * (int)sizeof(TIn) + 16, x);
      uint32_t c[8];
#pragma unroll
      for (int j = 0; j < 8; ++j)
        c[j] = exact_all ? (s == 0.f ? 0u : ((uint32_t)key_code_exact(x[j], s, -128, 127) & 0xffu))
                         : key_code_fma(x[j], s, rcp, -128, 127);
      st_u2(dst + u * 8, make_uint2(c[0] | (c[1] << 8) | (c[2] << 16) | (c[3] << 24),
                                    c[4] | (c[5] << 8) | (c[6] << 16) | (c[7] << 24)));
    }
    return;
  }
  // block32: one fp16 scale per 32 contiguous elements; 4 consecutive lanes own a block
  __half* bsc = a.k_bscale[it.layer];
#pragma unroll kB32Unroll
  for (int i = 0; i < kEncChunk / 8 / kGroupThreads; ++i) {
    const int u = i * kGroupThreads + gt;
    const bool valid = u * 8 < n;
    const uint32_t a0 = in_s + u * 8 * (int)sizeof(TIn);
    uint32_t m = valid ? lds_absmax8<TIn>(a0) : 0u;  // max |x| bits of the lane's 8
    m = max(m, __shfl_xor_sync(0xffffffffu, m, 1));
    m = max(m, __shfl_xor_sync(0xffffffffu, m, 2));
    if (!valid) continue;
    float x[8];
    lds_chunk8<TIn>(a0, a0 + 16, x);
    // f16(f32(peak / 127)) (keyquant.py:60 per block, then the fp16 store)
    const float pk = __uint_as_float(m);
    const bool in_range = m >= 0x0d800000u && m <= 0x71800000u;  // [2^-100, 2^100]: div127's verified range
    uint16_t s16b = __half_as_ushort(__float2half_rn(div127_core(pk)));
    const uint32_t ex = s16b & 0x7c00u;
    uint2 w;
    if (in_range && ex != 0u && ex != 0x7c00u) {
      // normal fp16 scale: s >= (peak/127)(1 - 2^-11), so |x|/s < 127.07 and
      // the clip never acts; paired fast path (rcp.approx is within 1 ulp:
      // 127.07 * 2^-23 < 2^-16, inside the kKeyGuard margin), FMA-exact
      // re-code near a half-point
      const float s = __half2float(__ushort_as_half(s16b));
      const float rcp = rcp_approx(s);
      bool bad;
      w = key_chunk_fast(x, make_float2(rcp, rcp), bad);
      if (bad) {
        uint32_t c[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = key_code_fma(x[j], s, rcp, -127, 127);
        w = make_uint2(c[0] | (c[1] << 8) | (c[2] << 16) | (c[3] << 24), c[4] | (c[5] << 8) | (c[6] << 16) | (c[7] << 24));
      }
    } else {
      // zero / non-finite peak, fp16 overflow or underflow, extreme range
      const bool nonfinite = m >= 0x7f800000u;
      s16b = __half_as_ushort(__float2half_rn(__fdiv_rn(pk, 127.0f)));
      bool overflow = false;
      if (nonfinite || m == 0) {
        s16b = 0;
      } else if ((s16b & 0x7fffu) >= 0x7c00u) {
        overflow = true;
        s16b = 0;
      } else if (s16b == 0) {
        s16b = 1;  // peak > 0 but the scale underflows fp16: smallest subnormal
      }
      if ((lane & 3) == 0) {
        if (nonfinite) atomicOr(&a.status[it.layer], PKV_FLAG_K_NONFINITE);
        if (overflow) atomicOr(&a.status[it.layer], PKV_FLAG_K_SCALE_OVERFLOW);
      }
      const float s = __half2float(__ushort_as_half(s16b));
      w = key_chunk<true>(x, s, 1.0f / s, !(s >= 1e-30f));
    }
    if ((lane & 3) == 0) bsc[(e0 + u * 8) >> 5] = __ushort_as_half(s16b);
    st_u2(dst + u * 8, w);
  }
}

// ---------------------------------------------------------------------------
// decode: key and value items
// ---------------------------------------------------------------------------
// B32: block32 keys (fp16 scales staged behind the codes); a separate
// instantiation keeps that code (and its registers) out of the per-tensor kernel
template <typename TOut, bool B32>
__device__ void dec_key_item(const DecArgs& a, const Item& it, uint32_t in_s, uint8_t* out, int gt) {
  const long long e0 = (long long)it.idx * kDecChunk;
  const int n = (int)min((long long)kDecChunk, a.nelem - e0);
  constexpr bool tensor = !B32;
  const float ts = tensor ? __ldg(a.k_scale[it.layer]) : 0.f;
  const __half* bsc = a.k_bscale[it.layer];
  const uint32_t out_s = tma::smem_u32(out);
  const bool full = n == kDecChunk;
  const int sm_scales = ((((n + 31) / 32) * 2) & ~15) / 2;  // block scales staged in smem
#pragma unroll
  for (int i = 0; i < kDecChunk / 8 / kGroupThreads; ++i) {
    const int u = i * kGroupThreads + gt;
    if (!full && u * 8 >= n) continue;
    const uint2 w = tma::lds64(in_s + u * 8);
    float s = ts;
    if (!tensor) {
      const int b = (u * 8) >> 5;
      s = b < sm_scales ? __half2float(__ushort_as_half((unsigned short)(tma::lds32(in_s + kDecChunk + (b & ~1) * 2) >>
                                                                          (16 * (b & 1)))))
                        : __half2float(__ldg(bsc + ((e0 + u * 8) >> 5)));
    }
    const uint32_t wx = w.x ^ 0x80808080u, wy = w.y ^ 0x80808080u;
    float y[8];
#pragma unroll
    for (int j = 0; j < 4; ++j) y[j] = i8_to_f32(wx, j) * s;  // dequantize_k: code * scale (keyquant.py:71)
#pragma unroll
    for (int j = 0; j < 4; ++j) y[4 + j] = i8_to_f32(wy, j) * s;
    if constexpr (sizeof(TOut) == 2) {
      tma::sts128(out_s + u * 16, make_uint4(pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]),
                                             pack_bf16x2(y[4], y[5]), pack_bf16x2(y[6], y[7])));
    } else {
      tma::sts128(out_s + u * 32, make_uint4(__float_as_uint(y[0]), __float_as_uint(y[1]), __float_as_uint(y[2]),
                                             __float_as_uint(y[3])));
      tma::sts128(out_s + u * 32 + 16, make_uint4(__float_as_uint(y[4]), __float_as_uint(y[5]),
                                                  __float_as_uint(y[6]), __float_as_uint(y[7])));
    }
  }
}

// NW packed 24-bit words (chunk order) from shared or global memory
// The block32 key decode as a separate (non-inlined) function: inlined, its
// register demand spilled in the value path of the same kernel (value decode
// 88 -> 107 us in block32 launches).
template <typename TOut>
__device__ __noinline__ void dec_key_item_b32(const DecArgs& a, const Item& it, uint32_t in_s, uint8_t* out, int gt) {
  dec_key_item<TOut, true>(a, it, in_s, out, gt);
}

template <int NW>
__device__ __forceinline__ void load_packed(const uint8_t* p, bool smem, uint32_t (&w)[NW]) {
  if constexpr (NW % 4 == 0) {
    constexpr int NU = 3 * NW / 4;
    uint32_t u[NU];
    if (smem) {
      const uint32_t s = tma::smem_u32(p);
      if constexpr (NU == 12) {
        const uint4 a = tma::lds128(s), b = tma::lds128(s + 16), c = tma::lds128(s + 32);
        u[0] = a.x; u[1] = a.y; u[2] = a.z; u[3] = a.w; u[4] = b.x; u[5] = b.y;
        u[6] = b.z; u[7] = b.w; u[8] = c.x; u[9] = c.y; u[10] = c.z; u[11] = c.w;
      } else if constexpr (NU == 6) {
        const uint2 a = tma::lds64(s), b = tma::lds64(s + 8), c = tma::lds64(s + 16);
        u[0] = a.x; u[1] = a.y; u[2] = b.x; u[3] = b.y; u[4] = c.x; u[5] = c.y;
      } else {
        u[0] = tma::lds32(s); u[1] = tma::lds32(s + 4); u[2] = tma::lds32(s + 8);
      }
    } else {
#pragma unroll
      for (int i = 0; i < NU; ++i)
        u[i] = (uint32_t)p[4 * i] | ((uint32_t)p[4 * i + 1] << 8) | ((uint32_t)p[4 * i + 2] << 16) |
               ((uint32_t)p[4 * i + 3] << 24);
    }
#pragma unroll
    for (int i = 0; i < NW / 4; ++i) {
      w[4 * i + 0] = u[3 * i] & 0xffffffu;
      w[4 * i + 1] = __funnelshift_r(u[3 * i], u[3 * i + 1], 24) & 0xffffffu;
      w[4 * i + 2] = __funnelshift_r(u[3 * i + 1], u[3 * i + 2], 16) & 0xffffffu;
      w[4 * i + 3] = u[3 * i + 2] >> 8;
    }
  } else {
#pragma unroll
    for (int j = 0; j < NW; ++j)
      w[j] = (uint32_t)p[3 * j] | ((uint32_t)p[3 * j + 1] << 8) | ((uint32_t)p[3 * j + 2] << 16);
  }
}

template <int D, typename TOut, bool SIGN>
__device__ void dec_value_item(const DecArgs& a, const Item& it, uint8_t* in, int in_packed_bytes,
                               int in_scale_bytes, uint8_t* out, float* tbl, int gt, int wig, int lane) {
  using G = VL<D>;
  using TL = Tile<D, (int)sizeof(TOut), kDecChunk>;
  constexpr int NCL = G::NCL, NP = G::NP;
  const int r = lane % G::VPW, s = lane / G::VPW;
  const long long vbase = (long long)it.idx * TL::VR;
  const uint8_t* gpk = a.v_packed[it.layer] + vbase * G::PB;
  const float* gsc = a.v_scales[it.layer] + vbase;
  const float* ssc = reinterpret_cast<const float*>(in + 3 * kDecChunk / 8);
  const uint32_t out_s = tma::smem_u32(out);
  const float2 nc2 = f2(-a.sqrt_d32, -a.sqrt_d32), r2 = f2(a.rcp_sqrt_d32, a.rcp_sqrt_d32);
  // table[code][gt] at tbl_s | code << 9 | gt << 2  (tables are 4 KB aligned)
  const uint32_t lane_off = tma::smem_u32(tbl) + (uint32_t)gt * 4u;
#pragma unroll 1
  for (int pass = 0; pass < TL::PASSES; ++pass) {
    const int vr = pass * TL::PER_PASS + wig * G::VPW + r;
    const bool valid = vbase + vr < a.nvec;
    uint32_t words[NCL];
    float sc = 0.f;
    if (valid) {
      const int o = vr * G::PB + s * G::PBL;
      const bool pk_smem = o + G::PBL <= in_packed_bytes;
      load_packed<NCL>(pk_smem ? in + o : gpk + o, pk_smem, words);
      sc = (vr + 1) * 4 <= in_scale_bytes ? ssc[vr] : __ldg(gsc + vr);
    } else {
#pragma unroll
      for (int j = 0; j < NCL; ++j) words[j] = 0;
    }
    // per-lane table of the 8 scaled centroids: table_f32[code] * scale
    // (valuequant.py:232-234), laid out [code][thread] -> conflict-free
#pragma unroll
    for (int k = 0; k < 8; ++k) tbl[k * kGroupThreads + gt] = a.cent32[k] * sc;
    float2 xp[NP];
#pragma unroll
    for (int c = 0; c < NCL; ++c) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        // shared address lane_off | (code << 9)   (kGroupThreads * 4 == 512)
        const int sh = 3 * e;
        const uint32_t off = (sh <= 9 ? (words[c] << (9 - sh)) : (words[c] >> (sh - 9))) & 0xe00u;
        const float val = __uint_as_float(tma::lds32(off | lane_off));
        if (e & 1) xp[4 * c + (e >> 1)].y = val;
        else xp[4 * c + (e >> 1)].x = val;
      }
    }
    fwht_vector<D>(xp, s);
    // / f32(sqrt(d)) (fwht.py:50): correctly rounded via one FMA correction
    // (exact for power-of-four d); scale == 0 or tiny -> IEEE division keeps
    // the signs of zeros and subnormal quotients.
    if (sc >= 0x1p-80f) {
      constexpr bool pow4 = (VG<D>::LOG2D % 2) == 0;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const float2 q = __fmul2_rn(xp[p], r2);
        if (pow4) {
          xp[p] = q;
        } else {
          const float2 e = __ffma2_rn(q, nc2, xp[p]);  // x - q*c, exact remainder
          xp[p] = __ffma2_rn(e, r2, q);
        }
      }
    } else {
#pragma unroll
      for (int p = 0; p < NP; ++p) xp[p] = f2(__fdiv_rn(xp[p].x, a.sqrt_d32), __fdiv_rn(xp[p].y, a.sqrt_d32));
    }
    if (SIGN) apply_sign<NP>(xp, a.sign_bits, s * G::CPT);
    // swizzled staging of the output tile (TMA tensor store layout)
#pragma unroll
    for (int c = 0; c < NCL; ++c) {
      const int gc = s * NCL + c;
      float y[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) y[e] = (e & 1) ? xp[4 * c + (e >> 1)].y : xp[4 * c + (e >> 1)].x;
      if constexpr (sizeof(TOut) == 2) {
        tma::sts128(out_s + TL::off(vr, gc), make_uint4(pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]),
                                                        pack_bf16x2(y[4], y[5]), pack_bf16x2(y[6], y[7])));
      } else {
        tma::sts128(out_s + TL::off(vr, 2 * gc), make_uint4(__float_as_uint(y[0]), __float_as_uint(y[1]),
                                                            __float_as_uint(y[2]), __float_as_uint(y[3])));
        tma::sts128(out_s + TL::off(vr, 2 * gc + 1), make_uint4(__float_as_uint(y[4]), __float_as_uint(y[5]),
                                                                __float_as_uint(y[6]), __float_as_uint(y[7])));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// ticket -> item
// ---------------------------------------------------------------------------
// Encode work lists. The grid is split by role (one code path per SM):
//   value CTAs [0, value_ctas):  V(l, j) for all layers, layer-major;
//   key CTAs (per-tensor mode): segments of nE items
//     A(0) .. A(lag-1) | A(lag) E(0) | A(lag+1) E(1) | ... | E(L-1)
//   i.e. the absmax pass runs `lag` layers ahead of the key encode, lag
//   chosen so that the grid's in-flight stages fit in the gap: E(l) waits
//   only for the A(l) items (counted in layer_done[l]), which every CTA has
//   finished by then, and re-reads layer l while it is still in L2. Block32
//   mode has no absmax: E(0) .. E(L-1).
// Each CTA walks a static round-robin slice of its role's list.
__device__ __forceinline__ Item enc_value_item_at(const EncArgs& a, long long t) {
  Item it{kValEnc, 0, 0, 0};
  it.layer = (int)(t / a.nV);
  it.idx = (int)(t - (long long)it.layer * a.nV);
  return it;
}
__device__ __forceinline__ Item enc_key_item_at(const EncArgs& a, long long t) {
  const int seg = (int)(t / a.nE);
  return Item{a.seg_absmax[seg] ? kAbsmax : kKeyEnc, a.seg_layer[seg], (int)(t - (long long)seg * a.nE), 0};
}

__device__ __forceinline__ Item dec_item(const DecArgs& a, unsigned int t) {
  const long long per = (long long)a.nK + a.nV;
  Item it{kEnd, 0, 0, 0};
  it.layer = (int)(t / per);
  long long off = t - (long long)it.layer * per;
  const long long both = 2 * (long long)min(a.nK, a.nV);
  if (off < both) {
    it.kind = (off & 1) ? kValDec : kKeyDec;
    it.idx = (int)(off >> 1);
  } else {
    off -= both;
    it.kind = a.nK > a.nV ? kKeyDec : kValDec;
    it.idx = (int)(min(a.nK, a.nV) + off);
  }
  return it;
}

// ---------------------------------------------------------------------------
// shared-memory plans
// ---------------------------------------------------------------------------
// Every consumer group owns a private ring of NSG input stages, so a slow item
// (a layer-max wait, an fp64 replay) only ever stalls its own group. Encode
// outputs are small and go straight to global memory; decode outputs are
// staged in two buffers per group and written back by TMA stores.
constexpr int kMaxGroups = 4;
constexpr int kMaxSG = 4;

template <int EB_IN>
struct EncPlan {
  static constexpr int NG = kEncGroups;
  static constexpr int STAGE = (EB_IN == 4 ? PKV_ENC_CHUNK_F32 : PKV_ENC_CHUNK) * EB_IN;
  static constexpr int NSG = kEncRingBytes / STAGE / NG;  // stages per group
  static_assert(NSG >= 1 && NSG <= kMaxSG, "ring depth");
};
template <int EB_OUT, int NG_>
struct DecPlan {
  static constexpr int NG = NG_;
#ifndef PKV_DEC_STAGE_EXTRA
#define PKV_DEC_STAGE_EXTRA 1024
#endif
  static constexpr int STAGE = kDecChunk + PKV_DEC_STAGE_EXTRA;  // key codes + block32 scales / packed values + scales
  static constexpr int OUT = kDecChunk * EB_OUT;
  static constexpr int NOB = 2;            // output buffers per group
  static constexpr int OUT_TOTAL = NG * NOB * OUT;
  static constexpr int NSG = 3;
  static_assert(OUT_TOTAL + NG * NSG * STAGE <= 200 * 1024, "decode shared memory");
};

struct alignas(8) Ctl {
  uint64_t full[kMaxGroups][kMaxSG];
  uint64_t empty[kMaxGroups][kMaxSG];
  Item items[kMaxGroups][kMaxSG];
  uint32_t layer_max[kMaxL];  // encode: max |K| bits per layer, staged once layer_done is complete
  uint32_t ready[kMaxL];      // encode: layer_max[l] staged
  // encode: absmax fold of the warps of one stage use; two slots per stage
  // (use parity): a warp releases the stage before folding, so a fast warp
  // can start the next use of the stage while a slow one still folds this one
  uint32_t gmax[kMaxGroups][kMaxSG][2];
  uint32_t gcnt[kMaxGroups][kMaxSG][2];
  // encode: this CTA's per-layer absmax fold (max bits, items folded)
  uint32_t cta_max[kMaxL];
  uint32_t cta_cnt[kMaxL];
};

// Items t in [0, x) with t = r (mod G).
__device__ __forceinline__ uint32_t residues_below(uint32_t x, uint32_t r, uint32_t G) {
  return x > r ? (x - 1 - r) / G + 1 : 0u;
}

// One absmax item's max (already folded over the group's warps) into the
// layer maximum. With abs_G > 0 it is folded into the CTA's per-layer slot and
// the CTA's LAST item of the layer publishes: one global atomicMax and one
// release per CTA and layer instead of per item (a release waits for all of
// the thread's earlier global stores -- the key codes it wrote -- so one per
// item stalled the key role: C3 f32 encode 318 -> 305 us without them).
__device__ __forceinline__ void fold_absmax(const EncArgs& a, Ctl* ctl, int l, uint32_t m, uint32_t rank) {
  if (a.abs_G <= 0) {
    if (m) atomicMax(a.layer_max + l, m);
    red_release_add(a.layer_done + l, 1u);  // orders the max before the count
    return;
  }
  if (m) atomicMax(&ctl->cta_max[l], m);
  __threadfence_block();
  const uint32_t G = (uint32_t)a.abs_G, lo = (uint32_t)l * (uint32_t)a.nA, hi = lo + (uint32_t)a.nA;
  const uint32_t mine = residues_below(hi, rank, G) - residues_below(lo, rank, G);
  if (atomicAdd(&ctl->cta_cnt[l], 1u) + 1u == mine) {
    __threadfence_block();
    const uint32_t cm = atomicOr(&ctl->cta_max[l], 0u);
    if (cm) atomicMax(a.layer_max + l, cm);
    red_release_add(a.layer_done + l, 1u);
  }
}

template <int D, typename TIn>
constexpr size_t enc_smem_bytes() {
  using P = EncPlan<(int)sizeof(TIn)>;
  return 1024 + (size_t)P::NG * P::NSG * P::STAGE + sizeof(Ctl) + (size_t)P::NG * kWarpsPerGroup * (D * 8 + D);
}
template <typename TOut>
constexpr size_t dec_smem_bytes() {
  using P = DecPlan<(int)sizeof(TOut), dec_groups<TOut>()>;
  return 4096 + (size_t)P::OUT_TOTAL + (size_t)P::NG * P::NSG * P::STAGE + sizeof(Ctl) +
         (size_t)P::NG * 8 * kGroupThreads * sizeof(float);
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  const uint32_t s = tma::smem_u32(p);
  return p + ((1024u - (s & 1023u)) & 1023u);
}

// Producer side of the per-group rings: hands out items to whichever group
// has a free stage. next_item(t) maps ticket/slot t to an Item; issue(it, dst,
// bar) starts its TMA loads.
template <int NG, int NSG, class Next, class Issue>
__device__ __forceinline__ void produce(Ctl* ctl, uint8_t* ring, int stage_bytes, Next next_item, Issue issue) {
  produce<NG, NSG>(ctl, ring, stage_bytes, next_item, issue, [] {});
}

// As above; an item of kind kBarrier is not issued: the producer waits until
// every stage issued so far has been released by its consumers, then runs
// on_barrier() and continues with the following items.
template <int NG, int NSG, class Next, class Issue, class Barrier>
__device__ __forceinline__ void produce(Ctl* ctl, uint8_t* ring, int stage_bytes, Next next_item, Issue issue,
                                        Barrier on_barrier) {
  int head[NG];
  bool ended[NG];
#pragma unroll
  for (int g = 0; g < NG; ++g) {
    head[g] = 0;
    ended[g] = false;
  }
  int ends = 0;
  uint32_t spins = 0;
  uint64_t t0 = 0;
  while (ends < NG) {
    bool any = false;
#pragma unroll
    for (int g = 0; g < NG; ++g) {
      if (ended[g]) continue;
      const int k = head[g] % NSG, use = head[g] / NSG;
      if (use >= 1 && !tma::mbar_test_wait(&ctl->empty[g][k], (uint32_t)(use - 1) & 1u)) continue;
      Item it = next_item();
      if (it.kind == kBarrier) {
        // drain: the last use of every stage of every group has been released
#pragma unroll
        for (int gg = 0; gg < NG; ++gg)
          for (int kk = 0; kk < NSG; ++kk) {
            const int uses = head[gg] / NSG + (kk < head[gg] % NSG ? 1 : 0);
            if (uses >= 1) tma::mbar_wait(&ctl->empty[gg][kk], (uint32_t)(uses - 1) & 1u);
          }
        on_barrier();
        it = next_item();
      }
      ctl->items[g][k] = it;
      ++head[g];
      any = true;
      if (it.kind == kEnd) {
        tma::mbar_arrive(&ctl->full[g][k]);
        ended[g] = true;
        ++ends;
        continue;
      }
      issue(it, ring + (g * NSG + k) * stage_bytes, &ctl->full[g][k]);
    }
    if (!any) {
      __nanosleep(32);
      tma::watchdog(spins, t0);  // traps only after ~10 s without progress
    } else {
      spins = 0;
      t0 = 0;
    }
  }
}

// ---------------------------------------------------------------------------
// encode kernel
// ---------------------------------------------------------------------------
template <int D, typename TIn, bool SYM, bool SIGN>
__global__ void __launch_bounds__(kEncThreads, 1) enc_kernel(const __grid_constant__ EncArgs a) {
  using P = EncPlan<(int)sizeof(TIn)>;
  using TL = Tile<D, (int)sizeof(TIn), enc_chunk<TIn>()>;
  constexpr int NG = P::NG, NSG = P::NSG;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = align1024(smem_raw);
  Ctl* ctl = reinterpret_cast<Ctl*>(ring + NG * NSG * P::STAGE);
  uint8_t* replay_base = reinterpret_cast<uint8_t*>(ctl + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int g = 0; g < NG; ++g)
      for (int k = 0; k < NSG; ++k) {
        tma::mbar_init(&ctl->full[g][k], 1);
        tma::mbar_init(&ctl->empty[g][k], kWarpsPerGroup);  // every warp releases
      }
    tma::fence_mbar_init();
  }
  if (threadIdx.x < kMaxL) {
    ctl->ready[threadIdx.x] = 0;
    ctl->cta_max[threadIdx.x] = 0;
    ctl->cta_cnt[threadIdx.x] = 0;
  }
  if (a.k_max_ext && threadIdx.x < a.num_layers) ctl->layer_max[threadIdx.x] = a.k_max_ext[threadIdx.x];
  if (threadIdx.x < kMaxGroups * kMaxSG * 2) {
    (&ctl->gmax[0][0][0])[threadIdx.x] = 0;
    (&ctl->gcnt[0][0][0])[threadIdx.x] = 0;
  }
  __syncthreads();
  // Role split. SMs that share instruction caches (neighbouring SMs) should
  // run the same code path, so each role takes a contiguous range of blocks
  // (PKV_ROLE_MAP=1: of SM ids; the grid is one CTA per SM, so %smid is a
  // permutation of 0..grid-1). Ranks are dense within each role.
  unsigned pos = blockIdx.x;
#if PKV_ROLE_MAP == 1
  asm volatile("mov.u32 %0, %%smid;" : "=r"(pos));
  if (pos >= gridDim.x) pos = blockIdx.x;  // not a dense numbering: fall back to block order
#endif
  const bool value_role = pos < (unsigned)a.value_ctas;
  const long long role_rank = value_role ? (long long)pos : (long long)pos - a.value_ctas;

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol_first = tma::policy_evict_first(), pol_last = tma::policy_evict_last();
      auto issue = [&](const Item& it, uint8_t* dst, uint64_t* bar) {
        if (it.kind == kValEnc) {
          tma::mbar_arrive_expect_tx(bar, (uint32_t)P::STAGE);
          const int row0 = it.idx * TL::VR;
#pragma unroll 1
          for (int rb = 0; rb < TL::NRB; ++rb)
#pragma unroll 1
            for (int cb = 0; cb < TL::NCB; ++cb)
              tma::tensor2d_g2s(dst + (rb * TL::NCB + cb) * TL::BOX_BYTES, &a.tm_v[it.layer],
                                cb * (TL::IB / (int)sizeof(TIn)), row0 + rb * TL::BR, bar, pol_first);
        } else {
          // absmax reads keep the keys in L2 for the key-encode phase
          constexpr int kEncChunk = enc_chunk<TIn>();
          const long long e0 = (long long)it.idx * kEncChunk;
          const uint32_t bytes = (uint32_t)(min((long long)kEncChunk, a.nelem - e0) * (long long)sizeof(TIn));
          if (a.dbg == 5 && it.kind == kKeyEnc) {  // timing experiment: no L2 re-read (wrong codes)
            tma::mbar_arrive(bar);
            return;
          }
          tma::mbar_arrive_expect_tx(bar, bytes);
          tma::bulk_g2s(dst, static_cast<const TIn*>(a.k_in[it.layer]) + e0, bytes, bar,
                        it.kind == kAbsmax ? pol_last : pol_first);
        }
      };
      if (value_role && a.abs_lead > 0 && a.nA > 0) {
        // The value CTAs are ALU-bound and their memory pipe is mostly idle:
        // they also stream the per-tensor absmax items (HBM reads kept in L2
        // with evict_last for the key encode), abs_lead layers ahead of their
        // value cursor, so the key CTAs only run the encode pass (L2 re-read).
        const long long G = a.value_ctas, totV = (long long)a.num_layers * a.nV;
        const long long totA = (long long)a.num_layers * a.nA;
        long long tv = role_rank, ta = role_rank;
        auto next_item = [&]() -> Item {
          const bool a_ok = ta < totA;
          if (a_ok && (tv >= totV || ta / a.nA <= tv / a.nV + a.abs_lead)) {
            const int l = (int)(ta / a.nA);
            const Item it{kAbsmax, l, (int)(ta - (long long)l * a.nA), 0};
            ta += G;
            return it;
          }
          if (tv >= totV) return Item{kEnd, 0, 0, 0};
          const Item it = enc_value_item_at(a, tv);
          tv += G;
          return it;
        };
        produce<NG, NSG>(ctl, ring, P::STAGE, next_item, issue);
      } else if (value_role) {
        const long long G = a.value_ctas, total = (long long)a.num_layers * a.nV;
        long long t = role_rank;
        auto next_item = [&]() -> Item {
          if (t >= total) return Item{kEnd, 0, 0, 0};
          const Item it = enc_value_item_at(a, t);
          t += G;
          return it;
        };
        produce<NG, NSG>(ctl, ring, P::STAGE, next_item, issue);
      } else if (a.nA == 0 || !kKeyDynamic) {
        const long long G = (long long)gridDim.x - a.value_ctas;
        const long long total = (long long)a.nseg * a.nE;
        long long t = role_rank;
        auto next_item = [&]() -> Item {
          if (t >= total) return Item{kEnd, 0, 0, 0};
          const Item it = enc_key_item_at(a, t);
          t += G;
          return it;
        };
        produce<NG, NSG>(ctl, ring, P::STAGE, next_item, issue);
      } else {
        // Per-tensor keys, readiness-driven order: two cursors over this
        // CTA's slice of the absmax list A and the key-encode list E (both
        // layer-major, nA == nE items per layer). An E item of layer l is
        // issued only once every CTA's A(l) items are folded (layer_done[l]),
        // after the producer has staged layer_max[l] in shared memory, so no
        // consumer ever holds a stage waiting for a scale; while layer l is
        // not ready the producer issues absmax items instead, at most `lag`
        // layers ahead of the encode cursor (L2 footprint).
        // (32-bit cursors: the host caps a launch at 2^31 items; the layer
        // count of the encode cursor is polled without blocking: the load
        // issued at one call is consumed at the next, so its L2 round trip
        // overlaps the TMA issue in between)
        const uint32_t G = gridDim.x - (uint32_t)a.value_ctas;
        const uint32_t nA = (uint32_t)a.nA, nE = (uint32_t)a.nE;
        // (absmax on the value CTAs: this role only encodes, waiting on layer_done)
        const uint32_t totA = a.abs_lead > 0 ? 0u : (uint32_t)a.num_layers * nA;
        const uint32_t totE = (uint32_t)a.num_layers * nE;
        uint32_t ta = (uint32_t)role_rank, te = (uint32_t)role_rank;
        int ready = -1;      // layers [0, ready] staged in ctl->layer_max
        int polled = -1;     // layer whose count is in `polled_cnt`
        uint32_t polled_cnt = 0;
        int pending = -1;    // layer whose max is in flight in `pending_max`
        uint32_t pending_max = 0;
        // Every global read here is RELAXED and consumed one call later, so
        // its L2 round trip overlaps the TMA issues in between (an ld.acquire
        // holds back the bulk copies issued after it). Acquire ordering is
        // established once per layer: a
        // relaxed read that sees the complete count (written with
        // red.release) followed by fence.acq_rel, then the max is read.
        auto stage = [&](int l, uint32_t mx) {
          ctl->layer_max[l] = mx;
          __threadfence_block();
          *reinterpret_cast<volatile uint32_t*>(&ctl->ready[l]) = 1u;
          ready = l;
        };
        auto request_max = [&](int l) {
          fence_acq_rel_gpu();
          pending_max = ld_relaxed_u32(a.layer_max + l);  // consumed at the next call
          pending = l;
        };
        auto next_item = [&]() -> Item {
          for (;;) {
            if (te >= totE) return Item{kEnd, 0, 0, 0};
            const int el = (int)(te / nE);
            if (el <= ready) {
              const Item it{kKeyEnc, el, (int)(te - (uint32_t)el * nE), 0};
              te += G;
              return it;
            }
            if (pending == el) {
              stage(el, pending_max);
              continue;
            }
            if (polled == el && polled_cnt >= (uint32_t)a.abs_target) {
              request_max(el);
            } else {
              polled = el;
              polled_cnt = ld_relaxed_u32(a.layer_done + el);  // consumed at the next call
            }
            if (ta < totA && (int)(ta / nA) < el + a.key_lag) {
              const int al = (int)(ta / nA);
              const Item it{kAbsmax, al, (int)(ta - (uint32_t)al * nA), 0};
              ta += G;
              return it;
            }
            if (pending != el) {  // nothing else to issue: wait for layer el's absmax items
              uint32_t spins = 0;
              uint64_t t0 = 0;
              while (ld_relaxed_u32(a.layer_done + el) < (uint32_t)a.abs_target) {
                __nanosleep(128);
                tma::watchdog(spins, t0);
              }
              request_max(el);
            }
            stage(el, pending_max);
          }
        };
        produce<NG, NSG>(ctl, ring, P::STAGE, next_item, issue);
      }
    }
    return;
  }

  // ---------------- consumers (warps work independently) ----------------
  // rank of this CTA among the CTAs that issue absmax items
  const uint32_t abs_rank = a.abs_lead > 0 ? (uint32_t)pos : (uint32_t)pos - (uint32_t)a.value_ctas;
  const int g = (warp - 1) / kWarpsPerGroup;
  const int wig = (warp - 1) % kWarpsPerGroup;
  const int gt = threadIdx.x - 32 - g * kGroupThreads;
  double* R = reinterpret_cast<double*>(replay_base) + (warp - 1) * D;
  uint8_t* C = replay_base + NG * kWarpsPerGroup * D * 8 + (warp - 1) * D;
  for (int n = 0;; ++n) {
    const int k = n % NSG;
    tma::mbar_wait(&ctl->full[g][k], (uint32_t)(n / NSG) & 1u);
    const Item it = ctl->items[g][k];
    if (it.kind == kEnd) break;
    const uint32_t in_s = tma::smem_u32(ring + (g * NSG + k) * P::STAGE);
    const bool skip = a.dbg == 1 || (a.dbg == 2 && it.kind == kValEnc) || (a.dbg == 3 && it.kind != kValEnc);
    bool released = false;
    auto release = [&]() {
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&ctl->empty[g][k]);
    };
    if (it.kind == kAbsmax) {
      const uint32_t m = skip ? 0u : enc_absmax_item<TIn, enc_chunk<TIn>(), kGroupThreads>(a, it, in_s, gt);
      release();  // the stage refills while the fold / publish below runs
      released = true;
      if (lane == 0) {
        // fold the group's warps; the last one publishes the item
        const int par = (n / NSG) & 1;
        atomicMax(&ctl->gmax[g][k][par], m);
        __threadfence_block();
        if (atomicAdd(&ctl->gcnt[g][k][par], 1u) == kWarpsPerGroup - 1) {
          const uint32_t gm = atomicExch(&ctl->gmax[g][k][par], 0u);
          ctl->gcnt[g][k][par] = 0;
          fold_absmax(a, ctl, it.layer, gm, abs_rank);
        }
      }
    } else if (skip) {
    } else if (it.kind == kKeyEnc) {
      if (a.nA && a.dbg != 4) {  // per-tensor scale: every absmax item of the layer must be in
        if (lane == 0 && !*reinterpret_cast<volatile const uint32_t*>(&ctl->ready[it.layer])) {
          uint32_t spins = 0;
          uint64_t t0 = 0;
          while (ld_acquire_u32(a.layer_done + it.layer) < (uint32_t)a.abs_target) {
            __nanosleep(64);
            tma::watchdog(spins, t0);
          }
          ctl->layer_max[it.layer] = *reinterpret_cast<volatile const uint32_t*>(a.layer_max + it.layer);
          __threadfence_block();
          *reinterpret_cast<volatile uint32_t*>(&ctl->ready[it.layer]) = 1u;
        }
        __threadfence_block();
        __syncwarp();
      }
      enc_key_item<TIn, enc_chunk<TIn>(), kGroupThreads>(a, it, in_s, gt, lane, ctl->layer_max, release, released);
    } else {
      enc_value_item<D, TIn, SYM, SIGN, enc_chunk<TIn>(), kWarpsPerGroup>(a, it, in_s, wig, lane, R, C);
    }
    if (!released) release();  // this warp is done with the stage
  }
}

// ---------------------------------------------------------------------------
// encode kernel, co-resident roles (every SM runs values AND keys)
// ---------------------------------------------------------------------------
// The role-split enc_kernel pays the SM-time of both roles in sequence: the
// value role is bound by instruction issue (register reads) and the key role
// by memory latency, on disjoint SMs. Here every CTA (one per SM) runs both,
// on different SM sub-partitions so that no SMSP's L0 instruction cache holds
// both code paths (warp w issues on SMSP w % 4; mixing the two paths on one
// SMSP thrashed it, 33% no_instructions):
//   group g = SMSP g: warps {g, g + 4, g + 8} (warp 0 is the TMA producer,
//   so group 0 is warps 4, 8, 12);
//   groups 0-2: value items, group 3: absmax + key-encode items.
// The key group's memory latency hides under the value groups' ALU work.
// Items: bf16 12288 / f32 6144 elements (24 KB stages, two per group); a
// value item is two (d=128) passes of the group's three warps.
constexpr int kCoWPG = 3;
constexpr int kCoGT = 32 * kCoWPG;
constexpr int kCoGroups = 4;
constexpr int kCoThreads = 32 + kCoGroups * kCoGT;  // 416: 13 warps
constexpr int kCoStage = 24 * 1024;
constexpr int kCoNSG = 2;
template <typename TIn>
constexpr int co_chunk() {
  return kCoStage / (int)sizeof(TIn);
}
inline int co_chunk_for(int elem_bytes) { return kCoStage / elem_bytes; }

template <int D>
constexpr size_t co_smem_bytes() {
  return 1024 + (size_t)kCoGroups * kCoNSG * kCoStage + sizeof(Ctl) + (size_t)12 * (D * 8 + D);
}

template <int D, typename TIn, bool SYM, bool SIGN>
__global__ void __launch_bounds__(kCoThreads, 1) enc_co_kernel(const __grid_constant__ EncArgs a) {
  constexpr int CH = co_chunk<TIn>();
  using TL = Tile<D, (int)sizeof(TIn), CH, kCoWPG>;
  constexpr int NG = kCoGroups, NSG = kCoNSG;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = align1024(smem_raw);
  Ctl* ctl = reinterpret_cast<Ctl*>(ring + NG * NSG * kCoStage);
  uint8_t* replay_base = reinterpret_cast<uint8_t*>(ctl + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int g = 0; g < NG; ++g)
      for (int k = 0; k < NSG; ++k) {
        tma::mbar_init(&ctl->full[g][k], 1);
        tma::mbar_init(&ctl->empty[g][k], kCoWPG);  // every warp of the group releases
      }
    tma::fence_mbar_init();
  }
  if (threadIdx.x < kMaxL) {
    ctl->ready[threadIdx.x] = 0;
    ctl->cta_max[threadIdx.x] = 0;
    ctl->cta_cnt[threadIdx.x] = 0;
  }
  if (a.k_max_ext && threadIdx.x < a.num_layers) ctl->layer_max[threadIdx.x] = a.k_max_ext[threadIdx.x];
  if (threadIdx.x < kMaxGroups * kMaxSG * 2) {
    (&ctl->gmax[0][0][0])[threadIdx.x] = 0;
    (&ctl->gcnt[0][0][0])[threadIdx.x] = 0;
  }
  __syncthreads();
  // role of group g: true = values
  auto value_group = [&](int g) { return a.co_roles == 1 || (a.co_roles == 0 && g < 3); };

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_first = tma::policy_evict_first(), pol_last = tma::policy_evict_last();
      auto issue = [&](const Item& it, uint8_t* dst, uint64_t* bar) {
        if (it.kind == kValEnc) {
          tma::mbar_arrive_expect_tx(bar, (uint32_t)(CH * (int)sizeof(TIn)));
          const int row0 = it.idx * TL::VR;
#pragma unroll 1
          for (int rb = 0; rb < TL::NRB; ++rb)
#pragma unroll 1
            for (int cb = 0; cb < TL::NCB; ++cb)
              tma::tensor2d_g2s(dst + (rb * TL::NCB + cb) * TL::BOX_BYTES, &a.tm_v[it.layer],
                                cb * (TL::IB / (int)sizeof(TIn)), row0 + rb * TL::BR, bar, pol_first);
        } else {
          const long long e0 = (long long)it.idx * CH;
          const uint32_t bytes = (uint32_t)(min((long long)CH, a.nelem - e0) * (long long)sizeof(TIn));
          tma::mbar_arrive_expect_tx(bar, bytes);
          tma::bulk_g2s(dst, static_cast<const TIn*>(a.k_in[it.layer]) + e0, bytes, bar,
                        it.kind == kAbsmax ? pol_last : pol_first);
        }
      };
      // ---- value cursor: this CTA's static slice of the layer-major V list ----
      const long long G = gridDim.x;
      const long long totV = (long long)a.num_layers * a.nV;
      long long tv = blockIdx.x;
      auto next_value = [&]() -> Item {
        if (tv >= totV) return Item{kEnd, 0, 0, 0};
        const Item it = enc_value_item_at(a, tv);
        tv += G;
        return it;
      };
      // ---- key cursor: absmax items A and key-encode items E (see enc_kernel);
      // never blocks (returns kNone), so the value groups keep being fed ----
      const uint32_t GK = gridDim.x;
      const uint32_t nA = (uint32_t)a.nA, nE = (uint32_t)a.nE;
      const uint32_t totA = (uint32_t)a.num_layers * nA, totE = (uint32_t)a.num_layers * nE;
      uint32_t ta = blockIdx.x, te = blockIdx.x;
      int ready = -1, polled = -1, pending = -1;
      uint32_t polled_cnt = 0, pending_max = 0;
      const bool tensor_keys = nA > 0;
      auto next_key = [&]() -> Item {
        for (;;) {
          if (te >= totE) return Item{kEnd, 0, 0, 0};
          const int el = (int)(te / nE);
          if (!tensor_keys || el <= ready) {
            const Item it{kKeyEnc, el, (int)(te - (uint32_t)el * nE), 0};
            te += GK;
            return it;
          }
          if (pending == el) {
            ctl->layer_max[el] = pending_max;
            __threadfence_block();
            *reinterpret_cast<volatile uint32_t*>(&ctl->ready[el]) = 1u;
            ready = el;
            continue;
          }
          if (polled == el && polled_cnt >= (uint32_t)a.abs_target) {
            fence_acq_rel_gpu();
            pending_max = ld_relaxed_u32(a.layer_max + el);  // staged at the next call
            pending = el;
          } else {
            polled = el;
            polled_cnt = ld_relaxed_u32(a.layer_done + el);  // consumed at the next call
          }
          if (ta < totA && (int)(ta / nA) < el + a.key_lag) {
            const int al = (int)(ta / nA);
            const Item it{kAbsmax, al, (int)(ta - (uint32_t)al * nA), 0};
            ta += GK;
            return it;
          }
          return Item{kNone, 0, 0, 0};
        }
      };
      // ---- per-group rings; kNone = nothing for this group right now ----
      int head[NG];
      bool ended[NG];
#pragma unroll
      for (int g = 0; g < NG; ++g) {
        head[g] = 0;
        ended[g] = false;
      }
      int ends = 0;
      uint32_t spins = 0;
      uint64_t t0 = 0;
      while (ends < NG) {
        bool any = false;
#pragma unroll
        for (int g = 0; g < NG; ++g) {
          if (ended[g]) continue;
          const int k = head[g] % NSG, use = head[g] / NSG;
          if (use >= 1 && !tma::mbar_test_wait(&ctl->empty[g][k], (uint32_t)(use - 1) & 1u)) continue;
          Item it;
          if (value_group(g)) {
            it = next_value();
          } else {
            it = next_key();
            if (it.kind == kNone) continue;
          }
          ctl->items[g][k] = it;
          ++head[g];
          any = true;
          if (it.kind == kEnd) {
            tma::mbar_arrive(&ctl->full[g][k]);
            ended[g] = true;
            ++ends;
            continue;
          }
          issue(it, ring + (g * NSG + k) * kCoStage, &ctl->full[g][k]);
        }
        if (!any) {
          __nanosleep(32);
          tma::watchdog(spins, t0);  // traps only after ~10 s without progress
        } else {
          spins = 0;
          t0 = 0;
        }
      }
    }
    return;
  }

  // ---------------- consumers: group = SMSP ----------------
  const int g = warp & 3;
  const int wig = (warp - 1) >> 2;  // 0..2 (warp 4 -> 0 for group 0)
  const int gt = wig * 32 + lane;
  double* R = reinterpret_cast<double*>(replay_base) + (warp - 1) * D;
  uint8_t* C = replay_base + 12 * D * 8 + (warp - 1) * D;
  for (int n = 0;; ++n) {
    const int k = n % NSG;
    tma::mbar_wait(&ctl->full[g][k], (uint32_t)(n / NSG) & 1u);
    const Item it = ctl->items[g][k];
    if (it.kind == kEnd) break;
    const uint32_t in_s = tma::smem_u32(ring + (g * NSG + k) * kCoStage);
    bool released = false;
    auto release = [&]() {
      __syncwarp();
      if (lane == 0) tma::mbar_arrive(&ctl->empty[g][k]);
    };
    if (it.kind == kAbsmax) {
      const uint32_t m = enc_absmax_item<TIn, CH, kCoGT>(a, it, in_s, gt);
      release();
      released = true;
      if (lane == 0) {
        const int par = (n / NSG) & 1;
        atomicMax(&ctl->gmax[g][k][par], m);
        __threadfence_block();
        if (atomicAdd(&ctl->gcnt[g][k][par], 1u) == kCoWPG - 1) {
          const uint32_t gm = atomicExch(&ctl->gmax[g][k][par], 0u);
          ctl->gcnt[g][k][par] = 0;
          fold_absmax(a, ctl, it.layer, gm, blockIdx.x);
        }
      }
    } else if (it.kind == kKeyEnc) {
      enc_key_item<TIn, CH, kCoGT>(a, it, in_s, gt, lane, ctl->layer_max, release, released);
    } else {
      enc_value_item<D, TIn, SYM, SIGN, CH, kCoWPG>(a, it, in_s, wig, lane, R, C);
    }
    if (!released) release();
  }
}

// ---------------------------------------------------------------------------
// decode kernel
// ---------------------------------------------------------------------------
template <int D, typename TOut, bool SIGN, bool B32>
__global__ void __launch_bounds__(threads_for<dec_groups<TOut>()>(), 1) dec_kernel(const __grid_constant__ DecArgs a) {
  using P = DecPlan<(int)sizeof(TOut), dec_groups<TOut>()>;
  using TL = Tile<D, (int)sizeof(TOut), kDecChunk>;
  constexpr int NG = P::NG, NSG = P::NSG;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* obuf = align1024(smem_raw);  // 1024-aligned swizzled output tiles
  uint8_t* base4k = smem_raw + ((4096u - (tma::smem_u32(smem_raw) & 4095u)) & 4095u);
  obuf = base4k;                         // 4 KB aligned (>= the 1 KB swizzle alignment)
  float* tables = reinterpret_cast<float*>(obuf + P::OUT_TOTAL);  // 4 KB aligned per group
  uint8_t* ring = obuf + P::OUT_TOTAL + P::NG * 8 * kGroupThreads * sizeof(float);
  Ctl* ctl = reinterpret_cast<Ctl*>(ring + NG * NSG * P::STAGE);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int g = 0; g < NG; ++g)
      for (int k = 0; k < NSG; ++k) {
        tma::mbar_init(&ctl->full[g][k], 1);
        tma::mbar_init(&ctl->empty[g][k], 1);
      }
    tma::fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_first = tma::policy_evict_first();
      // static slice of the item list per CTA; within the CTA items go to
      // whichever group frees a stage first. With a role split (key_ctas >
      // 0) each SM runs one code path: key CTAs stream the (HBM-bound) key
      // items of every layer, value CTAs the (ALU-bound) value items, and
      // the two overlap instead of alternating on every SM.
      const int vctas = a.key_ctas > 0 ? (int)gridDim.x - a.key_ctas : (int)gridDim.x;
      const bool key_role = a.key_ctas > 0 && (int)blockIdx.x >= vctas;
      const long long G = a.key_ctas > 0 ? (key_role ? a.key_ctas : vctas) : (long long)gridDim.x;
      const long long per = key_role ? a.nK : a.nV;
      const long long total = a.key_ctas > 0 ? (long long)a.num_layers * per : (long long)a.total;
      long long t = key_role ? (long long)blockIdx.x - vctas : (long long)blockIdx.x;
      auto next_item = [&]() -> Item {
        if (t >= total) return Item{kEnd, 0, 0, 0};
        Item it;
        if (a.key_ctas > 0) {
          const int l = (int)(t / per);
          it = Item{key_role ? kKeyDec : kValDec, l, (int)(t - (long long)l * per), 0};
        } else {
          it = dec_item(a, (unsigned int)t);
        }
        t += G;
        return it;
      };
      auto issue = [&](const Item& it, uint8_t* in, uint64_t* bar) {
        if (it.kind == kKeyDec) {
          const long long e0 = (long long)it.idx * kDecChunk;
          const uint32_t bytes = (uint32_t)min((long long)kDecChunk, a.nelem - e0);
          // block32: the item's fp16 scales follow the codes (whole 16-byte units;
          // a ragged last unit is read from global memory by the consumer)
          const uint32_t sb = B32 ? ((bytes + 31) / 32 * 2) & ~15u : 0u;
          tma::mbar_arrive_expect_tx(bar, bytes + sb);
          tma::bulk_g2s(in, a.k_codes[it.layer] + e0, bytes, bar, pol_first);
          if (sb) tma::bulk_g2s(in + kDecChunk, a.k_bscale[it.layer] + (e0 >> 5), sb, bar, pol_first);
        } else {
          const long long v0 = (long long)it.idx * TL::VR;
          const int nv = (int)min((long long)TL::VR, a.nvec - v0);
          const uint32_t pb = (uint32_t)(nv * VL<D>::PB) & ~15u, sb = (uint32_t)(nv * 4) & ~15u;
          tma::mbar_arrive_expect_tx(bar, pb + sb);
          if (pb) tma::bulk_g2s(in, a.v_packed[it.layer] + v0 * VL<D>::PB, pb, bar, pol_first);
          if (sb) tma::bulk_g2s(in + 3 * kDecChunk / 8, a.v_scales[it.layer] + v0, sb, bar, pol_first);
        }
      };
      produce<NG, NSG>(ctl, ring, P::STAGE, next_item, issue);
    }
    return;
  }

  const int g = (warp - 1) / kWarpsPerGroup;
  const int wig = (warp - 1) % kWarpsPerGroup;
  const int gt = threadIdx.x - 32 - g * kGroupThreads;
  float* tbl = tables + g * 8 * kGroupThreads;
  for (int n = 0;; ++n) {
    const int k = n % NSG;
    tma::mbar_wait(&ctl->full[g][k], (uint32_t)(n / NSG) & 1u);
    const Item it = ctl->items[g][k];
    if (it.kind == kEnd) break;
    uint8_t* in = ring + (g * NSG + k) * P::STAGE;
    uint8_t* out = obuf + (g * P::NOB + (n & 1)) * P::OUT;
    int nv = 0;
    long long v0 = 0;
    if (it.kind == kKeyDec) {
      if constexpr (B32) dec_key_item_b32<TOut>(a, it, tma::smem_u32(in), out, gt);
      else dec_key_item<TOut, false>(a, it, tma::smem_u32(in), out, gt);
    } else {
      v0 = (long long)it.idx * TL::VR;
      nv = (int)min((long long)TL::VR, a.nvec - v0);
      dec_value_item<D, TOut, SIGN>(a, it, in, (nv * VL<D>::PB) & ~15, (nv * 4) & ~15, out, tbl, gt, wig, lane);
    }
    tma::fence_proxy_async_smem();
    if (gt == 0) tma::bulk_wait_read<0>();  // the store of the previous item has left the other buffer
    tma::named_bar_sync(1 + g, kGroupThreads);
    if (gt == 0) {
      tma::mbar_arrive(&ctl->empty[g][k]);  // inputs consumed
      if (it.kind == kKeyDec) {
        const long long e0 = (long long)it.idx * kDecChunk;
        const int bytes = (int)min((long long)kDecChunk, a.nelem - e0) * (int)sizeof(TOut);
        tma::bulk_s2g(static_cast<TOut*>(a.k_out[it.layer]) + e0, out, (uint32_t)bytes);
      } else {
#pragma unroll 1
        for (int rb = 0; rb < TL::NRB; ++rb) {
          if (rb * TL::BR >= nv) break;
#pragma unroll 1
          for (int cb = 0; cb < TL::NCB; ++cb)
            tma::tensor2d_s2g(&a.tm_v[it.layer], cb * (TL::IB / (int)sizeof(TOut)), (int)(v0 + rb * TL::BR),
                              out + (rb * TL::NCB + cb) * TL::BOX_BYTES);
        }
      }
      tma::bulk_commit();
    }
  }
  if (gt == 0) tma::bulk_wait<0>();
}

}  // namespace stream
}  // namespace pkv

// ===========================================================================
// host side
// ===========================================================================
#include "stream_codec.h"
#include "tuning.h"

namespace pkv {
namespace stream {
namespace {

PFN_cuTensorMapEncodeTiled_v12000 encode_fn() {
  static PFN_cuTensorMapEncodeTiled_v12000 fn = nullptr;
  static std::once_flag once;
  std::call_once(once, [] {
    void* p = nullptr;
    cudaDriverEntryPointQueryResult q;
    if (cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &p, cudaEnableDefault, &q) == cudaSuccess &&
        q == cudaDriverEntryPointSuccess)
      fn = reinterpret_cast<PFN_cuTensorMapEncodeTiled_v12000>(p);
  });
  return fn;
}

// cuTensorMapEncodeTiled is a driver call and needs a current context. A
// host thread that has made no context-binding runtime call yet (a fresh
// Python thread reading the pool) has none: CUDA_ERROR_INVALID_CONTEXT.
// cudaFree(nullptr) binds the current device's primary context, once per
// thread and device.
bool bind_context() {
  static thread_local int bound = -1;
  int dev = 0;
  if (!pkv::cuda_ok(cudaGetDevice(&dev), "cudaGetDevice")) return false;
  if (bound == dev) return true;
  if (!pkv::cuda_ok(cudaFree(nullptr), "cudaFree(nullptr) (bind the primary context)")) return false;
  bound = dev;
  return true;
}

// [nvec, D] head-vector tensor of one layer as a 2-D TMA map with the box
// geometry of Tile<D, eb>.
bool make_map(CUtensorMap* m, const void* base, int eb, int D, long long nvec, int chunk) {
  if (!bind_context()) return false;
  auto fn = encode_fn();
  if (!fn) {
    pkv::driver_fail(-1, "cudaGetDriverEntryPoint(cuTensorMapEncodeTiled)");
    return false;
  }
  const int RB = D * eb, IB = RB < 128 ? RB : 128, VR = chunk / D, BR = VR / ((VR + 255) / 256);  // == Tile::BR
  cuuint64_t dims[2] = {(cuuint64_t)D, (cuuint64_t)nvec};
  cuuint64_t strides[1] = {(cuuint64_t)RB};
  cuuint32_t box[2] = {(cuuint32_t)(IB / eb), (cuuint32_t)BR};
  cuuint32_t estr[2] = {1, 1};
  const CUtensorMapSwizzle sw = IB == 128 ? CU_TENSOR_MAP_SWIZZLE_128B
                                : IB == 64 ? CU_TENSOR_MAP_SWIZZLE_64B
                                : IB == 32 ? CU_TENSOR_MAP_SWIZZLE_32B
                                           : CU_TENSOR_MAP_SWIZZLE_NONE;
  const CUresult r = fn(m, eb == 2 ? CU_TENSOR_MAP_DATA_TYPE_BFLOAT16 : CU_TENSOR_MAP_DATA_TYPE_FLOAT32, 2,
                        const_cast<void*>(base), dims, strides, box, estr, CU_TENSOR_MAP_INTERLEAVE_NONE, sw,
                        CU_TENSOR_MAP_L2_PROMOTION_L2_256B, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
  if (r != CUDA_SUCCESS) pkv::driver_fail((int)r, "cuTensorMapEncodeTiled");
  return r == CUDA_SUCCESS;
}

template <typename K>
int coop_launch(K kernel, const void* args, size_t smem, int threads, cudaStream_t st) {
  if (!pkv::cuda_ok(cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
                    "cudaFuncSetAttribute"))
    return PKV_ERR_CUDA;
  int per_sm = 0;
  if (!pkv::cuda_ok(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, threads, smem),
                    "cudaOccupancyMaxActiveBlocksPerMultiprocessor"))
    return PKV_ERR_CUDA;
  if (per_sm < 1) {
    pkv::cuda_ok(cudaErrorInvalidConfiguration, "occupancy: the kernel does not fit an SM");
    return PKV_ERR_CUDA;
  }
  void* params[] = {const_cast<void*>(args)};
  const cudaError_t e =
      // one persistent CTA per SM (the role split and static slices assume it)
      cudaLaunchCooperativeKernel((const void*)kernel, dim3((unsigned)sm_count()), dim3(threads), params,
                                  smem, st);
  return pkv::cuda_ok(e, "cudaLaunchCooperativeKernel") ? PKV_OK : PKV_ERR_CUDA;
}

template <int D, typename TIn>
int enc_launch_d(const EncArgs& a, bool sym, bool sign, cudaStream_t st) {
  const size_t smem = enc_smem_bytes<D, TIn>();
  if (sym) {
    return sign ? coop_launch(enc_kernel<D, TIn, true, true>, &a, smem, kEncThreads, st)
                : coop_launch(enc_kernel<D, TIn, true, false>, &a, smem, kEncThreads, st);
  }
  return sign ? coop_launch(enc_kernel<D, TIn, false, true>, &a, smem, kEncThreads, st)
              : coop_launch(enc_kernel<D, TIn, false, false>, &a, smem, kEncThreads, st);
}

template <typename TIn>
int enc_launch(const EncArgs& a, int d, bool sym, bool sign, cudaStream_t st) {
  switch (d) {
    case 16: return enc_launch_d<16, TIn>(a, sym, sign, st);
    case 32: return enc_launch_d<32, TIn>(a, sym, sign, st);
    case 64: return enc_launch_d<64, TIn>(a, sym, sign, st);
    case 128: return enc_launch_d<128, TIn>(a, sym, sign, st);
    default: return PKV_ERR_UNSUPPORTED_HEAD_DIM;
  }
}

template <int D, typename TIn>
int co_launch_d(const EncArgs& a, bool sym, bool sign, cudaStream_t st) {
  const size_t smem = co_smem_bytes<D>();
  if (sym) {
    return sign ? coop_launch(enc_co_kernel<D, TIn, true, true>, &a, smem, kCoThreads, st)
                : coop_launch(enc_co_kernel<D, TIn, true, false>, &a, smem, kCoThreads, st);
  }
  return sign ? coop_launch(enc_co_kernel<D, TIn, false, true>, &a, smem, kCoThreads, st)
              : coop_launch(enc_co_kernel<D, TIn, false, false>, &a, smem, kCoThreads, st);
}

template <typename TIn>
int co_launch(const EncArgs& a, int d, bool sym, bool sign, cudaStream_t st) {
  switch (d) {
    case 64: return co_launch_d<64, TIn>(a, sym, sign, st);
    case 128: return co_launch_d<128, TIn>(a, sym, sign, st);
    default: return PKV_ERR_UNSUPPORTED_HEAD_DIM;
  }
}

template <int D, typename TOut>
int dec_launch_d(const DecArgs& a, bool sign, cudaStream_t st) {
  const size_t smem = dec_smem_bytes<TOut>();
  constexpr int T = threads_for<dec_groups<TOut>()>();
  if (a.k_mode == PKV_K_TENSOR)
    return sign ? coop_launch(dec_kernel<D, TOut, true, false>, &a, smem, T, st)
                : coop_launch(dec_kernel<D, TOut, false, false>, &a, smem, T, st);
  return sign ? coop_launch(dec_kernel<D, TOut, true, true>, &a, smem, T, st)
              : coop_launch(dec_kernel<D, TOut, false, true>, &a, smem, T, st);
}

template <typename TOut>
int dec_launch(const DecArgs& a, int d, bool sign, cudaStream_t st) {
  switch (d) {
    case 16: return dec_launch_d<16, TOut>(a, sign, st);
    case 32: return dec_launch_d<32, TOut>(a, sign, st);
    case 64: return dec_launch_d<64, TOut>(a, sign, st);
    case 128: return dec_launch_d<128, TOut>(a, sign, st);
    default: return PKV_ERR_UNSUPPORTED_HEAD_DIM;
  }
}

bool a16(const void* p) { return p == nullptr || aligned(p, 16); }

}  // namespace

bool head_dim_streamable(int d) { return d == 16 || d == 32 || d == 64 || d == 128; }

size_t workspace_bytes(int num_layers, long long num_vectors, int head_dim) {
  (void)num_vectors;
  (void)head_dim;
  const long long L = std::min(std::max(num_layers, 0), kMaxL);
  return (size_t)(L * 8 + 16);  // [u32 layer_max L][u32 layer_done L / key barrier]
}

int encode(const EncodeRequest& r, cudaStream_t st) {
  const int L = r.num_layers;
  if (L < 1 || L > kMaxL) return PKV_ERR_INVALID_ARG;
  const bool do_k = r.k_in != nullptr, do_v = r.v_in != nullptr;
  const int eb = r.in_dtype == PKV_F32 ? 4 : 2;
  const long long nelem = r.num_vectors * (long long)r.head_dim;
  if (!do_k && !do_v) return PKV_OK;
  if (do_v && !head_dim_streamable(r.head_dim)) return PKV_ERR_UNSUPPORTED_HEAD_DIM;
  if (nelem % 16 != 0 || r.num_vectors >= (1LL << 31)) return PKV_ERR_ALIGNMENT;
  EncArgs* a = new EncArgs;
  std::memset(a, 0, sizeof(EncArgs));
  a->num_layers = L;
  a->head_dim = r.head_dim;
  a->k_mode = r.k_mode;
  a->in_bytes = eb;
  a->nvec = r.num_vectors;
  a->nelem = nelem;
  a->delta = guard_delta(r.head_dim);
  a->cb = r.cb;
  std::memcpy(a->sign_bits, r.sign_bits, sizeof(a->sign_bits));
  a->status = r.status;
  a->replay_count = r.replay_count;
  // role-split kernel by default; PKV_ENC_ROLES=co selects the co-resident
  // one (head_dim 64 / 128), measured slower: C3 f32 507 vs 320 us, bf16 399
  // vs 253 us -- one 3-warp key group per SM keeps too few key bytes in
  // flight (48 KB) and the 3-warp value groups lose ~4%
  const bool co = tuning().enc_co && (!do_v || r.head_dim == 64 || r.head_dim == 128);
  const int kEncChunk = co ? co_chunk_for(eb) : enc_chunk_for(eb);
  const long long kch = (nelem + kEncChunk - 1) / kEncChunk;
  const long long vr = kEncChunk / std::max(r.head_dim, 1);
  a->nE = do_k ? (int)kch : 0;
  a->nV = do_v ? (int)((r.num_vectors + vr - 1) / vr) : 0;
  const long long total = (long long)L * (a->nE + a->nV);
  if (total >= (1LL << 31)) {
    delete a;
    return PKV_ERR_INVALID_ARG;
  }
  // workspace: [u32 layer_max L]
  unsigned int* w32 = reinterpret_cast<unsigned int*>(r.ws);
  a->total = (unsigned int)total;
  a->dbg = tuning().dbg_enc;
  a->layer_max = w32;
  const size_t ws_need = workspace_bytes(L, r.num_vectors, r.head_dim);
  if (r.ws_bytes < ws_need) {
    delete a;
    return PKV_ERR_ALIGNMENT;  // too small for this path: the caller falls back
  }
  int rc = PKV_OK;
  for (int l = 0; l < L && rc == PKV_OK; ++l) {
    if (do_k) {
      a->k_in[l] = r.k_in[l];
      a->k_codes[l] = r.k_codes[l];
      a->k_scale[l] = r.k_scale ? r.k_scale[l] : nullptr;
      a->k_bscale[l] = r.k_bscale ? reinterpret_cast<__half*>(r.k_bscale[l]) : nullptr;
      if (!a16(a->k_in[l]) || !a16(a->k_codes[l])) rc = PKV_ERR_ALIGNMENT;
    }
    if (do_v) {
      a->v_in[l] = r.v_in[l];
      a->v_packed[l] = r.v_packed[l];
      a->v_scales[l] = r.v_scales[l];
      if (!a16(a->v_in[l]) || !a16(a->v_packed[l]) || !a16(a->v_scales[l])) rc = PKV_ERR_ALIGNMENT;
      else if (!make_map(&a->tm_v[l], a->v_in[l], eb, r.head_dim, r.num_vectors, kEncChunk)) rc = PKV_ERR_CUDA;
    }
  }
  if (rc == PKV_OK && !pkv::cuda_ok(cudaMemsetAsync(r.ws, 0, ws_need, st), "cudaMemsetAsync")) rc = PKV_ERR_CUDA;
  // One launch; the grid is split by role so every SM runs a single code
  // path (mixing the key and value paths on one SM thrashes its instruction
  // cache): value CTAs are ALU-bound, key CTAs (absmax pass, key barrier,
  // key encode) are HBM-bound, and the two overlap.
  const int dk = do_v ? r.head_dim : 64;  // key-only launches never touch the value tile geometry
  if (rc == PKV_OK) {
    a->k_max_ext = r.k_max_ext;
    a->nA = (do_k && r.k_mode == PKV_K_TENSOR && !r.k_max_ext) ? a->nE : 0;
    a->layer_done = w32 + L;
    const int grid = sm_count();  // one CTA per SM (checked by the launcher)
    // key-role segment order (see enc_key_item_at)
    a->nseg = 0;
    if (a->nA) {
      // lag: enough layers that the key CTAs' in-flight stages (~3 rings per
      // CTA) cannot reach E(l) before every A(l) item has been consumed
      int lag = 4;
      if (tuning().key_lag > 0) lag = tuning().key_lag;
      a->key_lag = lag;
      for (int j = 0; j < L + lag; ++j) {
        if (j < L) {
          a->seg_absmax[a->nseg] = 1;
          a->seg_layer[a->nseg++] = (uint8_t)j;
        }
        if (j >= lag && j - lag < L) {
          a->seg_absmax[a->nseg] = 0;
          a->seg_layer[a->nseg++] = (uint8_t)(j - lag);
        }
      }
    } else if (do_k) {
      for (int l = 0; l < L; ++l) {
        a->seg_absmax[a->nseg] = 0;
        a->seg_layer[a->nseg++] = (uint8_t)l;
      }
    }
    // absmax items on the value CTAs (per-tensor keys with values in the launch)
    a->abs_lead = 0;
    if (a->nA && do_v && tuning().abs_on_values) a->abs_lead = 2;
    int key_ctas = 0;
    if (do_k && do_v) {
      // share of SMs for the key role, swept on C3 bf16 (tools/ab_frac.sh):
      // per-tensor 0.32 -> 343 us, 0.35 -> 287, 0.378 -> 269, 0.405 -> 278;
      // block32 (one key pass) 0.36 -> 336, 0.4 -> 302, 0.43 -> 285. The curve is not
      // smooth: SMs sharing instruction caches should run one role, so
      // where the role boundary falls matters. PKV_KEY_SM_FRACTION overrides
      // (d64, whose value path is cheaper: C2 0.35 -> 188 us, 0.42 -> 169, 0.46 -> 178)
      // (round 2, after the key fast-path change: C3 bf16 0.34 -> 253 us, 0.38 -> 261,
      // 0.42 -> 275; C3 f32 0.38 -> 365 us, 0.42 -> 335, 0.45 -> 327, 0.49 -> 350)
      const bool d128 = r.head_dim >= 128;
      // (per-CTA absmax publication, C3 f32: 56 key CTAs 324 us, 58 316, 60 308, 62 301.5, 64 306,
      // 66 315; bf16: 46 246, 48 237, 50 235, 52 240 -- profiles/r02/frac3.txt)
      // (C2, d64: f32 0.42 -> 220 us, 0.459 -> 198, 0.486 -> 190, 0.514 -> 197; bf16 0.338 -> 157,
      // 0.365 -> 147.5, 0.392 -> 152 -- frac_c2*.txt)
      // (after the neighbour-pair FWHT layout, C3 f32: 62 key CTAs 301.5 us, 64 294, 66 288.4, 68 294)
      // (after the word-level code XORs: C3 f32 66 -> 287.6 us, 68 -> 281.9, 70 -> 284; bf16 50 -> 229.8,
      // 52 -> 222.7, 54 -> 228; C2 f32 0.5 -> 187.5, 0.527 -> 181.7; bf16 0.365 -> 149, 0.392 -> 141.2)
      double frac = r.k_mode == PKV_K_TENSOR ? (d128 ? (eb == 4 ? 0.459 : 0.351) : (eb == 4 ? 0.527 : 0.392))
                                             : (d128 ? (eb == 4 ? 0.446 : 0.43) : 0.46);  // block32 C3 f32: 62 -> 268.5, 66 -> 264.6, 68 -> 269.2 us
      if (a->abs_lead > 0) frac = d128 ? 0.27 : 0.3;  // the key role only encodes
      if (tuning().key_sm_fraction >= 0.0) frac = tuning().key_sm_fraction;
      // an even count: the two SMs of a TPC must run the same role (an odd
      // split puts both code paths on one TPC, which thrashes and, with the
      // static partition, stalls the whole role: 53 key CTAs 290 us vs 52: 267)
      key_ctas = std::max(2, std::min(grid - 2, 2 * (int)std::lround(frac * grid / 2.0)));
    } else if (do_k) {
      key_ctas = grid;
    }
    a->value_ctas = grid - key_ctas;
    // which CTAs issue the absmax items (round-robin over the layer-major
    // list), and the layer_done count that completes a layer's max: one
    // publication per contributing CTA (fold_absmax), or per item for the
    // static key schedule
    a->abs_G = 0;
    a->abs_target = a->nA;
    if (a->nA) {
      const int G = co ? grid : a->abs_lead > 0 ? a->value_ctas : kKeyDynamic ? key_ctas : 0;
      if (G > 0) {
        a->abs_G = G;
        a->abs_target = std::min(G, a->nA);
      }
    }
    if (co) {
      a->co_roles = (do_k && do_v) ? 0 : (do_v ? 1 : 2);
      a->value_ctas = grid;
      a->abs_lead = 0;
      rc = eb == 4 ? co_launch<float>(*a, dk, r.cb.symmetric != 0, r.sign, st)
                   : co_launch<__nv_bfloat16>(*a, dk, r.cb.symmetric != 0, r.sign, st);
    } else {
      rc = eb == 4 ? enc_launch<float>(*a, dk, r.cb.symmetric != 0, r.sign, st)
                   : enc_launch<__nv_bfloat16>(*a, dk, r.cb.symmetric != 0, r.sign, st);
    }
  }
  delete a;
  return rc;
}

int decode(const DecodeRequest& r, cudaStream_t st) {
  const int L = r.num_layers;
  if (L < 1 || L > kMaxL) return PKV_ERR_INVALID_ARG;
  const bool do_k = r.k_codes != nullptr, do_v = r.v_packed != nullptr;
  const int eb = r.out_dtype == PKV_F32 ? 4 : 2;
  const long long nelem = r.num_vectors * (long long)r.head_dim;
  if (!do_k && !do_v) return PKV_OK;
  if (do_v && !head_dim_streamable(r.head_dim)) return PKV_ERR_UNSUPPORTED_HEAD_DIM;
  if (nelem % 16 != 0 || r.num_vectors >= (1LL << 31)) return PKV_ERR_ALIGNMENT;
  DecArgs* a = new DecArgs;
  std::memset(a, 0, sizeof(DecArgs));
  a->num_layers = L;
  a->head_dim = r.head_dim;
  a->k_mode = r.k_mode;
  a->out_bytes = eb;
  a->nvec = r.num_vectors;
  a->nelem = nelem;
  a->sqrt_d32 = (float)std::sqrt((double)r.head_dim);  // np.float32(np.sqrt(d))
  a->rcp_sqrt_d32 = 1.0f / a->sqrt_d32;
  std::memcpy(a->sign_bits, r.sign_bits, sizeof(a->sign_bits));
  std::memcpy(a->cent32, r.cent32, sizeof(a->cent32));
  const long long kch = (nelem + kDecChunk - 1) / kDecChunk;
  const long long vr = kDecChunk / std::max(r.head_dim, 1);
  a->nK = do_k ? (int)kch : 0;
  a->nV = do_v ? (int)((r.num_vectors + vr - 1) / vr) : 0;
  const long long total = (long long)L * (a->nK + a->nV);
  if (total >= (1LL << 32) - (1LL << 20)) {
    delete a;
    return PKV_ERR_INVALID_ARG;
  }
  a->total = (unsigned int)total;
  a->key_ctas = 0;
  if (do_k && do_v) {
    // share of SMs for the key role, swept with tools/dec_frac.sh: C3 (d128)
    // 0 (interleaved items) -> 180 us, 0.3 -> 164, 0.35 -> 140, 0.39 -> 147;
    // C2 (d64, cheaper value path) 0 -> 109 us, 0.35 -> 96, 0.4 -> 89, 0.45 -> 97.
    // PKV_DEC_KEY_FRACTION overrides (0 = interleaved items on every SM)
    double frac = r.head_dim >= 128 ? 0.365 : 0.39;  // (C2 with even counts: 0.378 -> 90.3, 0.392 -> 88.6, 0.405 -> 91.0)
    // (C3 after the round-2 value-path changes: 50 key CTAs 145.5 us, 52 ~140, 54 135.4, 56 136.7)
    // block32 keys (per-32 fp16 scales): C3 0.35 -> 172.6 us, 0.4 -> 150.7, 0.45 -> 154.2
    if (r.k_mode == PKV_K_BLOCK32 && r.head_dim >= 128) frac = 0.4;
    if (tuning().dec_key_fraction >= 0.0) frac = tuning().dec_key_fraction;
    const int grid = sm_count();
    if (frac > 0.0) a->key_ctas = std::max(2, std::min(grid - 2, 2 * (int)std::lround(frac * grid / 2.0)));  // even: whole TPCs
  }
  int rc = PKV_OK;
  for (int l = 0; l < L && rc == PKV_OK; ++l) {
    if (do_k) {
      a->k_codes[l] = r.k_codes[l];
      a->k_scale[l] = r.k_scale ? r.k_scale[l] : nullptr;
      a->k_bscale[l] = r.k_bscale ? reinterpret_cast<const __half*>(r.k_bscale[l]) : nullptr;
      a->k_out[l] = r.k_out[l];
      if (!a16(a->k_codes[l]) || !a16(a->k_out[l])) rc = PKV_ERR_ALIGNMENT;
    }
    if (do_v) {
      a->v_packed[l] = r.v_packed[l];
      a->v_scales[l] = r.v_scales[l];
      if (!a16(a->v_packed[l]) || !a16(a->v_scales[l]) || !a16(r.v_out[l])) rc = PKV_ERR_ALIGNMENT;
      else if (!make_map(&a->tm_v[l], r.v_out[l], eb, r.head_dim, r.num_vectors, kDecChunk)) rc = PKV_ERR_CUDA;
    }
  }
  if (rc == PKV_OK)
    rc = eb == 4 ? dec_launch<float>(*a, do_v ? r.head_dim : 64, r.sign, st)
                 : dec_launch<__nv_bfloat16>(*a, do_v ? r.head_dim : 64, r.sign, st);
  delete a;
  return rc;
}

}  // namespace stream
}  // namespace pkv
