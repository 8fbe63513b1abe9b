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
// Encode work items, in ticket order, per round r = 0..L:
//     A(r, *)  absmax of key chunk (per-tensor scale mode only), loaded with an
//              L2 evict_last policy so the chunk stays resident,
//     V(r, *) interleaved with E(r-1, *)  value chunks / key-encode chunks.
// E(l, j) re-reads key chunk j of layer l (from L2) and waits until every
// A(l, *) has published its maximum. All A(l, *) tickets precede all E(l, *)
// tickets and every CTA is resident, so the wait always terminates.
#include <cudaTypedefs.h>

#include <mutex>

#include "../../include/polykv.h"
#include "codec_common.cuh"
#include "pkv_common.cuh"
#include "tma.cuh"

namespace pkv {
namespace stream {

constexpr int kGroups = 2;
constexpr int kWarpsPerGroup = 4;
constexpr int kGroupThreads = 32 * kWarpsPerGroup;
constexpr int kThreads = 32 + kGroups * kGroupThreads;  // producer warp + consumers
constexpr int kChunk = 16384;                            // elements per work item
constexpr int kRingBytes = 192 * 1024;
constexpr int kMaxL = kMaxLayers;

enum ItemKind : int { kEnd = 0, kAbsmax = 1, kKeyEnc = 2, kValEnc = 3, kKeyDec = 4, kValDec = 5 };

struct Item {
  int kind;
  int layer;
  int idx;
  int pad;
};

// Geometry of a head-vector tile of kChunk elements (VR vectors of D) held
// as TMA boxes of BR rows x IB bytes (IB = swizzle span), NCB boxes across a
// row and NRB boxes down.
template <int D, int EB>
struct Tile {
  static constexpr int RB = D * EB;                  // bytes per head vector
  static constexpr int IB = RB < 128 ? RB : 128;     // inner box bytes
  static constexpr int NCB = RB / IB;
  static constexpr int VR = kChunk / D;              // vectors per item
  static constexpr int BR = VR < 256 ? VR : 256;     // rows per box
  static constexpr int NRB = VR / BR;
  static constexpr int BOX_BYTES = BR * IB;
  static constexpr int PASSES = VR / kGroupThreads;  // lane-per-vector passes per item
  static constexpr int PB = 3 * D / 8;               // packed bytes per vector
  static_assert(VR % kGroupThreads == 0, "item must hold a multiple of 128 vectors");
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
  int nA, nE, nV;  // items per layer
  int lag;         // E(l) items are issued in round l + lag
  unsigned int total;
  float delta;
  Codebook3 cb;
  uint32_t sign_bits[8];
  uint32_t* status;
  uint32_t* replay_count;
  // Per-tensor key maxima are published without fences: every absmax item
  // stores ONE 64-bit word (valid flag << 32 | max bits), so a reader that
  // sees the flag sees the value (single-copy atomicity of aligned 64-bit
  // accesses). The first key-encode item that finds all of a layer's words
  // valid caches the layer maximum in layer_max[l] the same way.
  unsigned long long* slots;      // [L][nA]
  unsigned long long* layer_max;  // [L]
  unsigned int* ticket;
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

__device__ __forceinline__ uint32_t ld_relaxed(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.relaxed.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ unsigned long long ld_relaxed64(const unsigned long long* p) {
  unsigned long long v;
  asm volatile("ld.relaxed.gpu.global.u64 %0, [%1];" : "=l"(v) : "l"(p) : "memory");
  return v;
}
__device__ __forceinline__ void st_relaxed64(unsigned long long* p, unsigned long long v) {
  asm volatile("st.relaxed.gpu.global.u64 [%0], %1;" ::"l"(p), "l"(v) : "memory");
}

__device__ __forceinline__ float2 f2(float a, float b) { return make_float2(a, b); }
__device__ __forceinline__ float2 add2(float2 a, float2 b) { return __fadd2_rn(a, b); }
__device__ __forceinline__ float2 sub2(float2 a, float2 b) { return __ffma2_rn(b, f2(-1.f, -1.f), a); }

// ---------------------------------------------------------------------------
// Sylvester FWHT of one head vector held by one lane as D/2 f32 pairs:
//   xp[(c >> 1) * 8 + e] = (x[8c + e], x[8c + 8 + e])   for even c.
// Stages run half = 1, 2, 4, ..., D/2 with lo' = lo + hi, hi' = lo - hi,
// exactly kvpool/fwht.py:31-39, so every output is bit-identical to numpy.
// ---------------------------------------------------------------------------
template <int D>
__device__ __forceinline__ void fwht_pairs(float2* xp) {
  constexpr int NP = D / 2;
#pragma unroll
  for (int h = 1; h < 8; h <<= 1) {  // coordinate bits 0..2
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      if (p & h) continue;
      const float2 a = xp[p], b = xp[p + h];
      xp[p] = add2(a, b);
      xp[p + h] = sub2(a, b);
    }
  }
  // coordinate bit 3: inside each pair, (x, y) -> (x + y, x - y)
#pragma unroll
  for (int p = 0; p < NP; ++p) {
    const float2 a = xp[p];
    xp[p] = __ffma2_rn(f2(1.f, -1.f), f2(a.y, a.y), f2(a.x, a.x));
  }
  // coordinate bits 4.. : pair-index bits 3..
#pragma unroll
  for (int h = 8; h < NP; h <<= 1) {
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      if (p & h) continue;
      const float2 a = xp[p], b = xp[p + h];
      xp[p] = add2(a, b);
      xp[p + h] = sub2(a, b);
    }
  }
}

// coordinate index of pair p, half hh
template <int D>
__device__ __forceinline__ constexpr int coord_of(int p, int hh) {
  return ((p >> 3) * 2 + hh) * 8 + (p & 7);
}

template <int D>
__device__ __forceinline__ void apply_sign(float2* xp, const uint32_t* bits) {
#pragma unroll
  for (int p = 0; p < D / 2; ++p) {
    const int i0 = coord_of<D>(p, 0), i1 = coord_of<D>(p, 1);
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
__device__ __noinline__ void v_replay_staged(const EncArgs& a, const TIn* src, uint8_t* out_packed,
                                             float* out_scale, double* R, uint8_t* C) {
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
  double rms = 0.0;
  if (lane == 0) rms = sqrt(pairwise_sumsq(R, D) / (double)D);  // valuequant.py:207
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

// pack NW 24-bit words (chunk order) and store them at shared address `dst`
template <int NW>
__device__ __forceinline__ void sts_words(uint32_t dst, const uint32_t (&w)[NW]) {
  if constexpr (NW % 4 == 0) {
    uint32_t u[3 * NW / 4];
#pragma unroll
    for (int i = 0; i < NW / 4; ++i) {
      u[3 * i + 0] = w[4 * i] | (w[4 * i + 1] << 24);
      u[3 * i + 1] = (w[4 * i + 1] >> 8) | (w[4 * i + 2] << 16);
      u[3 * i + 2] = (w[4 * i + 2] >> 16) | (w[4 * i + 3] << 8);
    }
    if constexpr (NW == 16) {
      tma::sts128(dst, make_uint4(u[0], u[1], u[2], u[3]));
      tma::sts128(dst + 16, make_uint4(u[4], u[5], u[6], u[7]));
      tma::sts128(dst + 32, make_uint4(u[8], u[9], u[10], u[11]));
    } else if constexpr (NW == 8) {
      tma::sts64(dst, make_uint2(u[0], u[1]));
      tma::sts64(dst + 8, make_uint2(u[2], u[3]));
      tma::sts64(dst + 16, make_uint2(u[4], u[5]));
    } else {
      tma::sts32(dst, u[0]);
      tma::sts32(dst + 4, u[1]);
      tma::sts32(dst + 8, u[2]);
    }
  } else {  // NW == 2: 6 bytes, 2-byte aligned
    const uint32_t lo = w[0] | (w[1] << 24), hi = w[1] >> 8;
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(dst), "h"((unsigned short)(lo & 0xffff)) : "memory");
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(dst + 2), "h"((unsigned short)(lo >> 16)) : "memory");
    asm volatile("st.shared.u16 [%0], %1;" ::"r"(dst + 4), "h"((unsigned short)(hi & 0xffff)) : "memory");
  }
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
// encode: value item (VR head vectors), one lane per vector
// ---------------------------------------------------------------------------
template <int D, typename TIn, bool SYM, bool SIGN>
__device__ void enc_value_item(const EncArgs& a, const Item& it, uint32_t in_s, int wig, int lane, double* R,
                               uint8_t* C) {
  using TL = Tile<D, (int)sizeof(TIn)>;
  constexpr int NCH = D / 8, NP = D / 2;
  const long long vbase = (long long)it.idx * TL::VR;
  const float* m = a.cb.mid32;
  const float delta = a.delta;
  uint8_t* gpk = a.v_packed[it.layer] + vbase * TL::PB;
  float* gsc = a.v_scales[it.layer] + vbase;
#pragma unroll 1
  for (int pass = 0; pass < TL::PASSES; ++pass) {
    const int vr = pass * kGroupThreads + wig * 32 + lane;
    const long long v = vbase + vr;
    const bool valid = v < a.nvec;
    float2 xp[NP];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      float t[8];
      if constexpr (sizeof(TIn) == 2) {
        lds_chunk8<TIn>(in_s + TL::off(vr, c), 0, t);
      } else {
        lds_chunk8<TIn>(in_s + TL::off(vr, 2 * c), in_s + TL::off(vr, 2 * c + 1), t);
      }
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (c & 1) xp[(c >> 1) * 8 + e].y = t[e];
        else xp[(c >> 1) * 8 + e].x = t[e];
      }
    }
    // squared norm in fp64 from the inputs (the rotation is orthogonal);
    // every x^2 is exact in fp64 and the sum is good to ~D * 2^-53.
    double s0 = 0.0, s1 = 0.0;
#pragma unroll
    for (int p = 0; p < NP; ++p) {
      s0 = fma((double)xp[p].x, (double)xp[p].x, s0);
      s1 = fma((double)xp[p].y, (double)xp[p].y, s1);
    }
    const double S = s0 + s1;
    if (SIGN) apply_sign<D>(xp, a.sign_bits);
    fwht_pairs<D>(xp);  // U = H x (unnormalised)

    bool replay = false, nonfinite = false, zero = false;
    float scale = 0.f, N = 0.f;
    if (!(S <= 1.79e308)) {
      nonfinite = true;
    } else if (S == 0.0) {
      zero = true;
    } else if (S < 0x1p-200 || S > 0x1p+200) {
      replay = true;
    } else {
      const double r = sqrt(S * (1.0 / D));  // S/D is exact (D = 2^k)
      scale = (float)r;
      const double fd = (double)scale;
      const float nb = (r >= fd) ? nextafterf(scale, INFINITY) : nextafterf(scale, 0.f);
      const double half_ulp = fabs((double)nb - fd) * 0.5;
      if (half_ulp - fabs(r - fd) <= 1e-12 * r) replay = true;  // f32 rounding of the scale in doubt
      N = (float)sqrt(S);  // ||x||; z = U / ||x||
    }

    uint32_t words[NCH];
#pragma unroll
    for (int c = 0; c < NCH; ++c) words[c] = 0;
    if (SYM) {
      // thresholds folded into the U domain: |z| > t  <=>  |U| > t * ||x||
      const float2 T1 = f2(-m[4] * N, -m[4] * N), T2 = f2(-m[5] * N, -m[5] * N), T3 = f2(-m[6] * N, -m[6] * N);
      const float DL = delta * N;
      float g = INFINITY;
#pragma unroll
      for (int p = 0; p < NP; ++p) {
        const float2 u = xp[p];
        const float2 au = f2(fabsf(u.x), fabsf(u.y));
        const float2 d1 = __fadd2_rn(au, T1), d2 = __fadd2_rn(au, T2), d3 = __fadd2_rn(au, T3);
        g = fminf(g, fminf(fabsf(d1.x), fabsf(d1.y)));
        g = fminf(g, fminf(fabsf(d2.x), fabsf(d2.y)));
        g = fminf(g, fminf(fabsf(d3.x), fabsf(d3.y)));
        g = fminf(g, fminf(au.x, au.y));
        // m = #thresholds above |u|; code = neg ? m : 7 - m
        const uint32_t mx = (__float_as_uint(d1.x) >> 31) + (__float_as_uint(d2.x) >> 31) + (__float_as_uint(d3.x) >> 31);
        const uint32_t my = (__float_as_uint(d1.y) >> 31) + (__float_as_uint(d2.y) >> 31) + (__float_as_uint(d3.y) >> 31);
        const uint32_t cx = (mx ^ ~(uint32_t)((int32_t)__float_as_uint(u.x) >> 31)) & 7u;
        const uint32_t cy = (my ^ ~(uint32_t)((int32_t)__float_as_uint(u.y) >> 31)) & 7u;
        const int c0 = (p >> 3) * 2, e = p & 7;
        words[c0] |= cx << (3 * e);
        words[c0 + 1] |= cy << (3 * e);
      }
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
          words[(p >> 3) * 2 + hh] |= ((p1 ? 4u : 0u) | (p2 ? 2u : 0u) | (p3 ? 1u : 0u)) << (3 * (p & 7));
        }
      }
      replay |= g < delta;
    }
    if (zero || nonfinite) {
#pragma unroll
      for (int c = 0; c < NCH; ++c) words[c] = 0;
      scale = 0.f;
    }
    replay = replay && valid && !nonfinite && !zero;
    if (valid && nonfinite) atomicOr(&a.status[it.layer], PKV_FLAG_V_NONFINITE);
    if (valid && !replay) {
      stg_words<NCH>(gpk + vr * TL::PB, words);
      gsc[vr] = scale;
    }
    // rare: exact fp64 replay, one vector at a time, whole warp
    unsigned mask = __ballot_sync(0xffffffffu, replay);
    while (mask) {
      const int src_lane = __ffs(mask) - 1;
      mask &= mask - 1;
      const int rvr = pass * kGroupThreads + wig * 32 + src_lane;
      const TIn* src = static_cast<const TIn*>(a.v_in[it.layer]) + (vbase + rvr) * D;
      v_replay_staged<D, TIn>(a, src, gpk + rvr * TL::PB, gsc + rvr, R, C);
    }
  }
}


// ---------------------------------------------------------------------------
// encode: key items
// ---------------------------------------------------------------------------
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

template <typename TIn>
__device__ void enc_absmax_item(const EncArgs& a, const Item& it, uint32_t in_s, int gt, int lane,
                                uint32_t* warp_max) {
  const long long e0 = (long long)it.idx * kChunk;
  const int n = (int)min((long long)kChunk, a.nelem - e0);
  uint32_t m = 0;
#pragma unroll 4
  for (int i = 0; i < kChunk / 8 / kGroupThreads; ++i) {
    const int u = i * kGroupThreads + gt;
    if (u * 8 < n) m = max(m, lds_absmax8<TIn>(in_s + u * 8 * (int)sizeof(TIn)));
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) *warp_max = m;  // combined and published after the group barrier
}

template <typename TIn>
__device__ void enc_key_item(const EncArgs& a, const Item& it, uint32_t in_s, int gt, int lane) {
  const long long e0 = (long long)it.idx * kChunk;
  const int n = (int)min((long long)kChunk, a.nelem - e0);
  int8_t* dst = a.k_codes[it.layer] + e0;
  if (a.k_mode == PKV_K_TENSOR) {
    unsigned long long lw = ld_relaxed64(a.layer_max + it.layer);
    if (!(lw >> 32)) {
      const unsigned long long* sl = a.slots + (long long)it.layer * a.nA;
      uint32_t spins = 0;
      uint64_t t0 = 0;
      for (;;) {
        bool all = true;
        uint32_t m = 0;
        for (int j = lane; j < a.nA; j += 32) {
          const unsigned long long v = ld_relaxed64(sl + j);
          all = all && (v >> 32) != 0;
          m = max(m, (uint32_t)v);
        }
#pragma unroll
        for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
        if (__all_sync(0xffffffffu, all)) {
          lw = (1ull << 32) | m;
          if (lane == 0) st_relaxed64(a.layer_max + it.layer, lw);
          break;
        }
        __nanosleep(200);
        tma::watchdog(spins, t0);
      }
    }
    const uint32_t pb = (uint32_t)lw;
    const bool nonfinite = pb >= 0x7f800000u;
    const float s = (nonfinite || pb == 0) ? 0.f : __uint_as_float(pb) / 127.0f;  // f32(peak/127), keyquant.py:60
    if (it.idx == 0 && gt == 0) {
      a.k_scale[it.layer][0] = s;
      if (nonfinite) atomicOr(&a.status[it.layer], PKV_FLAG_K_NONFINITE);
    }
    const float rcp = 1.0f / s;
    const bool exact_all = !(s >= 1e-30f);
#pragma unroll 4
    for (int i = 0; i < kChunk / 8 / kGroupThreads; ++i) {
      const int u = i * kGroupThreads + gt;
      if (u * 8 >= n) continue;
      float x[8];
      lds_chunk8<TIn>(in_s + u * 8 * (int)sizeof(TIn), in_s + u * 8 * (int)sizeof(TIn) + 16, x);
      st_u2(dst + u * 8, key_chunk<false>(x, s, rcp, exact_all));
    }
    return;
  }
  // block32: one fp16 scale per 32 contiguous elements; 4 consecutive lanes own a block
  __half* bsc = a.k_bscale[it.layer];
#pragma unroll 2
  for (int i = 0; i < kChunk / 8 / kGroupThreads; ++i) {
    const int u = i * kGroupThreads + gt;
    const bool valid = u * 8 < n;
    float x[8];
    uint32_t m = 0;
    if (valid) {
      lds_chunk8<TIn>(in_s + u * 8 * (int)sizeof(TIn), in_s + u * 8 * (int)sizeof(TIn) + 16, x);
#pragma unroll
      for (int j = 0; j < 8; ++j) m = max(m, __float_as_uint(x[j]) & 0x7fffffffu);
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) x[j] = 0.f;
    }
    m = max(m, __shfl_xor_sync(0xffffffffu, m, 1));
    m = max(m, __shfl_xor_sync(0xffffffffu, m, 2));
    if (!valid) continue;
    const bool nonfinite = m >= 0x7f800000u;
    uint16_t s16b = __half_as_ushort(__float2half_rn(__uint_as_float(m) / 127.0f));
    bool overflow = false;
    if (nonfinite || m == 0) {
      s16b = 0;
    } else if ((s16b & 0x7fffu) >= 0x7c00u) {
      overflow = true;
      s16b = 0;
    } else if (s16b == 0) {
      s16b = 1;  // peak > 0 but the scale underflows fp16: smallest subnormal
    }
    const float s = __half2float(__ushort_as_half(s16b));
    if ((lane & 3) == 0) {
      bsc[(e0 + u * 8) >> 5] = __ushort_as_half(s16b);
      if (nonfinite) atomicOr(&a.status[it.layer], PKV_FLAG_K_NONFINITE);
      if (overflow) atomicOr(&a.status[it.layer], PKV_FLAG_K_SCALE_OVERFLOW);
    }
    st_u2(dst + u * 8, key_chunk<true>(x, s, 1.0f / s, !(s >= 1e-30f)));
  }
}

// ---------------------------------------------------------------------------
// decode: key and value items
// ---------------------------------------------------------------------------
template <typename TOut>
__device__ void dec_key_item(const DecArgs& a, const Item& it, uint32_t in_s, uint8_t* out, int gt) {
  const long long e0 = (long long)it.idx * kChunk;
  const int n = (int)min((long long)kChunk, a.nelem - e0);
  const bool tensor = a.k_mode == PKV_K_TENSOR;
  const float ts = tensor ? __ldg(a.k_scale[it.layer]) : 0.f;
  const __half* bsc = a.k_bscale[it.layer];
  const uint32_t out_s = tma::smem_u32(out);
#pragma unroll 4
  for (int i = 0; i < kChunk / 8 / kGroupThreads; ++i) {
    const int u = i * kGroupThreads + gt;
    if (u * 8 >= n) continue;
    const uint2 w = tma::lds64(in_s + u * 8);
    const float s = tensor ? ts : __half2float(__ldg(bsc + ((e0 + u * 8) >> 5)));
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

// packed words of one vector (chunk order) from shared or global memory
template <int D>
__device__ __forceinline__ void load_packed(const uint8_t* p, bool smem, uint32_t (&w)[D / 8]) {
  constexpr int NW = D / 8;
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
  using TL = Tile<D, (int)sizeof(TOut)>;
  constexpr int NCH = D / 8, NP = D / 2;
  const long long vbase = (long long)it.idx * TL::VR;
  const uint8_t* gpk = a.v_packed[it.layer] + vbase * TL::PB;
  const float* gsc = a.v_scales[it.layer] + vbase;
  const float* ssc = reinterpret_cast<const float*>(in + 3 * kChunk / 8);
  const uint32_t out_s = tma::smem_u32(out);
  const float2 c2 = f2(a.sqrt_d32, a.sqrt_d32), r2 = f2(a.rcp_sqrt_d32, a.rcp_sqrt_d32);
  char* tb = reinterpret_cast<char*>(tbl);
  const uint32_t lane_off = (uint32_t)gt * 4u;
#pragma unroll 1
  for (int pass = 0; pass < TL::PASSES; ++pass) {
    const int vr = pass * kGroupThreads + wig * 32 + lane;
    const bool valid = vbase + vr < a.nvec;
    uint32_t words[NCH];
    float sc = 0.f;
    if (valid) {
      const bool pk_smem = (vr + 1) * TL::PB <= in_packed_bytes;
      load_packed<D>(pk_smem ? in + vr * TL::PB : gpk + vr * TL::PB, pk_smem, words);
      sc = (vr + 1) * 4 <= in_scale_bytes ? ssc[vr] : __ldg(gsc + vr);
    } else {
#pragma unroll
      for (int j = 0; j < NCH; ++j) words[j] = 0;
    }
    // per-lane table of the 8 scaled centroids: table_f32[code] * scale
    // (valuequant.py:232-234), laid out [code][thread] -> conflict-free
#pragma unroll
    for (int k = 0; k < 8; ++k) tbl[k * kGroupThreads + gt] = a.cent32[k] * sc;
    float2 xp[NP];
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        // byte address (code << 9) | lane_off   (kGroupThreads * 4 == 512)
        const int sh = 3 * e;
        const uint32_t off = (sh <= 9 ? (words[c] << (9 - sh)) : (words[c] >> (sh - 9))) & 0xe00u;
        const float val = *reinterpret_cast<const float*>(tb + (off | lane_off));
        if (c & 1) xp[(c >> 1) * 8 + e].y = val;
        else xp[(c >> 1) * 8 + e].x = val;
      }
    }
    fwht_pairs<D>(xp);
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
          const float2 e = __ffma2_rn(f2(-q.x, -q.y), c2, xp[p]);
          xp[p] = __ffma2_rn(e, r2, q);
        }
      }
    } else {
#pragma unroll
      for (int p = 0; p < NP; ++p) xp[p] = f2(__fdiv_rn(xp[p].x, a.sqrt_d32), __fdiv_rn(xp[p].y, a.sqrt_d32));
    }
    if (SIGN) apply_sign<D>(xp, a.sign_bits);
    // swizzled staging of the output tile (TMA tensor store layout)
#pragma unroll
    for (int c = 0; c < NCH; ++c) {
      const int p0 = (c >> 1) * 8;
      float y[8];
#pragma unroll
      for (int e = 0; e < 8; ++e) y[e] = (c & 1) ? xp[p0 + e].y : xp[p0 + e].x;
      if constexpr (sizeof(TOut) == 2) {
        tma::sts128(out_s + TL::off(vr, c), make_uint4(pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]),
                                                       pack_bf16x2(y[4], y[5]), pack_bf16x2(y[6], y[7])));
      } else {
        tma::sts128(out_s + TL::off(vr, 2 * c), make_uint4(__float_as_uint(y[0]), __float_as_uint(y[1]),
                                                           __float_as_uint(y[2]), __float_as_uint(y[3])));
        tma::sts128(out_s + TL::off(vr, 2 * c + 1), make_uint4(__float_as_uint(y[4]), __float_as_uint(y[5]),
                                                               __float_as_uint(y[6]), __float_as_uint(y[7])));
      }
    }
  }
}

// ---------------------------------------------------------------------------
// ticket -> item
// ---------------------------------------------------------------------------
__device__ __forceinline__ long long enc_round_start(const EncArgs& a, int r) {
  const int L = a.num_layers;
  const long long er = min(max(r - a.lag, 0), L);
  return (long long)min(r, L) * (a.nA + a.nV) + er * a.nE;
}

// Round r holds A(r) [r < L], then V(r) [r < L] interleaved with E(r - lag)
// [lag <= r < L + lag].
__device__ __forceinline__ Item enc_item(const EncArgs& a, unsigned int t) {
  const int L = a.num_layers;
  int lo = 0, hi = L + a.lag;  // find the last r with start(r) <= t
  while (hi - lo > 1) {
    const int mid = (lo + hi) >> 1;
    if (enc_round_start(a, mid) <= (long long)t) lo = mid;
    else hi = mid;
  }
  const int r = lo;
  long long off = (long long)t - enc_round_start(a, r);
  const long long nAr = r < L ? a.nA : 0, nVr = r < L ? a.nV : 0;
  const long long nEr = (r >= a.lag && r - a.lag < L) ? a.nE : 0;
  Item it{kEnd, 0, 0, 0};
  if (off < nAr) {
    it.kind = kAbsmax; it.layer = r; it.idx = (int)off;
    return it;
  }
  off -= nAr;
  const long long both = 2 * min(nVr, nEr);
  if (off < both) {
    if ((off & 1) == 0) { it.kind = kValEnc; it.layer = r; }
    else { it.kind = kKeyEnc; it.layer = r - a.lag; }
    it.idx = (int)(off >> 1);
    return it;
  }
  off -= both;
  if (nVr > nEr) { it.kind = kValEnc; it.layer = r; }
  else { it.kind = kKeyEnc; it.layer = r - a.lag; }
  it.idx = (int)(min(nVr, nEr) + off);
  return it;
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
// shared-memory plan
// ---------------------------------------------------------------------------
// Encode: a ring of input stages only (outputs are small and go straight to
// global memory). Decode: a ring of input stages plus NOB output buffers per
// consumer group, written back by TMA stores.
template <int EB_IN>
struct EncPlan {
  static constexpr int IN = kChunk * EB_IN;
  static constexpr int STAGE = IN;
  static constexpr int NST = kRingBytes / STAGE;
  static_assert(NST >= 2 && NST <= 8, "ring depth");
};
template <int EB_OUT>
struct DecPlan {
  static constexpr int IN = kChunk;  // >= key codes, packed values + scales
  static constexpr int STAGE = IN;
  static constexpr int OUT = kChunk * EB_OUT;
  static constexpr int NOB = EB_OUT == 2 ? 2 : 1;  // output buffers per group
  static constexpr int OUT_TOTAL = kGroups * NOB * OUT;
  static constexpr int NST = (208 * 1024 - OUT_TOTAL) / STAGE;
  static_assert(NST >= 2 && NST <= 8, "ring depth");
};

struct alignas(8) Ctl {
  uint64_t full[8];
  uint64_t empty[8];
  Item items[8];
  uint32_t warp_max[kGroups][kWarpsPerGroup];
};

template <int D>
constexpr int replay_bytes() {
  return kGroups * kWarpsPerGroup * (D * 8 + D);
}

template <int D, typename TIn>
constexpr size_t enc_smem_bytes() {
  return 1024 + (size_t)EncPlan<(int)sizeof(TIn)>::NST * EncPlan<(int)sizeof(TIn)>::STAGE + sizeof(Ctl) +
         replay_bytes<D>();
}
template <typename TOut>
constexpr size_t dec_smem_bytes() {
  using P = DecPlan<(int)sizeof(TOut)>;
  return 1024 + (size_t)P::OUT_TOTAL + (size_t)P::NST * P::STAGE + sizeof(Ctl) +
         kGroups * 8 * kGroupThreads * sizeof(float);
}

__device__ __forceinline__ uint8_t* align1024(uint8_t* p) {
  const uint32_t s = tma::smem_u32(p);
  return p + ((1024u - (s & 1023u)) & 1023u);
}


// ---------------------------------------------------------------------------
// encode kernel
// ---------------------------------------------------------------------------
template <int D, typename TIn, bool SYM, bool SIGN>
__global__ void __launch_bounds__(kThreads, 1) enc_kernel(const __grid_constant__ EncArgs a) {
  using P = EncPlan<(int)sizeof(TIn)>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* ring = align1024(smem_raw);
  Ctl* ctl = reinterpret_cast<Ctl*>(ring + P::NST * P::STAGE);
  uint8_t* replay_base = reinterpret_cast<uint8_t*>(ctl + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < P::NST; ++s) {
      tma::mbar_init(&ctl->full[s], 1);
      tma::mbar_init(&ctl->empty[s], 1);
    }
    tma::fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    // ---------------- producer ----------------
    if (lane == 0) {
      const uint64_t pol_last = tma::policy_evict_last(), pol_first = tma::policy_evict_first();
      unsigned int* ticket = a.ticket;
      int ends = 0;
      for (int seq = 0;; ++seq) {
        const int s = seq % P::NST;
        const uint32_t ph = (uint32_t)(seq / P::NST) & 1u;
        if (seq >= P::NST) tma::mbar_wait(&ctl->empty[s], ph ^ 1u);
        const unsigned int t = atomicAdd(ticket, 1u);
        const Item it = t < a.total ? enc_item(a, t) : Item{kEnd, 0, 0, 0};
        ctl->items[s] = it;
        uint8_t* in = ring + s * P::STAGE;
        if (it.kind == kEnd) {
          tma::mbar_arrive(&ctl->full[s]);
          if (++ends == kGroups) break;
          continue;
        }
        if (it.kind == kValEnc) {
          using TL = Tile<D, (int)sizeof(TIn)>;
          tma::mbar_arrive_expect_tx(&ctl->full[s], (uint32_t)P::IN);
          const int row0 = it.idx * TL::VR;
#pragma unroll 1
          for (int rb = 0; rb < TL::NRB; ++rb)
#pragma unroll 1
            for (int cb = 0; cb < TL::NCB; ++cb)
              tma::tensor2d_g2s(in + (rb * TL::NCB + cb) * TL::BOX_BYTES, &a.tm_v[it.layer],
                                cb * (TL::IB / (int)sizeof(TIn)), row0 + rb * TL::BR, &ctl->full[s], pol_first);
        } else {
          const long long e0 = (long long)it.idx * kChunk;
          const uint32_t bytes = (uint32_t)(min((long long)kChunk, a.nelem - e0) * (long long)sizeof(TIn));
          tma::mbar_arrive_expect_tx(&ctl->full[s], bytes);
          const TIn* src = static_cast<const TIn*>(a.k_in[it.layer]) + e0;
          tma::bulk_g2s(in, src, bytes, &ctl->full[s], it.kind == kAbsmax ? pol_last : pol_first);
        }
      }
    }
    return;
  }

  // ---------------- consumers ----------------
  const int g = (warp - 1) / kWarpsPerGroup;
  const int wig = (warp - 1) % kWarpsPerGroup;
  const int gt = threadIdx.x - 32 - g * kGroupThreads;
  double* R = reinterpret_cast<double*>(replay_base) + (warp - 1) * D;
  uint8_t* C = replay_base + kGroups * kWarpsPerGroup * D * 8 + (warp - 1) * D;
  for (int seq = g;; seq += kGroups) {
    const int s = seq % P::NST;
    const uint32_t ph = (uint32_t)(seq / P::NST) & 1u;
    tma::mbar_wait(&ctl->full[s], ph);
    const Item it = ctl->items[s];
    if (it.kind == kEnd) break;
    const uint32_t in_s = tma::smem_u32(ring + s * P::STAGE);
    if (it.kind == kAbsmax) {
      enc_absmax_item<TIn>(a, it, in_s, gt, lane, &ctl->warp_max[g][wig]);
    } else if (it.kind == kKeyEnc) {
      enc_key_item<TIn>(a, it, in_s, gt, lane);
    } else {
      enc_value_item<D, TIn, SYM, SIGN>(a, it, in_s, wig, lane, R, C);
    }
    // every warp of the group is done reading the stage: hand it back
    tma::named_bar_sync(1 + g, kGroupThreads);
    if (gt == 0) {
      tma::mbar_arrive(&ctl->empty[s]);
      if (it.kind == kAbsmax) {
        uint32_t m = 0;
#pragma unroll
        for (int w = 0; w < kWarpsPerGroup; ++w) m = max(m, ctl->warp_max[g][w]);
        st_relaxed64(a.slots + (long long)it.layer * a.nA + it.idx, (1ull << 32) | m);
      }
    }
  }
}

// ---------------------------------------------------------------------------
// decode kernel
// ---------------------------------------------------------------------------
template <int D, typename TOut, bool SIGN>
__global__ void __launch_bounds__(kThreads, 1) dec_kernel(const __grid_constant__ DecArgs a) {
  using P = DecPlan<(int)sizeof(TOut)>;
  using TL = Tile<D, (int)sizeof(TOut)>;
  extern __shared__ uint8_t smem_raw[];
  uint8_t* obuf = align1024(smem_raw);  // 1024-aligned swizzled output tiles
  uint8_t* ring = obuf + P::OUT_TOTAL;
  Ctl* ctl = reinterpret_cast<Ctl*>(ring + P::NST * P::STAGE);
  float* tables = reinterpret_cast<float*>(ctl + 1);
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (threadIdx.x == 0) {
    for (int s = 0; s < P::NST; ++s) {
      tma::mbar_init(&ctl->full[s], 1);
      tma::mbar_init(&ctl->empty[s], 1);
    }
    tma::fence_mbar_init();
  }
  __syncthreads();

  if (warp == 0) {
    if (lane == 0) {
      const uint64_t pol_first = tma::policy_evict_first();
      int ends = 0;
      for (int seq = 0;; ++seq) {
        const int s = seq % P::NST;
        const uint32_t ph = (uint32_t)(seq / P::NST) & 1u;
        if (seq >= P::NST) tma::mbar_wait(&ctl->empty[s], ph ^ 1u);
        // static round-robin schedule: items are independent and near-uniform
        const unsigned long long t64 = (unsigned long long)blockIdx.x + (unsigned long long)seq * gridDim.x;
        const unsigned int t = t64 < a.total ? (unsigned int)t64 : a.total;
        const Item it = t < a.total ? dec_item(a, t) : Item{kEnd, 0, 0, 0};
        ctl->items[s] = it;
        uint8_t* in = ring + s * P::STAGE;
        if (it.kind == kEnd) {
          tma::mbar_arrive(&ctl->full[s]);
          if (++ends == kGroups) break;
          continue;
        }
        if (it.kind == kKeyDec) {
          const long long e0 = (long long)it.idx * kChunk;
          const uint32_t bytes = (uint32_t)min((long long)kChunk, a.nelem - e0);
          tma::mbar_arrive_expect_tx(&ctl->full[s], bytes);
          tma::bulk_g2s(in, a.k_codes[it.layer] + e0, bytes, &ctl->full[s], pol_first);
        } else {
          const long long v0 = (long long)it.idx * TL::VR;
          const int nv = (int)min((long long)TL::VR, a.nvec - v0);
          const uint32_t pb = (uint32_t)(nv * TL::PB) & ~15u, sb = (uint32_t)(nv * 4) & ~15u;
          tma::mbar_arrive_expect_tx(&ctl->full[s], pb + sb);
          if (pb) tma::bulk_g2s(in, a.v_packed[it.layer] + v0 * TL::PB, pb, &ctl->full[s], pol_first);
          if (sb) tma::bulk_g2s(in + 3 * kChunk / 8, a.v_scales[it.layer] + v0, sb, &ctl->full[s], pol_first);
        }
      }
    }
    return;
  }

  const int g = (warp - 1) / kWarpsPerGroup;
  const int wig = (warp - 1) % kWarpsPerGroup;
  const int gt = threadIdx.x - 32 - g * kGroupThreads;
  float* tbl = tables + g * 8 * kGroupThreads;
  int nitems = 0;
  for (int seq = g;; seq += kGroups) {
    const int s = seq % P::NST;
    const uint32_t ph = (uint32_t)(seq / P::NST) & 1u;
    tma::mbar_wait(&ctl->full[s], ph);
    const Item it = ctl->items[s];
    if (it.kind == kEnd) break;
    uint8_t* in = ring + s * P::STAGE;
    uint8_t* out = obuf + (g * P::NOB + (nitems % P::NOB)) * P::OUT;
    ++nitems;
    int nv = 0;
    long long v0 = 0;
    if (it.kind == kKeyDec) {
      dec_key_item<TOut>(a, it, tma::smem_u32(in), out, gt);
    } else {
      v0 = (long long)it.idx * TL::VR;
      nv = (int)min((long long)TL::VR, a.nvec - v0);
      dec_value_item<D, TOut, SIGN>(a, it, in, (nv * TL::PB) & ~15, (nv * 4) & ~15, out, tbl, gt, wig, lane);
    }
    tma::fence_proxy_async_smem();
    if (P::NOB == 2 && gt == 0) tma::bulk_wait_read<0>();  // the other buffer is free for the next item
    tma::named_bar_sync(1 + g, kGroupThreads);
    if (gt == 0) {
      tma::mbar_arrive(&ctl->empty[s]);  // inputs consumed
      if (it.kind == kKeyDec) {
        const long long e0 = (long long)it.idx * kChunk;
        const int bytes = (int)min((long long)kChunk, a.nelem - e0) * (int)sizeof(TOut);
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
      if (P::NOB == 1) tma::bulk_wait_read<0>();
    }
    if (P::NOB == 1) tma::named_bar_sync(1 + g, kGroupThreads);  // single buffer: wait for its read-out
  }
  if (gt == 0) tma::bulk_wait<0>();
}

}  // namespace stream
}  // namespace pkv

// ===========================================================================
// host side
// ===========================================================================
#include "stream_codec.h"

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

// [nvec, D] head-vector tensor of one layer as a 2-D TMA map with the box
// geometry of Tile<D, eb>.
bool make_map(CUtensorMap* m, const void* base, int eb, int D, long long nvec) {
  auto fn = encode_fn();
  if (!fn) return false;
  const int RB = D * eb, IB = RB < 128 ? RB : 128, VR = kChunk / D, BR = VR < 256 ? VR : 256;
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
  return r == CUDA_SUCCESS;
}

template <typename K>
int coop_launch(K kernel, const void* args, size_t smem, cudaStream_t st) {
  if (cudaFuncSetAttribute(kernel, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem) != cudaSuccess)
    return PKV_ERR_CUDA;
  int per_sm = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, kernel, kThreads, smem) != cudaSuccess || per_sm < 1)
    return PKV_ERR_CUDA;
  void* params[] = {const_cast<void*>(args)};
  const cudaError_t e =
      cudaLaunchCooperativeKernel((const void*)kernel, dim3((unsigned)(sm_count() * per_sm)), dim3(kThreads), params,
                                  smem, st);
  return e == cudaSuccess ? PKV_OK : PKV_ERR_CUDA;
}

template <int D, typename TIn>
int enc_launch_d(const EncArgs& a, bool sym, bool sign, cudaStream_t st) {
  const size_t smem = enc_smem_bytes<D, TIn>();
  if (sym) {
    return sign ? coop_launch(enc_kernel<D, TIn, true, true>, &a, smem, st)
                : coop_launch(enc_kernel<D, TIn, true, false>, &a, smem, st);
  }
  return sign ? coop_launch(enc_kernel<D, TIn, false, true>, &a, smem, st)
              : coop_launch(enc_kernel<D, TIn, false, false>, &a, smem, st);
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

template <int D, typename TOut>
int dec_launch_d(const DecArgs& a, bool sign, cudaStream_t st) {
  const size_t smem = dec_smem_bytes<TOut>();
  return sign ? coop_launch(dec_kernel<D, TOut, true>, &a, smem, st)
              : coop_launch(dec_kernel<D, TOut, false>, &a, smem, st);
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
  const long long nelem = num_vectors * (long long)std::max(head_dim, 1);
  const long long kch = (nelem + kChunk - 1) / kChunk;
  const long long L = std::min(std::max(num_layers, 0), kMaxL);
  return (size_t)(L * kch * 8 + L * 8 + 16);
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
  // workspace: [u64 slots L*nA][u64 layer_max L][u32 ticket]
  unsigned long long* w64 = reinterpret_cast<unsigned long long*>(r.ws);
  const long long kch = (nelem + kChunk - 1) / kChunk;
  const long long vch = (r.num_vectors + (kChunk / std::max(r.head_dim, 1)) - 1) / (kChunk / std::max(r.head_dim, 1));
  a->nE = do_k ? (int)kch : 0;
  a->nA = (do_k && r.k_mode == PKV_K_TENSOR) ? (int)kch : 0;
  a->nV = do_v ? (int)vch : 0;
  const long long total = (long long)L * (a->nA + a->nE + a->nV);
  if (total >= (1LL << 32) - 1024) {
    delete a;
    return PKV_ERR_INVALID_ARG;
  }
  a->total = (unsigned int)total;
  a->slots = w64;
  a->layer_max = w64 + (long long)L * a->nA;
  a->ticket = reinterpret_cast<unsigned int*>(a->layer_max + L);
  const size_t ws_need = workspace_bytes(L, r.num_vectors, r.head_dim);
  if (r.ws_bytes < ws_need) {
    delete a;
    return PKV_ERR_ALIGNMENT;  // too small for this path: the caller falls back
  }
  // lag between a layer's absmax items and its key-encode items: about twice
  // the items in flight in all rings, bounded so the lagged key tensors stay
  // L2-resident (~40 MB).
  {
    const long long inflight = (long long)sm_count() * (eb == 2 ? EncPlan<2>::NST : EncPlan<4>::NST);
    const long long round = std::max(1LL, (long long)a->nA + a->nV + a->nE);
    long long lag = 1 + (2 * inflight + round - 1) / round;
    const long long layer_bytes = std::max(1LL, nelem * eb);
    lag = std::min(lag, std::max(1LL, (40LL << 20) / layer_bytes));
    a->lag = (int)std::max(1LL, std::min(lag, (long long)L));
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
      else if (!make_map(&a->tm_v[l], a->v_in[l], eb, r.head_dim, r.num_vectors)) rc = PKV_ERR_CUDA;
    }
  }
  if (rc == PKV_OK && cudaMemsetAsync(r.ws, 0, ws_need, st) != cudaSuccess) rc = PKV_ERR_CUDA;
  if (rc == PKV_OK)
    rc = eb == 4 ? enc_launch<float>(*a, do_v ? r.head_dim : 64, r.cb.symmetric != 0, r.sign, st)
                 : enc_launch<__nv_bfloat16>(*a, do_v ? r.head_dim : 64, r.cb.symmetric != 0, r.sign, st);
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
  const long long kch = (nelem + kChunk - 1) / kChunk;
  const long long vr = kChunk / std::max(r.head_dim, 1);
  a->nK = do_k ? (int)kch : 0;
  a->nV = do_v ? (int)((r.num_vectors + vr - 1) / vr) : 0;
  const long long total = (long long)L * (a->nK + a->nV);
  if (total >= (1LL << 32) - (1LL << 20)) {
    delete a;
    return PKV_ERR_INVALID_ARG;
  }
  a->total = (unsigned int)total;
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
      else if (!make_map(&a->tm_v[l], r.v_out[l], eb, r.head_dim, r.num_vectors)) rc = PKV_ERR_CUDA;
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
