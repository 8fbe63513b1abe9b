// PolyKV SharedKVPool codec for B200 (sm_100a): encode (write side) and
// decode (materialising read side) kernels plus their C ABI (include/polykv.h).
//
// Reference semantics (all citations into /root/reference/pkg/src/kvpool):
//   quantize_k      keyquant.py:52-65   per-tensor q8_0, round half away
//   dequantize_k    keyquant.py:68-71   code * scale in f32
//   quantize_v      valuequant.py:193-219  (sign) -> FWHT/sqrt(d) in f64 ->
//                   rms (numpy pairwise mean) -> f32 scale -> z = rot/rms ->
//                   searchsorted(pinned midpoints) -> zero-scale rows -> 0
//   pack_indices_3bit valuequant.py:312-328  8 codes per 24-bit LE word
//   dequantize_v    valuequant.py:222-238  table[code]*scale, f32 FWHT,
//                   / f32(sqrt(d)), * sign
//   round_to_bfloat16 pool.py:66-76       RNE on the f32 bit pattern
//
// Exactness strategy for the write side:
//   keys   - fp32 reciprocal estimate; elements within 4e-5 of a rounding
//            half-point are recomputed with the reference's fp64 formula.
//   values - fp32 FWHT + fp64 sum of squares of the inputs; a vector whose
//            f32 scale sits within 1e-12 (relative) of an f32 rounding
//            boundary, or any of whose normalised coordinates lies within a
//            proven error bound `delta` of a decision threshold, is replayed
//            warp-cooperatively in fp64 in numpy's exact operation order.
//
// Work decomposition: every kernel runs a static, warp-granular schedule
// (no block barriers); the encode kernel is launched cooperatively so that
// all warps are co-resident, which makes its one cross-warp dependency (keys
// of layer l wait for layer l's absmax) deadlock-free without atomics on a
// ticket counter.
#include <algorithm>
#include <cstdlib>
#include <cmath>
#include <cstring>

#include "../../include/polykv.h"
#include "diag.h"
#include "pkv_common.cuh"
#include "codec_common.cuh"
#include "stream_codec.h"
#include "tuning.h"

namespace pkv {


constexpr int kMaxRounds = kMaxLayers + 16;

struct EncodeArgs {
  int num_layers;
  int head_dim;
  int k_mode;
  int vec_ok;                     // all pointers aligned and n % 8 == 0
  long long nvec;                 // vectors per layer
  long long nelem;                // elements per layer
  int a_items, e_items, v_items;  // warp items per layer
  int lag;                        // key-encode of layer l runs in round l + lag
  int num_rounds;
  long long round_start[kMaxRounds + 1];
  long long total_items;
  float delta;                    // guard band on normalised coordinates
  uint32_t sign_bits[8];
  Codebook3 cb;
  uint32_t* status;               // [L]
  uint32_t* replay_count;         // [1] or null
  uint32_t* ws;                   // [0..L) max bits, [L..2L) done counters
  const void* k_in[kMaxLayers];
  const void* v_in[kMaxLayers];
  int8_t* k_codes[kMaxLayers];
  float* k_scale[kMaxLayers];
  __half* k_bscale[kMaxLayers];
  uint8_t* v_packed[kMaxLayers];
  float* v_scales[kMaxLayers];
};

struct DecodeArgs {
  int num_layers;
  int head_dim;
  int k_mode;
  int vec_ok;
  long long nvec, nelem;
  int k_items, v_items;  // warp items per layer
  long long total_items;
  float sqrt_d32;        // f32(sqrt(d))
  float rcp_sqrt_d32;    // RN(1 / f32(sqrt(d)))
  uint32_t sign_bits[8];
  float cent32[8];
  const int8_t* k_codes[kMaxLayers];
  const float* k_scale[kMaxLayers];
  const __half* k_bscale[kMaxLayers];
  const uint8_t* v_packed[kMaxLayers];
  const float* v_scales[kMaxLayers];
  void* k_out[kMaxLayers];
  void* v_out[kMaxLayers];
};

constexpr int kWarps = kThreads / 32;
constexpr int kKChunks = 32;                 // 8-element chunks per lane per key item
constexpr int kKElems = 32 * 8 * kKChunks;   // key elements per warp item (8192)

template <int D>
struct VItem {
  // value vectors per warp item: ~16K coordinates
  static constexpr int ITERS = (16384 / (VG<D>::VPW * D)) > 0 ? (16384 / (VG<D>::VPW * D)) : 1;
  static constexpr int VECS = ITERS * VG<D>::VPW;
};

__device__ __forceinline__ uint32_t ld_acquire(const uint32_t* p) {
  uint32_t v;
  asm volatile("ld.acquire.gpu.global.u32 %0, [%1];" : "=r"(v) : "l"(p) : "memory");
  return v;
}

// ---------------------------------------------------------------------------
// keys
// ---------------------------------------------------------------------------



// |x| bit patterns of 8 inputs, max-reduced without unpacking bf16
__device__ __forceinline__ uint32_t chunk_absmax_bits(const float* p) {
  const uint4 a = ld_stream_u4(p), b = ld_stream_u4(p + 4);
  uint32_t m = max(max(a.x & 0x7fffffffu, a.y & 0x7fffffffu), max(a.z & 0x7fffffffu, a.w & 0x7fffffffu));
  return max(m, max(max(b.x & 0x7fffffffu, b.y & 0x7fffffffu), max(b.z & 0x7fffffffu, b.w & 0x7fffffffu)));
}
__device__ __forceinline__ uint32_t chunk_absmax_bits(const __nv_bfloat16* p) {
  const uint4 a = ld_stream_u4(p);
  uint32_t m = __vmaxu2(__vmaxu2(a.x & 0x7fff7fffu, a.y & 0x7fff7fffu),
                        __vmaxu2(a.z & 0x7fff7fffu, a.w & 0x7fff7fffu));
  m = max(m & 0xffffu, m >> 16);
  return m << 16;  // bf16 -> f32 bit pattern
}

template <typename TIn>
__device__ void k_absmax_item(const EncodeArgs& a, int layer, int item, int lane) {
  const TIn* src = static_cast<const TIn*>(a.k_in[layer]);
  const long long e0 = (long long)item * kKElems;
  const long long n = a.nelem;
  uint32_t m = 0;
  if (a.vec_ok) {
#pragma unroll 8
    for (int i = 0; i < kKChunks; ++i) {
      const long long e = e0 + ((long long)i * 32 + lane) * 8;
      if (e < n) m = max(m, chunk_absmax_bits(src + e));
    }
  } else {
    for (int i = lane; i < kKElems; i += 32) {
      const long long e = e0 + i;
      if (e < n) m = max(m, __float_as_uint(load1(src + e)) & 0x7fffffffu);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  if (lane == 0) {
    atomicMax(&a.ws[layer], m);
    __threadfence();
    atomicAdd(&a.ws[a.num_layers + layer], 1u);
  }
}

template <typename TIn>
__device__ void k_encode_item(const EncodeArgs& a, int layer, int item, int lane) {
  const TIn* src = static_cast<const TIn*>(a.k_in[layer]);
  int8_t* dst = a.k_codes[layer];
  const long long e0 = (long long)item * kKElems;
  const long long n = a.nelem;

  if (a.k_mode == PKV_K_TENSOR) {
    uint32_t pb = 0;
    if (lane == 0) {
      const uint32_t* done = a.ws + a.num_layers + layer;
      while (ld_acquire(done) < (uint32_t)a.a_items) __nanosleep(64);
      pb = ld_acquire(a.ws + layer);
    }
    pb = __shfl_sync(0xffffffffu, pb, 0);
    const bool nonfinite = pb >= 0x7f800000u;
    const float s = (nonfinite || pb == 0) ? 0.f : __uint_as_float(pb) / 127.0f;  // f32(peak/127)
    if (item == 0 && lane == 0) {
      a.k_scale[layer][0] = s;
      if (nonfinite) atomicOr(&a.status[layer], PKV_FLAG_K_NONFINITE);
    }
    const float rcp = 1.0f / s;
    const bool exact_all = !(s >= 1e-30f);  // s == 0 or tiny: exact path (zeros for s == 0)
    if (a.vec_ok) {
#pragma unroll 4
      for (int i = 0; i < kKChunks; ++i) {
        const long long e = e0 + ((long long)i * 32 + lane) * 8;
        if (e >= n) continue;
        float x[8];
        load8(src + e, x);
        st_u2(dst + e, key_chunk<false>(x, s, rcp, exact_all));
      }
    } else {
      for (int i = lane; i < kKElems; i += 32) {
        const long long e = e0 + i;
        if (e >= n) continue;
        const float x = load1(src + e);
        dst[e] = (s == 0.f) ? (int8_t)0 : (int8_t)key_code_exact(x, s, -128, 127);
      }
    }
    return;
  }

  // ---- block32: one fp16 scale per 32 contiguous elements (q8_0) ----
  __half* bsc = a.k_bscale[layer];
  if (a.vec_ok) {
#pragma unroll 2
    for (int i = 0; i < kKChunks; ++i) {
      const long long e = e0 + ((long long)i * 32 + lane) * 8;
      const bool valid = e < n;
      float x[8];
      uint32_t m = 0;
      if (valid) {
        load8(src + e, x);
#pragma unroll
        for (int j = 0; j < 8; ++j) m = max(m, __float_as_uint(x[j]) & 0x7fffffffu);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = 0.f;
      }
      // 4 consecutive lanes hold one 32-element block
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
        bsc[e >> 5] = __ushort_as_half(s16b);
        if (nonfinite) atomicOr(&a.status[layer], PKV_FLAG_K_NONFINITE);
        if (overflow) atomicOr(&a.status[layer], PKV_FLAG_K_SCALE_OVERFLOW);
      }
      st_u2(dst + e, key_chunk<true>(x, s, 1.0f / s, !(s >= 1e-30f)));
    }
  } else {
    const long long nb = (n + 31) / 32;
    for (int bi = lane; bi < kKElems / 32; bi += 32) {
      const long long b = e0 / 32 + bi;
      if (b >= nb) continue;
      const long long lo = b * 32, hi = min(lo + 32, n);
      uint32_t m = 0;
      for (long long e = lo; e < hi; ++e) m = max(m, __float_as_uint(load1(src + e)) & 0x7fffffffu);
      const bool nonfinite = m >= 0x7f800000u;
      uint16_t s16b = __half_as_ushort(__float2half_rn(__uint_as_float(m) / 127.0f));
      bool overflow = false;
      if (nonfinite || m == 0) s16b = 0;
      else if ((s16b & 0x7fffu) >= 0x7c00u) { overflow = true; s16b = 0; }
      else if (s16b == 0) s16b = 1;
      bsc[b] = __ushort_as_half(s16b);
      if (nonfinite) atomicOr(&a.status[layer], PKV_FLAG_K_NONFINITE);
      if (overflow) atomicOr(&a.status[layer], PKV_FLAG_K_SCALE_OVERFLOW);
      const float s = __half2float(__ushort_as_half(s16b));
      for (long long e = lo; e < hi; ++e)
        dst[e] = (s == 0.f) ? (int8_t)0 : (int8_t)key_code_exact(load1(src + e), s, -127, 127);
    }
  }
}

// ---------------------------------------------------------------------------
// values
// ---------------------------------------------------------------------------

// Exact fp64 replay of kvpool.valuequant.quantize_v for one head vector,
// executed by the whole warp. R: D doubles of warp scratch; C: D bytes.
template <int D, typename TIn>
__device__ __noinline__ void v_replay(const EncodeArgs& a, int layer, long long v, double* R,
                                      uint8_t* C) {
  const int lane = threadIdx.x & 31;
  const TIn* p = static_cast<const TIn*>(a.v_in[layer]) + v * D;
  for (int i = lane; i < D; i += 32) {
    double x = (double)load1(p + i);
    if (sign_bit(a.sign_bits, i)) x = -x;  // vals * sign_diagonal (bits are 0 without a seed)
    R[i] = x;
  }
  __syncwarp();
  for (int h = 1; h < D; h <<= 1) {  // fwht.py:31-39, in f64
    for (int q = lane; q < D / 2; q += 32) {
      const int i = (q / h) * 2 * h + (q % h);
      const double lo = R[i], hi = R[i + h];
      R[i] = lo + hi;
      R[i + h] = lo - hi;
    }
    __syncwarp();
  }
  const double sq = sqrt((double)D);  // dt.type(np.sqrt(d)), fwht.py:50
  for (int i = lane; i < D; i += 32) R[i] = R[i] / sq;
  __syncwarp();
  double rms = 0.0;
  if (lane == 0) {
    const double mean = pairwise_sumsq(R, D) / (double)D;  // np.mean(np.square(rot))
    rms = sqrt(mean);
  }
  rms = __shfl_sync(0xffffffffu, rms, 0);
  const float scale = (float)rms;
  const double den = rms > 0.0 ? rms : 1.0;
  for (int i = lane; i < D; i += 32) {
    const double z = R[i] / den;
    int c = 0;
#pragma unroll
    for (int k = 0; k < 7; ++k) c += (a.cb.mid64[k] < z) ? 1 : 0;  // searchsorted 'left'
    C[i] = scale == 0.0f ? 0 : (uint8_t)c;
  }
  __syncwarp();
  uint8_t* out = a.v_packed[layer] + v * VG<D>::PACKED_BYTES;
  for (int w = lane; w < D / 8; w += 32) {
    uint32_t word = 0;
#pragma unroll
    for (int e = 0; e < 8; ++e) word |= (uint32_t)C[8 * w + e] << (3 * e);
    out[3 * w + 0] = (uint8_t)(word & 0xff);
    out[3 * w + 1] = (uint8_t)((word >> 8) & 0xff);
    out[3 * w + 2] = (uint8_t)((word >> 16) & 0xff);
  }
  if (lane == 0) {
    a.v_scales[layer][v] = scale;
    if (a.replay_count) atomicAdd(a.replay_count, 1u);
  }
  __syncwarp();
}

// Store Q packed 24-bit words (contiguous in the vector) at byte pointer p.
template <int Q>
__device__ __forceinline__ void store_words(uint8_t* p, const uint32_t (&q)[Q]) {
  if constexpr (Q == 8) {
    uint32_t u[6];
    u[0] = q[0] | (q[1] << 24);
    u[1] = (q[1] >> 8) | (q[2] << 16);
    u[2] = (q[2] >> 16) | (q[3] << 8);
    u[3] = q[4] | (q[5] << 24);
    u[4] = (q[5] >> 8) | (q[6] << 16);
    u[5] = (q[6] >> 16) | (q[7] << 8);
    st_u2(p, make_uint2(u[0], u[1]));
    st_u2(p + 8, make_uint2(u[2], u[3]));
    st_u2(p + 16, make_uint2(u[4], u[5]));
  } else if constexpr (Q == 4) {
    uint32_t* w = reinterpret_cast<uint32_t*>(p);
    w[0] = q[0] | (q[1] << 24);
    w[1] = (q[1] >> 8) | (q[2] << 16);
    w[2] = (q[2] >> 16) | (q[3] << 8);
  } else if constexpr (Q == 2) {
    uint16_t* w = reinterpret_cast<uint16_t*>(p);
    w[0] = (uint16_t)(q[0] & 0xffff);
    w[1] = (uint16_t)((q[0] >> 16) | ((q[1] & 0xff) << 8));
    w[2] = (uint16_t)(q[1] >> 8);
  } else {
    p[0] = (uint8_t)(q[0] & 0xff);
    p[1] = (uint8_t)((q[0] >> 8) & 0xff);
    p[2] = (uint8_t)((q[0] >> 16) & 0xff);
  }
}

// Load Q packed words (inverse of store_words).
template <int Q>
__device__ __forceinline__ void load_words(const uint8_t* p, uint32_t (&q)[Q]) {
  if constexpr (Q == 8) {
    const uint2 u0 = ld_stream_u2(p), u1 = ld_stream_u2(p + 8), u2 = ld_stream_u2(p + 16);
    q[0] = u0.x & 0xffffffu;
    q[1] = __funnelshift_r(u0.x, u0.y, 24) & 0xffffffu;
    q[2] = __funnelshift_r(u0.y, u1.x, 16) & 0xffffffu;
    q[3] = u1.x >> 8;
    q[4] = u1.y & 0xffffffu;
    q[5] = __funnelshift_r(u1.y, u2.x, 24) & 0xffffffu;
    q[6] = __funnelshift_r(u2.x, u2.y, 16) & 0xffffffu;
    q[7] = u2.y >> 8;
  } else if constexpr (Q == 4) {
    const uint32_t u0 = ld_stream_u1(p), u1 = ld_stream_u1(p + 4), u2 = ld_stream_u1(p + 8);
    q[0] = u0 & 0xffffffu;
    q[1] = __funnelshift_r(u0, u1, 24) & 0xffffffu;
    q[2] = __funnelshift_r(u1, u2, 16) & 0xffffffu;
    q[3] = u2 >> 8;
  } else {
#pragma unroll
    for (int j = 0; j < Q; ++j)
      q[j] = (uint32_t)p[3 * j] | ((uint32_t)p[3 * j + 1] << 8) | ((uint32_t)p[3 * j + 2] << 16);
  }
}

// Per-warp shared memory of the encode kernel.
template <int D>
struct VSmem {
  uint32_t stage[VG<D>::VPW][VG<D>::W + 1];  // packed-word transpose
  double R[D];                               // replay scratch
  uint8_t C[D];
};

// Lane's 64-bit sign mask over its CPT coordinates (bit c*8+e).
template <int D>
__device__ __forceinline__ unsigned long long lane_sign_mask(const uint32_t* bits, int s) {
  using G = VG<D>;
  unsigned long long m = 0;
#pragma unroll
  for (int c = 0; c < G::NCH; ++c)
#pragma unroll
    for (int e = 0; e < 8; ++e)
      if (sign_bit(bits, 8 * (s + G::TPV * c) + e)) m |= 1ull << (c * 8 + e);
  return m;
}

template <int D, typename TIn, bool SYM, bool SIGN>
__device__ void v_encode_item(const EncodeArgs& a, int layer, int item, int warp, int lane,
                              VSmem<D>& sm, unsigned long long smask) {
  using G = VG<D>;
  static_assert(G::CPT <= 64, "sign mask holds 64 coordinates");
  const int vw = lane / G::TPV, s = lane % G::TPV;
  const TIn* src = static_cast<const TIn*>(a.v_in[layer]);
  uint8_t* packed = a.v_packed[layer];
  float* scales = a.v_scales[layer];
  const long long vbase = (long long)item * VItem<D>::VECS;
  const float delta = a.delta;
  const float* m = a.cb.mid32;

#pragma unroll 1
  for (int it = 0; it < VItem<D>::ITERS; ++it) {
    const long long v = vbase + (long long)it * G::VPW + vw;
    const bool valid = v < a.nvec;
    float x[G::CPT];
    if (valid) {
      const TIn* p = src + v * D;
#pragma unroll
      for (int c = 0; c < G::NCH; ++c) {
        float t[8];
        load8(p + 8 * (s + G::TPV * c), t);
#pragma unroll
        for (int e = 0; e < 8; ++e) x[c * 8 + e] = t[e];
      }
    } else {
#pragma unroll
      for (int i = 0; i < G::CPT; ++i) x[i] = 0.f;
    }
    if (SIGN) {
#pragma unroll
      for (int i = 0; i < G::CPT; ++i)
        x[i] = __uint_as_float(__float_as_uint(x[i]) ^ ((uint32_t)(smask >> i) << 31));
    }
    // squared norm in fp64 from the inputs (the rotation is orthogonal):
    // every x^2 is exact in fp64, the sum is good to ~D*2^-53 relative.
    double S = 0.0;
#pragma unroll
    for (int i = 0; i < G::CPT; ++i) S = fma((double)x[i], (double)x[i], S);
#pragma unroll
    for (int lb = 0; lb < G::LB; ++lb) S += __shfl_xor_sync(0xffffffffu, S, 1 << lb);

    fwht_lanes<D>(x, s);  // U = H x (unnormalised)

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
      if (half_ulp - fabs(r - fd) <= 1e-12 * r) replay = true;
      N = (float)sqrt(S);  // ||x||; z = U / ||x||
    }

    uint32_t words[G::NCH];
    if (SYM) {
      // thresholds folded into the U domain: |z| > t  <=>  |U| > t*||x||
      const float T1 = m[4] * N, T2 = m[5] * N, T3 = m[6] * N, DL = delta * N;
      float gmin = INFINITY, amin = INFINITY;
#pragma unroll
      for (int c = 0; c < G::NCH; ++c) {
        uint32_t w = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float u = x[c * 8 + e];
          const float au = fabsf(u);
          const bool p2 = au > T2;
          const float thr = p2 ? T3 : T1;
          const bool p1 = au > thr;
          const uint32_t k4 = (p2 ? 6u : 4u) + (p1 ? 1u : 0u);              // (2*p2 + p1) ^ 4
          const uint32_t sa = (uint32_t)((int32_t)__float_as_uint(u) >> 31);  // -1 if negative
          const uint32_t code = (k4 ^ sa) & 7u;  // neg ? 3 - k : 4 + k
          w |= code << (3 * e);
          gmin = fminf(gmin, fminf(fabsf(au - T2), fabsf(au - thr)));
          amin = fminf(amin, au);
        }
        words[c] = w;
      }
      replay |= (gmin < DL) | (amin < DL);
    } else {
      const float inv = N > 0.f ? 1.0f / N : 0.f;
      float gmin = INFINITY;
#pragma unroll
      for (int c = 0; c < G::NCH; ++c) {
        uint32_t w = 0;
#pragma unroll
        for (int e = 0; e < 8; ++e) {
          const float z = x[c * 8 + e] * inv;
          // binary search over the 7 thresholds; both boundaries of the final
          // cell are on the search path, so the guard checks only those three.
          const bool p1 = z > m[3];
          const float t2 = p1 ? m[5] : m[1];
          const bool p2 = z > t2;
          const float t3 = p1 ? (p2 ? m[6] : m[4]) : (p2 ? m[2] : m[0]);
          const bool p3 = z > t3;
          gmin = fminf(gmin, fminf(fabsf(z - m[3]), fminf(fabsf(z - t2), fabsf(z - t3))));
          w |= ((p1 ? 4u : 0u) | (p2 ? 2u : 0u) | (p3 ? 1u : 0u)) << (3 * e);
        }
        words[c] = w;
      }
      replay |= gmin < delta;
    }
    if (zero || nonfinite) {
#pragma unroll
      for (int c = 0; c < G::NCH; ++c) words[c] = 0;
      scale = 0.f;
    }
    // all lanes of a vector agree on replay
#pragma unroll
    for (int lb = 0; lb < G::LB; ++lb) replay |= __shfl_xor_sync(0xffffffffu, (int)replay, 1 << lb) != 0;
    replay = replay && valid && !nonfinite && !zero;
    if (valid && nonfinite && s == 0) atomicOr(&a.status[layer], PKV_FLAG_V_NONFINITE);

    // redistribute words so each lane owns Q contiguous words of its vector
#pragma unroll
    for (int c = 0; c < G::NCH; ++c) sm.stage[vw][s + G::TPV * c] = words[c];
    __syncwarp();
    uint32_t q[G::Q];
#pragma unroll
    for (int j = 0; j < G::Q; ++j) q[j] = sm.stage[vw][s * G::Q + j];
    __syncwarp();
    if (valid && !replay) {
      store_words<G::Q>(packed + v * G::PACKED_BYTES + s * 3 * G::Q, q);
      if (s == 0) scales[v] = scale;
    }
    // rare: exact fp64 replay, one vector at a time, whole warp
    unsigned mask = __ballot_sync(0xffffffffu, replay && s == 0);
    while (mask) {
      const int src_lane = __ffs(mask) - 1;
      mask &= mask - 1;
      v_replay<D, TIn>(a, layer, vbase + (long long)it * G::VPW + src_lane / G::TPV, sm.R, sm.C);
    }
  }
}

// ---------------------------------------------------------------------------
// encode kernel: static warp schedule over rounds
// ---------------------------------------------------------------------------
// Round r holds the absmax items of layer r, then the value items of layer r
// interleaved with the key-encode items of layer r - lag. Warp w processes
// items w, w + W, w + 2W, ... in order. A key-encode item waits for its
// layer's absmax; all of those carry smaller item indices and never wait, and
// every warp is co-resident (cooperative launch), so progress is guaranteed.
struct ItemRef {
  int kind;  // 0 absmax, 1 key encode, 2 value encode
  int layer;
  int idx;
};

__device__ __forceinline__ ItemRef decode_item(const EncodeArgs& a, long long t, int& r) {
  while (r + 1 < a.num_rounds && t >= a.round_start[r + 1]) ++r;
  long long off = t - a.round_start[r];
  const int L = a.num_layers;
  ItemRef it;
  const long long nA = (r < L) ? a.a_items : 0;
  const long long nV = (r < L) ? a.v_items : 0;
  const long long nE = (r >= a.lag && r - a.lag < L) ? a.e_items : 0;
  if (off < nA) {
    it.kind = 0; it.layer = r; it.idx = (int)off;
    return it;
  }
  off -= nA;
  const long long both = 2 * min(nV, nE);
  if (off < both) {
    if ((off & 1) == 0) { it.kind = 2; it.layer = r; it.idx = (int)(off >> 1); }
    else { it.kind = 1; it.layer = r - a.lag; it.idx = (int)(off >> 1); }
    return it;
  }
  off -= both;
  if (nV > nE) { it.kind = 2; it.layer = r; }
  else { it.kind = 1; it.layer = r - a.lag; }
  it.idx = (int)(min(nV, nE) + off);
  return it;
}

template <int D, typename TIn, bool SYM, bool SIGN>
__global__ void __launch_bounds__(kThreads, 2) encode_kernel(const __grid_constant__ EncodeArgs a) {
  __shared__ VSmem<D> vsm[kWarps];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * kWarps + warp;
  const long long nw = (long long)gridDim.x * kWarps;
  const unsigned long long smask = SIGN ? lane_sign_mask<D>(a.sign_bits, lane % VG<D>::TPV) : 0ull;
  int r = 0;
  for (long long t = gw; t < a.total_items; t += nw) {
    const ItemRef it = decode_item(a, t, r);
    if (it.kind == 0) {
      k_absmax_item<TIn>(a, it.layer, it.idx, lane);
    } else if (it.kind == 1) {
      k_encode_item<TIn>(a, it.layer, it.idx, lane);
    } else {
      v_encode_item<D, TIn, SYM, SIGN>(a, it.layer, it.idx, warp, lane, vsm[warp], smask);
    }
  }
}

// ---------------------------------------------------------------------------
// decode (materialise) kernel
// ---------------------------------------------------------------------------


template <typename TOut>
__device__ void k_decode_item(const DecodeArgs& a, int layer, int item, int lane) {
  const int8_t* codes = a.k_codes[layer];
  TOut* out = static_cast<TOut*>(a.k_out[layer]);
  const long long e0 = (long long)item * kKElems;
  const long long n = a.nelem;
  const bool tensor = a.k_mode == PKV_K_TENSOR;
  const float ts = tensor ? __ldg(a.k_scale[layer]) : 0.f;
  if (a.vec_ok) {
#pragma unroll 4
    for (int i = 0; i < kKChunks; ++i) {
      const long long e = e0 + ((long long)i * 32 + lane) * 8;
      if (e >= n) continue;
      const uint2 w = ld_stream_u2(codes + e);
      const float s = tensor ? ts : __half2float(__ldg(a.k_bscale[layer] + (e >> 5)));
      const uint32_t wx = w.x ^ 0x80808080u, wy = w.y ^ 0x80808080u;
      float y[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) y[j] = i8_to_f32(wx, j) * s;
#pragma unroll
      for (int j = 0; j < 4; ++j) y[4 + j] = i8_to_f32(wy, j) * s;
      store8(out + e, y);
    }
  } else {
    for (int i = lane; i < kKElems; i += 32) {
      const long long e = e0 + i;
      if (e >= n) continue;
      const float s = tensor ? ts : __half2float(__ldg(a.k_bscale[layer] + (e >> 5)));
      store1(out + e, (float)codes[e] * s);
    }
  }
}


template <int D, typename TOut, bool SIGN>
__device__ void v_decode_item(const DecodeArgs& a, int layer, int item, int warp, int lane,
                              uint32_t (*stage)[VG<D>::W + 1], float* tbl, unsigned long long smask) {
  using G = VG<D>;
  const int vw = lane / G::TPV, s = lane % G::TPV;
  const uint8_t* packed = a.v_packed[layer];
  const float* scales = a.v_scales[layer];
  TOut* out = static_cast<TOut*>(a.v_out[layer]);
  const long long vbase = (long long)item * VItem<D>::VECS;
  const float sqd = a.sqrt_d32, rsqd = a.rcp_sqrt_d32;
  const uint32_t lane_off = (uint32_t)threadIdx.x * 4u;  // byte offset of this lane's table column
  char* tbl_base = reinterpret_cast<char*>(tbl);

#pragma unroll 1
  for (int itr = 0; itr < VItem<D>::ITERS; ++itr) {
    const long long v = vbase + (long long)itr * G::VPW + vw;
    const bool valid = v < a.nvec;
    // each lane fetches its Q contiguous packed words, then a warp transpose
    // hands every lane the words of its own chunks
    uint32_t q[G::Q];
    if (valid) {
      load_words<G::Q>(packed + v * G::PACKED_BYTES + s * 3 * G::Q, q);
    } else {
#pragma unroll
      for (int j = 0; j < G::Q; ++j) q[j] = 0;
    }
#pragma unroll
    for (int j = 0; j < G::Q; ++j) stage[vw][s * G::Q + j] = q[j];
    __syncwarp();
    uint32_t words[G::NCH];
#pragma unroll
    for (int c = 0; c < G::NCH; ++c) words[c] = stage[vw][s + G::TPV * c];
    __syncwarp();

    // per-lane table of the 8 scaled centroids: table_f32[code] * scale
    // (valuequant.py:232-234), laid out [code][thread] -> conflict-free
    const float sc = valid ? __ldg(scales + v) : 0.f;
#pragma unroll
    for (int k = 0; k < 8; ++k) tbl[k * kThreads + threadIdx.x] = a.cent32[k] * sc;
    float x[G::CPT];
#pragma unroll
    for (int c = 0; c < G::NCH; ++c)
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        // byte address (code << 10) | lane_off  (kThreads * 4 == 1024)
        const uint32_t sh = 3 * e;
        const uint32_t off = (sh <= 10 ? (words[c] << (10 - sh)) : (words[c] >> (sh - 10))) & 0x1c00u;
        x[c * 8 + e] = *reinterpret_cast<const float*>(tbl_base + (off | lane_off));
      }

    fwht_lanes<D>(x, s);

    if (sc >= 0x1p-80f || sc == 0.f) {
#pragma unroll
      for (int i = 0; i < G::CPT; ++i) x[i] = div_sqrt_d<D>(x[i], sqd, rsqd);  // fwht.py:50
    } else {
      // tiny scales can produce subnormal quotients: plain IEEE division
#pragma unroll
      for (int i = 0; i < G::CPT; ++i) x[i] = __fdiv_rn(x[i], sqd);
    }
    if (SIGN) {
#pragma unroll
      for (int i = 0; i < G::CPT; ++i)
        x[i] = __uint_as_float(__float_as_uint(x[i]) ^ ((uint32_t)(smask >> i) << 31));
    }
    if (valid) {
      TOut* o = out + v * D;
#pragma unroll
      for (int c = 0; c < G::NCH; ++c) {
        float y[8];
#pragma unroll
        for (int e = 0; e < 8; ++e) y[e] = x[c * 8 + e];
        store8(o + 8 * (s + G::TPV * c), y);
      }
    }
    __syncwarp();
  }
}

template <int D, typename TOut, bool SIGN>
__global__ void __launch_bounds__(kThreads, 2) decode_kernel(const __grid_constant__ DecodeArgs a) {
  using G = VG<D>;
  __shared__ uint32_t stage[kWarps][G::VPW][G::W + 1];
  __shared__ float tbl[8 * kThreads];
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const long long gw = (long long)blockIdx.x * kWarps + warp;
  const long long nw = (long long)gridDim.x * kWarps;
  const unsigned long long smask = SIGN ? lane_sign_mask<D>(a.sign_bits, lane % G::TPV) : 0ull;
  const long long per_layer = (long long)a.k_items + a.v_items;
  const long long both = 2 * (long long)min(a.k_items, a.v_items);
  for (long long t = gw; t < a.total_items; t += nw) {
    const int layer = (int)(t / per_layer);
    long long off = t - (long long)layer * per_layer;
    // interleave key and value items so memory- and ALU-heavy work overlap
    int kind, idx;
    if (off < both) {
      kind = (int)(off & 1);
      idx = (int)(off >> 1);
    } else {
      off -= both;
      kind = a.k_items > a.v_items ? 0 : 1;
      idx = (int)(min(a.k_items, a.v_items) + off);
    }
    if (kind == 0) k_decode_item<TOut>(a, layer, idx, lane);
    else v_decode_item<D, TOut, SIGN>(a, layer, idx, warp, lane, stage[warp], tbl, smask);
  }
}

// ---------------------------------------------------------------------------
// values at head_dim 1, 2, 4 (legal in the reference: model.py:47-76 only asks
// for a power of two). One thread per packed 24-bit word, i.e. 8 / d whole
// vectors; the encode is the exact fp64 computation in numpy's operation
// order (the same arithmetic as v_replay), the decode the f32 sequence of
// dequantize_v. A tiny-vector path: these shapes carry no bandwidth.
// ---------------------------------------------------------------------------
constexpr int kSmallThreads = 256;

template <typename TIn>
__global__ void __launch_bounds__(kSmallThreads) v_encode_small_kernel(const __grid_constant__ EncodeArgs a) {
  const int D = a.head_dim;
  const long long groups = (a.nelem + 7) / 8;
  const long long total = groups * a.num_layers;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int layer = (int)(t / groups);
    const long long g = t - (long long)layer * groups;
    const TIn* src = static_cast<const TIn*>(a.v_in[layer]);
    uint32_t word = 0;
    bool nonfinite = false;
    for (int e0 = 0; e0 < 8; e0 += D) {
      const long long v = (g * 8 + e0) / D;
      if (v >= a.nvec) break;
      double r[4];
      for (int i = 0; i < D; ++i) {
        const double x = (double)load1(src + v * D + i);
        r[i] = sign_bit(a.sign_bits, i) ? -x : x;  // vals * sign_diagonal
      }
      for (int h = 1; h < D; h <<= 1)  // fwht.py:31-39 in f64
        for (int q = 0; q < D / 2; ++q) {
          const int i = (q / h) * 2 * h + (q % h);
          const double lo = r[i], hi = r[i + h];
          r[i] = __dadd_rn(lo, hi);
          r[i + h] = __dsub_rn(lo, hi);
        }
      const double sq = sqrt((double)D);
      for (int i = 0; i < D; ++i) r[i] = __ddiv_rn(r[i], sq);  // fwht.py:50
      const double S = pairwise_sumsq(r, D);  // np.square then the pairwise mean
      float scale = 0.f;
      if (!(S <= 1.79e308)) {
        nonfinite = true;
      } else {
        const double rms = sqrt(__ddiv_rn(S, (double)D));
        scale = (float)rms;
        const double den = rms > 0.0 ? rms : 1.0;
        for (int i = 0; i < D; ++i) {
          const double z = __ddiv_rn(r[i], den);
          uint32_t c = 0;
#pragma unroll
          for (int k = 0; k < 7; ++k) c += (a.cb.mid64[k] < z) ? 1u : 0u;  // searchsorted 'left'
          if (scale != 0.f) word |= c << (3 * (e0 + i));
        }
      }
      a.v_scales[layer][v] = scale;
    }
    if (nonfinite) {
      word = 0;
      atomicOr(&a.status[layer], PKV_FLAG_V_NONFINITE);
    }
    uint8_t* p = a.v_packed[layer] + 3 * g;
    p[0] = (uint8_t)(word & 0xff);
    p[1] = (uint8_t)((word >> 8) & 0xff);
    p[2] = (uint8_t)((word >> 16) & 0xff);
  }
}

template <typename TOut>
__global__ void __launch_bounds__(kSmallThreads) v_decode_small_kernel(const __grid_constant__ DecodeArgs a) {
  const int D = a.head_dim;
  const long long groups = (a.nelem + 7) / 8;
  const long long total = groups * a.num_layers;
  for (long long t = blockIdx.x * (long long)blockDim.x + threadIdx.x; t < total;
       t += (long long)gridDim.x * blockDim.x) {
    const int layer = (int)(t / groups);
    const long long g = t - (long long)layer * groups;
    const uint8_t* p = a.v_packed[layer] + 3 * g;
    const uint32_t word = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16);
    TOut* out = static_cast<TOut*>(a.v_out[layer]);
    for (int e0 = 0; e0 < 8; e0 += D) {
      const long long v = (g * 8 + e0) / D;
      if (v >= a.nvec) break;
      const float sc = a.v_scales[layer][v];
      float y[4];
      for (int i = 0; i < D; ++i) y[i] = __fmul_rn(a.cent32[(word >> (3 * (e0 + i))) & 7u], sc);  // table[code] * scale
      for (int h = 1; h < D; h <<= 1)
        for (int q = 0; q < D / 2; ++q) {
          const int i = (q / h) * 2 * h + (q % h);
          const float lo = y[i], hi = y[i + h];
          y[i] = __fadd_rn(lo, hi);
          y[i + h] = __fsub_rn(lo, hi);
        }
      for (int i = 0; i < D; ++i) {
        float x = __fdiv_rn(y[i], a.sqrt_d32);  // fwht.py:50 in f32
        if (sign_bit(a.sign_bits, i)) x = -x;
        store1(out + v * D + i, x);
      }
    }
  }
}

template <typename K>
int launch_small(K kernel, const void* args, long long work, cudaStream_t st) {
  if (work <= 0) return PKV_OK;
  const long long grid = std::min<long long>((work + kSmallThreads - 1) / kSmallThreads, (long long)sm_count() * 8);
  void* params[] = {const_cast<void*>(args)};
  return pkv::cuda_ok(cudaLaunchKernel((const void*)kernel, dim3((unsigned)grid), dim3(kSmallThreads), params, 0, st),
                      "cudaLaunchKernel")
             ? PKV_OK
             : PKV_ERR_CUDA;
}

// ---------------------------------------------------------------------------
// canonical codes <-> packed payload
// ---------------------------------------------------------------------------
__global__ void unpack_kernel(const uint8_t* __restrict__ packed, long long count,
                              uint8_t* __restrict__ codes) {
  const long long groups = (count + 7) / 8;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < groups;
       g += (long long)gridDim.x * blockDim.x) {
    const uint32_t w = (uint32_t)packed[3 * g] | ((uint32_t)packed[3 * g + 1] << 8) |
                       ((uint32_t)packed[3 * g + 2] << 16);
    for (int e = 0; e < 8; ++e) {
      const long long i = 8 * g + e;
      if (i < count) codes[i] = (uint8_t)((w >> (3 * e)) & 7u);
    }
  }
}

__global__ void pack_kernel(const uint8_t* __restrict__ codes, long long count,
                            uint8_t* __restrict__ packed, uint32_t* bad) {
  const long long groups = (count + 7) / 8;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < groups;
       g += (long long)gridDim.x * blockDim.x) {
    uint32_t w = 0;
    bool oob = false;
    for (int e = 0; e < 8; ++e) {
      const long long i = 8 * g + e;
      const uint32_t c = i < count ? codes[i] : 0u;
      oob |= c > 7u;
      w |= (c & 7u) << (3 * e);
    }
    if (oob && bad) atomicOr(bad, PKV_FLAG_BAD_CODE);
    packed[3 * g] = (uint8_t)(w & 0xff);
    packed[3 * g + 1] = (uint8_t)((w >> 8) & 0xff);
    packed[3 * g + 2] = (uint8_t)((w >> 16) & 0xff);
  }
}

// Exhaustive check of div_sqrt_d<D> against IEEE division for every f32
// mantissa in [1, 2) (exponent scaling is exact in the normal range).
template <int D>
__global__ void selftest_div_kernel(uint32_t* mismatches) {
  const float c = (float)sqrt((double)D);
  const float r = 1.0f / c;
  uint32_t bad = 0;
  for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < (1u << 23); m += gridDim.x * blockDim.x) {
    const float x = __uint_as_float(0x3f800000u | m);
    bad += __float_as_uint(div_sqrt_d<D>(x, c, r)) != __float_as_uint(__fdiv_rn(x, c));
    bad += __float_as_uint(div_sqrt_d<D>(-x * 0x1p-60f, c, r)) != __float_as_uint(__fdiv_rn(-x * 0x1p-60f, c));
  }
  if (bad) atomicAdd(mismatches, bad);
}

// The same for div127 (block32 key scales).
__global__ void selftest_div127_kernel(uint32_t* mismatches) {
  uint32_t bad = 0;
  for (uint32_t m = blockIdx.x * blockDim.x + threadIdx.x; m < (1u << 23); m += gridDim.x * blockDim.x) {
    const float x = __uint_as_float(0x3f800000u | m);
    bad += __float_as_uint(div127(x)) != __float_as_uint(__fdiv_rn(x, 127.0f));
    bad += __float_as_uint(div127(x * 0x1p-90f)) != __float_as_uint(__fdiv_rn(x * 0x1p-90f, 127.0f));
    bad += __float_as_uint(div127(x * 0x1p+90f)) != __float_as_uint(__fdiv_rn(x * 0x1p+90f, 127.0f));
  }
  if (bad) atomicAdd(mismatches, bad);
}

}  // namespace pkv

// ===========================================================================
// host side: C ABI
// ===========================================================================
namespace {

using namespace pkv;







int blocks_per_sm(const void* fn) {
  int per_sm = 1;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, 0) != cudaSuccess || per_sm < 1)
    per_sm = 1;
  return per_sm;
}

template <int D, typename TIn, bool SYM, bool SIGN>
int launch_encode(EncodeArgs& a, cudaStream_t st) {
  auto fn = encode_kernel<D, TIn, SYM, SIGN>;
  const int per_sm = blocks_per_sm((const void*)fn);
  long long grid = (long long)sm_count() * per_sm;
  const long long need = (a.total_items + kWarps - 1) / kWarps;
  if (grid > need) grid = need;
  if (grid < 1) return PKV_OK;
  void* params[] = {(void*)&a};
  const cudaError_t e = cudaLaunchCooperativeKernel((const void*)fn, dim3((unsigned)grid), dim3(kThreads),
                                                    params, 0, st);
  return pkv::cuda_ok(e, "cudaLaunchCooperativeKernel") ? PKV_OK : PKV_ERR_CUDA;
}

template <int D, typename TIn>
int launch_encode_d(EncodeArgs& a, cudaStream_t st, bool sym, bool sign) {
  if (sym) return sign ? launch_encode<D, TIn, true, true>(a, st) : launch_encode<D, TIn, true, false>(a, st);
  return sign ? launch_encode<D, TIn, false, true>(a, st) : launch_encode<D, TIn, false, false>(a, st);
}

template <typename TIn>
int dispatch_encode(EncodeArgs& a, cudaStream_t st, bool do_v, bool sym, bool sign) {
  switch (do_v ? a.head_dim : 128) {
    case 8: return launch_encode_d<8, TIn>(a, st, sym, sign);
    case 16: return launch_encode_d<16, TIn>(a, st, sym, sign);
    case 32: return launch_encode_d<32, TIn>(a, st, sym, sign);
    case 64: return launch_encode_d<64, TIn>(a, st, sym, sign);
    case 128: return launch_encode_d<128, TIn>(a, st, sym, sign);
    case 256: return launch_encode_d<256, TIn>(a, st, sym, sign);
    default: return PKV_ERR_UNSUPPORTED_HEAD_DIM;
  }
}

template <int D, typename TOut, bool SIGN>
int launch_decode(DecodeArgs& a, cudaStream_t st) {
  auto fn = decode_kernel<D, TOut, SIGN>;
  long long grid = (long long)sm_count() * blocks_per_sm((const void*)fn);
  const long long need = (a.total_items + kWarps - 1) / kWarps;
  if (grid > need) grid = need;
  if (grid < 1) return PKV_OK;
  fn<<<(unsigned)grid, kThreads, 0, st>>>(a);
  return pkv::cuda_ok(cudaGetLastError(), "kernel launch") ? PKV_OK : PKV_ERR_CUDA;
}

template <int D, typename TOut>
int launch_decode_d(DecodeArgs& a, cudaStream_t st, bool sign) {
  return sign ? launch_decode<D, TOut, true>(a, st) : launch_decode<D, TOut, false>(a, st);
}

template <typename TOut>
int dispatch_decode(DecodeArgs& a, cudaStream_t st, bool do_v, bool sign) {
  switch (do_v ? a.head_dim : 128) {
    case 8: return launch_decode_d<8, TOut>(a, st, sign);
    case 16: return launch_decode_d<16, TOut>(a, st, sign);
    case 32: return launch_decode_d<32, TOut>(a, st, sign);
    case 64: return launch_decode_d<64, TOut>(a, st, sign);
    case 128: return launch_decode_d<128, TOut>(a, st, sign);
    case 256: return launch_decode_d<256, TOut>(a, st, sign);
    default: return PKV_ERR_UNSUPPORTED_HEAD_DIM;
  }
}


template <int D>
int v_items_for(long long nvec) {
  return (int)((nvec + VItem<D>::VECS - 1) / VItem<D>::VECS);
}

int v_items_dispatch(int d, long long nvec) {
  switch (d) {
    case 8: return v_items_for<8>(nvec);
    case 16: return v_items_for<16>(nvec);
    case 32: return v_items_for<32>(nvec);
    case 64: return v_items_for<64>(nvec);
    case 128: return v_items_for<128>(nvec);
    case 256: return v_items_for<256>(nvec);
    default: return -1;
  }
}

// alignment the value kernels need for the packed stream of head_dim d
uintptr_t packed_align(int d) {
  const int q = (d / 8) / (d >= 256 ? 4 : (d >= 16 ? 2 : 1));
  return q >= 8 ? 8 : (q >= 4 ? 4 : (q >= 2 ? 2 : 1));
}

}  // namespace

namespace {
// head_dim 1, 2, 4: values through the thread-per-word kernels above
bool v_small(int d) { return d < 8; }
// PKV_CODEC_PATH=warp forces the warp-granular kernels (debug / A-B timing).
bool stream_enabled() { return !tuning().codec_warp; }
bool stream_fallback(int rc) { return rc == PKV_ERR_ALIGNMENT || rc == PKV_ERR_UNSUPPORTED_HEAD_DIM; }
}  // namespace

extern "C" {

int pkv_abi_version(void) { return PKV_ABI_VERSION; }

const char* pkv_status_string(int status) {
  switch (status) {
    case PKV_OK: return "ok";
    case PKV_ERR_INVALID_ARG: return "invalid argument";
    case PKV_ERR_UNSUPPORTED_HEAD_DIM: return "head_dim not supported by the value kernels (1..256, power of two)";
    case PKV_ERR_CUDA: return "CUDA launch error";
    case PKV_ERR_WORKSPACE: return "workspace too small";
    case PKV_ERR_ALIGNMENT: return "misaligned pointer";
    case PKV_ERR_UNSUPPORTED_CODEBOOK: return "codebook must have 8 strictly increasing finite centroids";
    default: return "unknown status";
  }
}

int pkv_v_head_dim_supported(int d) {
  return d == 1 || d == 2 || d == 4 || d == 8 || d == 16 || d == 32 || d == 64 || d == 128 || d == 256;
}

size_t pkv_encode_workspace_bytes(int num_layers, int64_t num_vectors, int head_dim) {
  if (num_layers < 0 || num_vectors < 0 || head_dim < 1) return 0;
  const int l = std::min(num_layers, (int)PKV_MAX_LAYERS_PER_LAUNCH);
  const size_t warp_path = (size_t)(2 * l + 2) * sizeof(uint32_t);
  return std::max(warp_path, stream::workspace_bytes(l, num_vectors, head_dim));
}

int pkv_encode(int num_layers, int64_t num_vectors, int head_dim, int in_dtype,
               const void* const* k_in, const void* const* v_in, int k_mode,
               int8_t* const* k_codes, float* const* k_scale, uint16_t* const* k_bscale,
               uint8_t* const* v_packed, float* const* v_scales, const double* centroids_host,
               const uint32_t* sign_bits_host, uint32_t* status, uint32_t* replay_count,
               const uint32_t* k_layer_max, void* workspace, size_t workspace_bytes, void* stream) {
  if (num_layers < 0 || num_vectors < 0 || head_dim < 1) return PKV_ERR_INVALID_ARG;
  if (in_dtype != PKV_F32 && in_dtype != PKV_BF16) return PKV_ERR_INVALID_ARG;
  if (k_mode != PKV_K_TENSOR && k_mode != PKV_K_BLOCK32) return PKV_ERR_INVALID_ARG;
  if (!status) return PKV_ERR_INVALID_ARG;
  const bool do_k = k_in != nullptr, do_v = v_in != nullptr;
  if (num_layers == 0 || num_vectors == 0 || (!do_k && !do_v)) return PKV_OK;
  if (do_v && !pkv_v_head_dim_supported(head_dim)) return PKV_ERR_UNSUPPORTED_HEAD_DIM;
  if (workspace_bytes < pkv_encode_workspace_bytes(num_layers, num_vectors, head_dim) || !workspace)
    return PKV_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long nelem = (long long)num_vectors * head_dim;
  const bool small_v = do_v && v_small(head_dim);

  for (int l0 = 0; l0 < num_layers; l0 += PKV_MAX_LAYERS_PER_LAUNCH) {
    const int L = std::min(num_layers - l0, (int)PKV_MAX_LAYERS_PER_LAUNCH);
    EncodeArgs a;
    std::memset(&a, 0, sizeof(a));
    a.num_layers = L;
    a.head_dim = head_dim;
    a.k_mode = k_mode;
    a.nvec = num_vectors;
    a.nelem = nelem;
    a.delta = guard_delta(head_dim);
    const bool sign = fill_sign(sign_bits_host, head_dim, a.sign_bits);
    if (do_v && !fill_codebook(centroids_host, a.cb)) return PKV_ERR_UNSUPPORTED_CODEBOOK;
    a.status = status + l0;
    a.replay_count = replay_count;
    a.ws = static_cast<uint32_t*>(workspace);
    bool ok = (nelem % 8) == 0;
    for (int l = 0; l < L; ++l) {
      if (do_k) {
        a.k_in[l] = k_in[l0 + l];
        a.k_codes[l] = k_codes[l0 + l];
        if (!a.k_in[l] || !a.k_codes[l]) return PKV_ERR_INVALID_ARG;
        if (k_mode == PKV_K_TENSOR) {
          a.k_scale[l] = k_scale ? k_scale[l0 + l] : nullptr;
          if (!a.k_scale[l]) return PKV_ERR_INVALID_ARG;
        } else {
          a.k_bscale[l] = k_bscale ? reinterpret_cast<__half*>(k_bscale[l0 + l]) : nullptr;
          if (!a.k_bscale[l]) return PKV_ERR_INVALID_ARG;
        }
        ok = ok && aligned(a.k_in[l], 16) && aligned(a.k_codes[l], 8);
      }
      if (do_v) {
        a.v_in[l] = v_in[l0 + l];
        a.v_packed[l] = v_packed ? v_packed[l0 + l] : nullptr;
        a.v_scales[l] = v_scales ? v_scales[l0 + l] : nullptr;
        if (!a.v_in[l] || !a.v_packed[l] || !a.v_scales[l]) return PKV_ERR_INVALID_ARG;
        // the value kernels use 16 B chunk loads and word-aligned packed stores
        // (the head_dim < 8 kernels load and store scalars)
        if (!small_v && (!aligned(a.v_in[l], 16) || !aligned(a.v_packed[l], packed_align(head_dim)) ||
                         !aligned(a.v_scales[l], 4)))
          return PKV_ERR_ALIGNMENT;
      }
    }
    if (stream_enabled() && !small_v) {
      stream::EncodeRequest q;
      std::memset(&q, 0, sizeof(q));
      q.num_layers = L;
      q.num_vectors = num_vectors;
      q.head_dim = head_dim;
      q.in_dtype = in_dtype;
      q.k_mode = k_mode;
      q.k_in = do_k ? k_in + l0 : nullptr;
      q.v_in = do_v ? v_in + l0 : nullptr;
      q.k_codes = do_k ? k_codes + l0 : nullptr;
      q.k_scale = (do_k && k_scale) ? k_scale + l0 : nullptr;
      q.k_bscale = (do_k && k_bscale) ? k_bscale + l0 : nullptr;
      q.v_packed = do_v ? v_packed + l0 : nullptr;
      q.v_scales = do_v ? v_scales + l0 : nullptr;
      q.cb = a.cb;
      std::memcpy(q.sign_bits, a.sign_bits, sizeof(q.sign_bits));
      q.sign = sign;
      q.status = status + l0;
      q.replay_count = replay_count;
      q.k_max_ext = (do_k && k_mode == PKV_K_TENSOR && k_layer_max) ? k_layer_max + l0 : nullptr;
      q.ws = workspace;
      q.ws_bytes = workspace_bytes;
      const int src = stream::encode(q, st);
      if (src == PKV_OK) continue;
      if (!stream_fallback(src)) return src;
    }
    a.vec_ok = ok ? 1 : 0;
    const int k_items = do_k ? (int)((nelem + kKElems - 1) / kKElems) : 0;
    a.e_items = k_items;
    const bool ext_max = do_k && k_mode == PKV_K_TENSOR && k_layer_max;
    a.a_items = (do_k && k_mode == PKV_K_TENSOR && !ext_max) ? k_items : 0;
    a.v_items = (do_v && !small_v) ? v_items_dispatch(head_dim, num_vectors) : 0;
    // lag: keep >= ~2 waves of warps between a layer's absmax and its key encode
    const long long round = (long long)a.a_items + a.v_items + a.e_items;
    const long long warps = (long long)sm_count() * 2 * kWarps;
    int lag = 1;
    if (a.a_items > 0) {
      while (lag < 8 && (long long)lag * round < 2 * warps) ++lag;
    }
    a.lag = lag;
    a.num_rounds = L + lag;
    long long acc = 0;
    for (int r = 0; r < a.num_rounds; ++r) {
      a.round_start[r] = acc;
      if (r < L) acc += a.a_items + a.v_items;
      if (r >= lag && r - lag < L) acc += a.e_items;
    }
    a.round_start[a.num_rounds] = acc;
    a.total_items = acc;
    if (!pkv::cuda_ok(cudaMemsetAsync(workspace, 0, (size_t)(2 * L + 2) * sizeof(uint32_t), st), "cudaMemsetAsync")) return PKV_ERR_CUDA;
    // external per-layer maxima: the key encode reads them where the absmax
    // items would have left theirs (and, with a_items == 0, never waits)
    if (ext_max && !pkv::cuda_ok(cudaMemcpyAsync(workspace, k_layer_max + l0, (size_t)L * sizeof(uint32_t),
                                                 cudaMemcpyDeviceToDevice, st),
                                 "cudaMemcpyAsync"))
      return PKV_ERR_CUDA;
    const bool sym = do_v ? a.cb.symmetric != 0 : true;
    const bool tiled_v = do_v && !small_v;
    int rc = in_dtype == PKV_F32 ? dispatch_encode<float>(a, st, tiled_v, sym, sign)
                                 : dispatch_encode<__nv_bfloat16>(a, st, tiled_v, sym, sign);
    if (rc == PKV_OK && small_v) {
      const long long work = (long long)L * ((nelem + 7) / 8);
      rc = in_dtype == PKV_F32 ? launch_small(v_encode_small_kernel<float>, &a, work, st)
                               : launch_small(v_encode_small_kernel<__nv_bfloat16>, &a, work, st);
    }
    if (rc != PKV_OK) return rc;
  }
  return PKV_OK;
}

int pkv_decode(int num_layers, int64_t num_vectors, int head_dim, int out_dtype, int k_mode,
               const int8_t* const* k_codes, const float* const* k_scale,
               const uint16_t* const* k_bscale, const uint8_t* const* v_packed,
               const float* const* v_scales, const double* centroids_host,
               const uint32_t* sign_bits_host, void* const* k_out, void* const* v_out,
               void* stream) {
  if (num_layers < 0 || num_vectors < 0 || head_dim < 1) return PKV_ERR_INVALID_ARG;
  if (out_dtype != PKV_F32 && out_dtype != PKV_BF16) return PKV_ERR_INVALID_ARG;
  if (k_mode != PKV_K_TENSOR && k_mode != PKV_K_BLOCK32) return PKV_ERR_INVALID_ARG;
  const bool do_k = k_codes != nullptr && k_out != nullptr;
  const bool do_v = v_packed != nullptr && v_out != nullptr;
  if (num_layers == 0 || num_vectors == 0 || (!do_k && !do_v)) return PKV_OK;
  if (do_v && !pkv_v_head_dim_supported(head_dim)) return PKV_ERR_UNSUPPORTED_HEAD_DIM;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const long long nelem = (long long)num_vectors * head_dim;
  const bool small_v = do_v && v_small(head_dim);
  for (int l0 = 0; l0 < num_layers; l0 += PKV_MAX_LAYERS_PER_LAUNCH) {
    const int L = std::min(num_layers - l0, (int)PKV_MAX_LAYERS_PER_LAUNCH);
    DecodeArgs a;
    std::memset(&a, 0, sizeof(a));
    a.num_layers = L;
    a.head_dim = head_dim;
    a.k_mode = k_mode;
    a.nvec = num_vectors;
    a.nelem = nelem;
    a.sqrt_d32 = (float)std::sqrt((double)head_dim);  // np.float32(np.sqrt(d))
    a.rcp_sqrt_d32 = 1.0f / a.sqrt_d32;
    const bool sign = fill_sign(sign_bits_host, head_dim, a.sign_bits);
    if (do_v) {
      Codebook3 cb;
      if (!fill_codebook(centroids_host, cb)) return PKV_ERR_UNSUPPORTED_CODEBOOK;
      for (int i = 0; i < 8; ++i) a.cent32[i] = cb.cent32[i];
    }
    bool ok = (nelem % 8) == 0;
    for (int l = 0; l < L; ++l) {
      if (do_k) {
        a.k_codes[l] = k_codes[l0 + l];
        a.k_out[l] = k_out[l0 + l];
        if (k_mode == PKV_K_TENSOR) a.k_scale[l] = k_scale ? k_scale[l0 + l] : nullptr;
        else a.k_bscale[l] = k_bscale ? reinterpret_cast<const __half*>(k_bscale[l0 + l]) : nullptr;
        if (!a.k_codes[l] || !a.k_out[l] || (k_mode == PKV_K_TENSOR ? !a.k_scale[l] : !a.k_bscale[l]))
          return PKV_ERR_INVALID_ARG;
        ok = ok && aligned(a.k_codes[l], 8) && aligned(a.k_out[l], 16);
      }
      if (do_v) {
        a.v_packed[l] = v_packed[l0 + l];
        a.v_scales[l] = v_scales ? v_scales[l0 + l] : nullptr;
        a.v_out[l] = v_out[l0 + l];
        if (!a.v_packed[l] || !a.v_scales[l] || !a.v_out[l]) return PKV_ERR_INVALID_ARG;
        if (!small_v && (!aligned(a.v_out[l], 16) || !aligned(a.v_packed[l], packed_align(head_dim))))
          return PKV_ERR_ALIGNMENT;
      }
    }
    if (stream_enabled() && !small_v) {
      stream::DecodeRequest q;
      std::memset(&q, 0, sizeof(q));
      q.num_layers = L;
      q.num_vectors = num_vectors;
      q.head_dim = head_dim;
      q.out_dtype = out_dtype;
      q.k_mode = k_mode;
      q.k_codes = do_k ? k_codes + l0 : nullptr;
      q.k_scale = (do_k && k_scale) ? k_scale + l0 : nullptr;
      q.k_bscale = (do_k && k_bscale) ? k_bscale + l0 : nullptr;
      q.k_out = do_k ? k_out + l0 : nullptr;
      q.v_packed = do_v ? v_packed + l0 : nullptr;
      q.v_scales = do_v ? v_scales + l0 : nullptr;
      q.v_out = do_v ? v_out + l0 : nullptr;
      std::memcpy(q.cent32, a.cent32, sizeof(q.cent32));
      std::memcpy(q.sign_bits, a.sign_bits, sizeof(q.sign_bits));
      q.sign = sign;
      const int src = stream::decode(q, st);
      if (src == PKV_OK) continue;
      if (!stream_fallback(src)) return src;
    }
    a.vec_ok = ok ? 1 : 0;
    a.k_items = do_k ? (int)((nelem + kKElems - 1) / kKElems) : 0;
    a.v_items = (do_v && !small_v) ? v_items_dispatch(head_dim, num_vectors) : 0;
    a.total_items = (long long)L * (a.k_items + a.v_items);
    int rc = out_dtype == PKV_F32 ? dispatch_decode<float>(a, st, do_v && !small_v, sign)
                                  : dispatch_decode<__nv_bfloat16>(a, st, do_v && !small_v, sign);
    if (rc == PKV_OK && small_v) {
      const long long work = (long long)L * ((nelem + 7) / 8);
      rc = out_dtype == PKV_F32 ? launch_small(v_decode_small_kernel<float>, &a, work, st)
                                : launch_small(v_decode_small_kernel<__nv_bfloat16>, &a, work, st);
    }
    if (rc != PKV_OK) return rc;
  }
  return PKV_OK;
}

int pkv_unpack_codes(const uint8_t* packed, int64_t count, uint8_t* codes, void* stream) {
  if (count < 0 || (count > 0 && (!packed || !codes))) return PKV_ERR_INVALID_ARG;
  if (count == 0) return PKV_OK;
  const long long groups = (count + 7) / 8;
  const int grid = (int)std::min<long long>((groups + 255) / 256, 148LL * 16);
  unpack_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(packed, count, codes);
  return pkv::cuda_ok(cudaGetLastError(), "kernel launch") ? PKV_OK : PKV_ERR_CUDA;
}

int pkv_pack_codes(const uint8_t* codes, int64_t count, uint8_t* packed, uint32_t* bad_code,
                   void* stream) {
  if (count < 0 || (count > 0 && (!packed || !codes))) return PKV_ERR_INVALID_ARG;
  if (count == 0) return PKV_OK;
  const long long groups = (count + 7) / 8;
  const int grid = (int)std::min<long long>((groups + 255) / 256, 148LL * 16);
  pack_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(codes, count, packed, bad_code);
  return pkv::cuda_ok(cudaGetLastError(), "kernel launch") ? PKV_OK : PKV_ERR_CUDA;
}

int64_t pkv_selftest(int what, void* scratch, size_t scratch_bytes, void* stream) {
  if (what != PKV_SELFTEST_DIVISION) return PKV_ERR_INVALID_ARG;
  if (!scratch || scratch_bytes < 4 * sizeof(uint32_t)) return PKV_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  uint32_t* cnt = static_cast<uint32_t*>(scratch);
  if (!pkv::cuda_ok(cudaMemsetAsync(cnt, 0, 4 * sizeof(uint32_t), st), "cudaMemsetAsync")) return PKV_ERR_CUDA;
  selftest_div_kernel<8><<<1024, 256, 0, st>>>(cnt + 0);
  selftest_div_kernel<32><<<1024, 256, 0, st>>>(cnt + 1);
  selftest_div_kernel<128><<<1024, 256, 0, st>>>(cnt + 2);
  selftest_div127_kernel<<<1024, 256, 0, st>>>(cnt + 3);
  uint32_t host[4] = {0, 0, 0, 0};
  if (!pkv::cuda_ok(cudaMemcpyAsync(host, cnt, sizeof(host), cudaMemcpyDeviceToHost, st), "cudaMemcpyAsync")) return PKV_ERR_CUDA;
  if (!pkv::cuda_ok(cudaStreamSynchronize(st), "cudaStreamSynchronize")) return PKV_ERR_CUDA;
  return (int64_t)host[0] + host[1] + host[2] + host[3];
}

}  // extern "C"
