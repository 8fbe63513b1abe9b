// Shared device helpers for the PolyKV B200 kernels (sm_100a).
//
// Numerics notes:
//  * The value rotation is the Sylvester FWHT with stages half = 1, 2, 4, ...
//    and butterflies lo' = lo + hi, hi' = lo - hi (kvpool/fwht.py:24-41).
//    The same stage order is used in every kernel, so the fp32 inverse
//    rotation on the read side is bit-identical to numpy's.
//  * Nothing here may be compiled with --use_fast_math: IEEE division and
//    square root are required (kvpool/fwht.py:50, valuequant.py:207-209).
#pragma once

#include <cuda_bf16.h>
#include <cuda_fp16.h>
#include <cuda_runtime.h>
#include <stdint.h>

namespace pkv {

constexpr int kThreads = 256;
constexpr int kMaxLayers = 64;

// ---- value geometry: how a head vector of D coordinates maps onto lanes ----
// A vector is split over TPV consecutive lanes. Lane s of a vector holds the
// 8-coordinate chunks s, s+TPV, s+2*TPV, ... so that coordinate
//     i = 8 * (s + TPV * c) + e,     e in [0,8), c in [0, NCH)
// Coordinate bits 0-2 (e) and the high bits (c) are rotated in registers;
// the log2(TPV) bits in between go through warp shuffles. Global loads of a
// chunk are 16 B (bf16) / 32 B (f32) and the TPV lanes of a vector read
// contiguous bytes, so every warp-wide load instruction is sector-complete.
template <int D>
struct VG {
  static_assert(D == 8 || D == 16 || D == 32 || D == 64 || D == 128 || D == 256,
                "unsupported head_dim");
  static constexpr int TPV = D >= 256 ? 4 : (D >= 16 ? 2 : 1);
  static constexpr int CPT = D / TPV;  // coordinates per lane
  static constexpr int NCH = CPT / 8;  // chunks per lane
  static constexpr int LB = TPV == 4 ? 2 : (TPV == 2 ? 1 : 0);
  static constexpr int W = D / 8;      // 24-bit packed words per vector
  static constexpr int Q = W / TPV;    // words per lane after redistribution
  static constexpr int VPW = 32 / TPV; // vectors per warp
  static constexpr int VPI = kThreads / TPV;  // vectors per CTA iteration
  static constexpr int PACKED_BYTES = 3 * D / 8;
  static constexpr int LOG2D = D == 8 ? 3 : D == 16 ? 4 : D == 32 ? 5 : D == 64 ? 6 : D == 128 ? 7 : 8;
};

// ---- loads / stores -------------------------------------------------------
__device__ __forceinline__ uint4 ld_stream_u4(const void* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.u32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint2 ld_stream_u2(const void* p) {
  uint2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.u32 {%0,%1}, [%2];"
               : "=r"(r.x), "=r"(r.y)
               : "l"(p));
  return r;
}
__device__ __forceinline__ uint32_t ld_stream_u1(const void* p) {
  uint32_t r;
  asm volatile("ld.global.nc.L1::no_allocate.u32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_u4(void* p, uint4 v) {
  asm volatile("st.global.v4.u32 [%0], {%1,%2,%3,%4};" ::"l"(p), "r"(v.x), "r"(v.y),
               "r"(v.z), "r"(v.w)
               : "memory");
}
__device__ __forceinline__ void st_u2(void* p, uint2 v) {
  asm volatile("st.global.v2.u32 [%0], {%1,%2};" ::"l"(p), "r"(v.x), "r"(v.y) : "memory");
}

__device__ __forceinline__ float bf16lo(uint32_t w) { return __uint_as_float(w << 16); }
__device__ __forceinline__ float bf16hi(uint32_t w) { return __uint_as_float(w & 0xffff0000u); }

// 8 consecutive input elements -> f32 registers (exact for both dtypes).
__device__ __forceinline__ void load8(const float* p, float (&x)[8]) {
  uint4 a = ld_stream_u4(p), b = ld_stream_u4(p + 4);
  x[0] = __uint_as_float(a.x); x[1] = __uint_as_float(a.y);
  x[2] = __uint_as_float(a.z); x[3] = __uint_as_float(a.w);
  x[4] = __uint_as_float(b.x); x[5] = __uint_as_float(b.y);
  x[6] = __uint_as_float(b.z); x[7] = __uint_as_float(b.w);
}
__device__ __forceinline__ void load8(const __nv_bfloat16* p, float (&x)[8]) {
  uint4 a = ld_stream_u4(p);
  x[0] = bf16lo(a.x); x[1] = bf16hi(a.x); x[2] = bf16lo(a.y); x[3] = bf16hi(a.y);
  x[4] = bf16lo(a.z); x[5] = bf16hi(a.z); x[6] = bf16lo(a.w); x[7] = bf16hi(a.w);
}
__device__ __forceinline__ float load1(const float* p) { return __ldg(p); }
__device__ __forceinline__ float load1(const __nv_bfloat16* p) {
  return __bfloat162float(__ldg(p));
}

// 8 f32 values -> output dtype at p (16 B for bf16, 32 B for f32).
__device__ __forceinline__ void store8(float* p, const float (&y)[8]) {
  st_u4(p, make_uint4(__float_as_uint(y[0]), __float_as_uint(y[1]), __float_as_uint(y[2]),
                      __float_as_uint(y[3])));
  st_u4(p + 4, make_uint4(__float_as_uint(y[4]), __float_as_uint(y[5]),
                          __float_as_uint(y[6]), __float_as_uint(y[7])));
}
__device__ __forceinline__ uint32_t pack_bf16x2(float lo, float hi) {
  __nv_bfloat162 h = __floats2bfloat162_rn(lo, hi);  // RNE, == round_to_bfloat16
  return *reinterpret_cast<uint32_t*>(&h);
}
__device__ __forceinline__ void store8(__nv_bfloat16* p, const float (&y)[8]) {
  st_u4(p, make_uint4(pack_bf16x2(y[0], y[1]), pack_bf16x2(y[2], y[3]),
                      pack_bf16x2(y[4], y[5]), pack_bf16x2(y[6], y[7])));
}
__device__ __forceinline__ void store1(float* p, float v) { *p = v; }
__device__ __forceinline__ void store1(__nv_bfloat16* p, float v) { *p = __float2bfloat16_rn(v); }

// ---- the Sylvester FWHT over one lane-distributed vector (fp32) ------------
// x[c*8+e] holds coordinate 8*(s + TPV*c) + e. Stages run half = 1, 2, 4, ...
// exactly like kvpool/fwht.py:31-39, so results are bit-identical to numpy.
template <int D>
__device__ __forceinline__ void fwht_lanes(float* x, int s) {
  using G = VG<D>;
#pragma unroll
  for (int h = 1; h < 8; h <<= 1) {
#pragma unroll
    for (int c = 0; c < G::NCH; ++c) {
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        if (e & h) continue;
        float a = x[c * 8 + e], b = x[c * 8 + e + h];
        x[c * 8 + e] = a + b;
        x[c * 8 + e + h] = a - b;
      }
    }
  }
#pragma unroll
  for (int lb = 0; lb < G::LB; ++lb) {
    // lo lane (bit clear) keeps lo + hi = mine + partner; hi lane keeps
    // lo - hi = partner - mine. fmaf(+-1, mine, partner) is one rounding of
    // the exact sum/difference, i.e. identical to numpy's add/subtract.
    const float sg = ((s >> lb) & 1) ? -1.f : 1.f;
#pragma unroll
    for (int i = 0; i < G::CPT; ++i) {
      float p = __shfl_xor_sync(0xffffffffu, x[i], 1 << lb);
      x[i] = fmaf(sg, x[i], p);
    }
  }
#pragma unroll
  for (int hc = 1; hc < G::NCH; hc <<= 1) {
#pragma unroll
    for (int c = 0; c < G::NCH; ++c) {
      if (c & hc) continue;
#pragma unroll
      for (int e = 0; e < 8; ++e) {
        float a = x[c * 8 + e], b = x[(c + hc) * 8 + e];
        x[c * 8 + e] = a + b;
        x[(c + hc) * 8 + e] = a - b;
      }
    }
  }
}

// sign diagonal bit for coordinate i (bit set = multiply by -1)
__device__ __forceinline__ bool sign_bit(const uint32_t* bits, int i) {
  return (bits[i >> 5] >> (i & 31)) & 1u;
}

// numpy's pairwise summation of v[i]*v[i] over n contiguous doubles
// (numpy/_core/src/umath/loops_utils.h.src, pairwise_sum): n < 8 sequential,
// n <= 128 eight interleaved accumulators, larger n split at n/2 rounded
// down to a multiple of 8. This is the reduction order behind
// np.mean(np.square(rot), axis=-1) in kvpool/valuequant.py:207.
//
// np.square rounds every product before the pairwise add, so each square and
// each add is written with an explicit rounding intrinsic: nvcc would
// otherwise contract `r += v * v` into one DFMA (a single rounding), which
// differs from numpy in the last bit for ~1 in 5 vectors and can flip an f32
// scale that sits on a rounding boundary -- exactly the vectors the replay
// exists for. tests/test_capi.py checks the SASS of every replay for DFMA.
__device__ __forceinline__ double sq_rn(double x) { return __dmul_rn(x, x); }

__device__ inline double pairwise_block8(const double* v, int n) {
  // n >= 8: eight accumulators, then the remainder sequentially
  double r[8];
#pragma unroll
  for (int j = 0; j < 8; ++j) r[j] = sq_rn(v[j]);
  int i = 8;
  for (; i < n - (n % 8); i += 8)
#pragma unroll
    for (int j = 0; j < 8; ++j) r[j] = __dadd_rn(r[j], sq_rn(v[i + j]));
  double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                         __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
  for (; i < n; ++i) res = __dadd_rn(res, sq_rn(v[i]));
  return res;
}

__device__ inline double pairwise_sumsq(const double* v, int n) {
  if (n < 8) {
    double r = 0.0;
    for (int i = 0; i < n; ++i) r = __dadd_rn(r, sq_rn(v[i]));
    return r;
  }
  if (n <= 128) return pairwise_block8(v, n);
  int n2 = n / 2;
  n2 -= n2 % 8;
  // depth is at most log2(256/128) = 1 for the supported head dims
  return __dadd_rn(pairwise_block8(v, n2), pairwise_block8(v + n2, n - n2));
}

}  // namespace pkv
