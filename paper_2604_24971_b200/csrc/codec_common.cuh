// Codec pieces shared by the warp-granular kernels (codec.cu) and the
// TMA-streamed kernels (stream_codec.cu): exact key coding, the decode
// division sequence, and host-side codebook / sign / guard-band setup.
#pragma once

#include <algorithm>
#include <cmath>
#include <cstring>

#include "../../include/polykv.h"
#include "pkv_common.cuh"

namespace pkv {

struct Codebook3 {
  float mid32[7];
  float cent32[8];
  double mid64[7];
  int symmetric;
};

constexpr float kMagic = 12582912.0f;        // 1.5 * 2^23: x + kMagic rounds x to an integer

constexpr float kKeyEps = 4e-5f;             // |q - n| half-point guard for keys

// Reference formula (keyquant.py:61-64), evaluated exactly as numpy does in
// fp64: q = f64(x)/scale, code = floor(|q| + 0.5) * sign(q), clipped.
__device__ __forceinline__ int key_code_exact(float x, float s, int lo, int hi) {
  double q = (double)x / (double)s;
  double r = floor(fabs(q) + 0.5);
  if (q < 0.0) r = -r;
  if (r < lo) r = lo;
  if (r > hi) r = hi;
  return (int)r;
}

// The same decision without fp64: |x|/s >= k + 0.5  <=>  fma(-(k + 0.5), s, |x|)
// >= 0, and the FMA's single rounding keeps the sign of the exact difference.
// The approximate quotient |x| * (1/s) is within 2^-22 relative of |x|/s, so
// its nearest integer is off by at most one, next to a half-point; one test
// each way fixes it. Needs s >= 1e-30 (1/s finite); ties round away from 0.
__device__ __forceinline__ uint32_t key_code_fma(float x, float s, float rcp, int lo, int hi) {
  const float ax = fabsf(x);
  float r = rintf(ax * rcp);
  if (fmaf(-(r - 0.5f), s, ax) < 0.f) {
    r -= 1.f;
  } else if (fmaf(-(r + 0.5f), s, ax) >= 0.f) {
    r += 1.f;
  }
  int c = (int)r;
  if (x < 0.f) c = -c;
  return (uint32_t)max(lo, min(hi, c)) & 0xffu;
}

// 8 key codes of one chunk. Fast path: q = x * (1/s) rounded to nearest via
// the 2^23 magic; the low byte of the magic sum is the two's-complement code.
// Chunks with an element within kKeyEps of a half-point are re-coded exactly
// (FMA half-point tests; fp64 only when force_exact, i.e. s < 1e-30).
template <bool CLIP>
__device__ __forceinline__ uint2 key_chunk(const float (&x)[8], float s, float rcp, bool force_exact) {
  float m[8];
  float worst = 0.f;
#pragma unroll
  for (int j = 0; j < 8; ++j) {
    float q = x[j] * rcp;
    if (CLIP) q = fminf(fmaxf(q, -127.f), 127.f);
    m[j] = q + kMagic;
    const float n = m[j] - kMagic;
    worst = fmaxf(worst, fabsf(q - n));
  }
  uint2 w;
  w.x = __byte_perm(__byte_perm(__float_as_uint(m[0]), __float_as_uint(m[1]), 0x0040),
                    __byte_perm(__float_as_uint(m[2]), __float_as_uint(m[3]), 0x0040), 0x5410);
  w.y = __byte_perm(__byte_perm(__float_as_uint(m[4]), __float_as_uint(m[5]), 0x0040),
                    __byte_perm(__float_as_uint(m[6]), __float_as_uint(m[7]), 0x0040), 0x5410);
  if (force_exact || worst > 0.5f - kKeyEps) {
    uint32_t c[8];
#pragma unroll
    for (int j = 0; j < 8; ++j)
      c[j] = (s == 0.f) ? 0u
             : force_exact ? ((uint32_t)key_code_exact(x[j], s, CLIP ? -127 : -128, 127) & 0xffu)
                           : key_code_fma(x[j], s, rcp, CLIP ? -127 : -128, 127);
    w.x = c[0] | (c[1] << 8) | (c[2] << 16) | (c[3] << 24);
    w.y = c[4] | (c[5] << 8) | (c[6] << 16) | (c[7] << 24);
  }
  return w;
}

// Branch-free fast path of key_chunk (keyquant.py:61-64) on f32 pairs:
// m = x * rcp + 2^23 * 1.5 in ONE rounding (FFMA2), so n = m - magic is the
// nearest integer to the exact product x * rcp, and the low byte of m is its
// two's-complement code; d = x * rcp - n, again one rounding. With rcp within
// 1 ulp of 1/s, |x * rcp - x / s| <= 127.5 * 2^-23 < 2^-16, so every element
// with |d| <= 0.5 - 2^-15 has |x / s - n| < 0.5: n is the unique nearest
// integer of the exact quotient, i.e. keyquant.py's round-half-away result
// (a tie cannot pass). Otherwise `bad` is set and the caller re-codes the
// chunk exactly (key_code_fma). 3 paired FMAs + 1 max per pair of elements.
constexpr float kKeyGuard = 0.5f - 0x1p-15f;
__device__ __forceinline__ uint2 key_chunk_fast(const float (&x)[8], float2 rcp2, bool& bad) {
  const float2 mg = make_float2(kMagic, kMagic), nmg = make_float2(-kMagic, -kMagic);
  uint32_t mb[8];
  float worst = 0.f;
#pragma unroll
  for (int j = 0; j < 4; ++j) {
    const float2 xp = make_float2(x[2 * j], x[2 * j + 1]);
    const float2 m = __ffma2_rn(xp, rcp2, mg);
    const float2 n = __fadd2_rn(m, nmg);
    const float2 d = __ffma2_rn(xp, rcp2, make_float2(-n.x, -n.y));
    worst = fmaxf(worst, fmaxf(fabsf(d.x), fabsf(d.y)));
    mb[2 * j] = __float_as_uint(m.x);
    mb[2 * j + 1] = __float_as_uint(m.y);
  }
  bad = worst > kKeyGuard;
  uint2 w;
  w.x = __byte_perm(__byte_perm(mb[0], mb[1], 0x0040), __byte_perm(mb[2], mb[3], 0x0040), 0x5410);
  w.y = __byte_perm(__byte_perm(mb[4], mb[5], 0x0040), __byte_perm(mb[6], mb[7], 0x0040), 0x5410);
  return w;
}

// int8 code -> exact f32 via the 2^23 magic (no I2F on the conversion pipe)
__device__ __forceinline__ float i8_to_f32(uint32_t word_x80, int byte) {
  return __uint_as_float(__byte_perm(word_x80, 0x4B000000u, 0x7650 + byte)) - 8388736.0f;
}

// x / c correctly rounded for the constant c = 127 (block32 key scales,
// keyquant.py:60 applied per block): q = x*r corrected once with the exact FMA
// remainder, verified over every f32 mantissa by pkv_selftest; inputs outside
// [2^-100, 2^100] take IEEE division.
constexpr float kRcp127 = 1.0f / 127.0f;
__device__ __forceinline__ float div127_core(float x) {  // |x| in [2^-100, 2^100]
  const float q = x * kRcp127;
  const float e = fmaf(-q, 127.0f, x);
  return fmaf(e, kRcp127, q);
}
__device__ __forceinline__ float div127(float x) {
  const float ax = fabsf(x);
  if (!(ax >= 0x1p-100f && ax <= 0x1p100f)) return __fdiv_rn(x, 127.0f);
  return div127_core(x);
}

// 1/x within 1 ulp (PTX rcp.approx.f32), for normal x
__device__ __forceinline__ float rcp_approx(float x) {
  float r;
  asm("rcp.approx.ftz.f32 %0, %1;" : "=f"(r) : "f"(x));
  return r;
}

// x / f32(sqrt(D)), correctly rounded. Power-of-four D: exact multiply.
// Otherwise q = x*r corrected once with the exact FMA remainder; the
// sequence is verified exhaustively over all f32 mantissas by
// pkv_selftest(PKV_SELFTEST_DIVISION) and falls back to IEEE division
// outside the normal range.
template <int D>
__device__ __forceinline__ float div_sqrt_d(float x, float c, float r) {
  constexpr bool pow4 = (VG<D>::LOG2D % 2) == 0;
  if (pow4) return x * r;
  const float q = x * r;
  const float e = fmaf(-q, c, x);
  const float q1 = fmaf(e, r, q);
  // the correction turns -0 / c into +0; the quotient has the sign of x
  return __uint_as_float((__float_as_uint(q1) & 0x7fffffffu) | (__float_as_uint(x) & 0x80000000u));
}

// ---------------------------------------------------------------------------
// host helpers
// ---------------------------------------------------------------------------
static inline bool pinned_midpoints(const double* c, double* mid) {
  for (int i = 0; i < 8; ++i)
    if (!std::isfinite(c[i])) return false;
  for (int i = 0; i < 7; ++i) {
    if (!(c[i + 1] > c[i])) return false;
    // largest double not above the exact rational midpoint
    // (valuequant.py:62-71): TwoSum gives the exact a+b = s + e.
    const double x = c[i], y = c[i + 1];
    const double s = x + y;
    const double bb = s - x;
    const double e = (x - (s - bb)) + (y - bb);
    double m = s * 0.5;
    if (e < 0.0) m = std::nextafter(m, -INFINITY);
    mid[i] = m;
  }
  return true;
}

static inline bool fill_codebook(const double* centroids, Codebook3& cb) {
  if (!centroids) return false;
  if (!pinned_midpoints(centroids, cb.mid64)) return false;
  for (int i = 0; i < 7; ++i) cb.mid32[i] = (float)cb.mid64[i];
  for (int i = 0; i < 8; ++i) cb.cent32[i] = (float)centroids[i];
  bool sym = true;
  for (int i = 0; i < 8; ++i) sym = sym && centroids[i] == -centroids[7 - i];
  cb.symmetric = sym ? 1 : 0;
  return true;
}

static inline int log2i(int d) {
  int l = 0;
  while ((1 << l) < d) ++l;
  return l;
}

// Proven bound on |z32 - z_exact| for the fp32 fast path plus the error of
// the f32 thresholds, with a 1.5x margin.
static inline float guard_delta(int d) {
  const double u = std::ldexp(1.0, -24);
  return (float)(1.5 * u * (log2i(d) * std::sqrt((double)d) + 6.0) + 1e-12);
}

static inline bool aligned(const void* p, uintptr_t a) { return (reinterpret_cast<uintptr_t>(p) & (a - 1)) == 0; }

static inline int sm_count() {
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  return sms;
}

static inline bool fill_sign(const uint32_t* sign_bits_host, int d, uint32_t* dst) {
  std::memset(dst, 0, 8 * sizeof(uint32_t));
  if (!sign_bits_host) return false;
  const int words = (d + 31) / 32;
  bool any = false;
  for (int i = 0; i < words && i < 8; ++i) dst[i] = sign_bits_host[i];
  if (d % 32) dst[words - 1] &= (1u << (d % 32)) - 1u;
  for (int i = 0; i < 8; ++i) any = any || dst[i] != 0;
  return any;
}

}  // namespace pkv
