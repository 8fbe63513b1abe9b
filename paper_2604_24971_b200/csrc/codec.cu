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
};

struct EncodeArgs {
  int num_layers;
  int head_dim;
  int k_mode;
  int do_k, do_v;
  int use_sign;
  int vec_ok;               // all pointers aligned and n % 8 == 0
  long long nvec;           // vectors per layer
  long long nelem;          // elements per layer
  int a_items, e_items, v_items;  // per layer
  long long total_items;
  float delta;              // guard band on normalised coordinates
  uint32_t sign_bits[8];
  Codebook3 cb;
  uint32_t* status;         // [L]
  uint32_t* replay_count;   // [1] or null
  uint32_t* ws;             // [0] ticket, [1..L] max bits, [1+L..2L] done
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
  int do_k, do_v;
  int use_sign;
  int vec_ok;
  long long nvec, nelem;
  int k_items, v_items;  // per layer
  long long total_items;
  float sqrt_d32;
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

constexpr int kKElems = kThreads * 32;  // key elements per work item
constexpr float kMagic = 12582912.0f;   // 1.5 * 2^23: x + kMagic rounds x to an integer
constexpr float kKeyEps = 4e-5f;        // |q - n| half-point guard for keys

template <int D>
struct VItem {
  // value vectors per work item: ~32K coordinates
  static constexpr int ITERS = (32768 / (VG<D>::VPI * D)) > 0 ? (32768 / (VG<D>::VPI * D)) : 1;
  static constexpr int VECS = ITERS * VG<D>::VPI;
};

// ---------------------------------------------------------------------------
// keys
// ---------------------------------------------------------------------------

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

// Fast key code with exactness guard. Returns the int8 code in the low byte
// of the result; sets `near` if the element must take the exact path.
__device__ __forceinline__ uint32_t key_code_fast(float x, float rcp, bool clip, bool& near) {
  float q = x * rcp;
  if (clip) q = fminf(fmaxf(q, -200.f), 200.f);
  float m = q + kMagic;             // RNE to an integer
  float n = m - kMagic;
  float diff = q - n;               // in [-0.5, 0.5]
  near |= fabsf(diff) > (0.5f - kKeyEps);
  int code = (int)(__float_as_uint(m) - 0x4B400000u);
  if (clip) code = max(-127, min(127, code));
  return (uint32_t)code & 0xffu;
}

__device__ __forceinline__ uint32_t abs_bits(float x) { return __float_as_uint(x) & 0x7fffffffu; }

template <typename TIn>
__device__ void k_absmax_item(const EncodeArgs& a, int layer, int item, uint32_t* red) {
  const TIn* src = static_cast<const TIn*>(a.k_in[layer]);
  const long long e0 = (long long)item * kKElems;
  const long long n = a.nelem;
  uint32_t m = 0;
  if (a.vec_ok) {
#pragma unroll
    for (int i = 0; i < kKElems / (kThreads * 8); ++i) {
      long long e = e0 + ((long long)i * kThreads + threadIdx.x) * 8;
      if (e < n) {
        float x[8];
        load8(src + e, x);
#pragma unroll
        for (int j = 0; j < 8; ++j) m = max(m, abs_bits(x[j]));
      }
    }
  } else {
    for (int i = threadIdx.x; i < kKElems; i += kThreads) {
      long long e = e0 + i;
      if (e < n) m = max(m, abs_bits(load1(src + e)));
    }
  }
  // block reduce
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  if (lane == 0) red[warp] = m;
  __syncthreads();
  if (threadIdx.x == 0) {
    uint32_t mm = 0;
    for (int w = 0; w < kThreads / 32; ++w) mm = max(mm, red[w]);
    uint32_t* maxbits = a.ws + 1;
    uint32_t* done = a.ws + 1 + a.num_layers;
    atomicMax(&maxbits[layer], mm);
    __threadfence();
    atomicAdd(&done[layer], 1u);
  }
}

// Encode one item of keys. Per-tensor mode waits for the layer's absmax.
template <typename TIn>
__device__ void k_encode_item(const EncodeArgs& a, int layer, int item, uint32_t* shared_u32) {
  const TIn* src = static_cast<const TIn*>(a.k_in[layer]);
  int8_t* dst = a.k_codes[layer];
  const long long e0 = (long long)item * kKElems;
  const long long n = a.nelem;

  if (a.k_mode == PKV_K_TENSOR) {
    if (threadIdx.x == 0) {
      volatile uint32_t* done = a.ws + 1 + a.num_layers;
      while (done[layer] < (uint32_t)a.a_items) __nanosleep(200);
      __threadfence();
      volatile uint32_t* maxbits = a.ws + 1;
      shared_u32[0] = maxbits[layer];
    }
    __syncthreads();
    const uint32_t pb = shared_u32[0];
    __syncthreads();
    const bool nonfinite = pb >= 0x7f800000u;
    const float peak = __uint_as_float(pb);
    const float s = (nonfinite || pb == 0) ? 0.f : peak / 127.0f;  // f32(peak/127)
    if (item == 0 && threadIdx.x == 0) {
      a.k_scale[layer][0] = s;
      if (nonfinite) atomicOr(&a.status[layer], PKV_FLAG_K_NONFINITE);
    }
    const float rcp = 1.0f / s;
    const bool tiny = !(s >= 1e-30f);  // covers s == 0: exact path / zeros
    if (a.vec_ok) {
#pragma unroll
      for (int i = 0; i < kKElems / (kThreads * 8); ++i) {
        long long e = e0 + ((long long)i * kThreads + threadIdx.x) * 8;
        if (e >= n) continue;
        float x[8];
        load8(src + e, x);
        bool near = tiny;
        uint32_t c[8];
#pragma unroll
        for (int j = 0; j < 8; ++j) c[j] = key_code_fast(x[j], rcp, false, near);
        if (near) {
#pragma unroll
          for (int j = 0; j < 8; ++j)
            c[j] = (s == 0.f) ? 0u : ((uint32_t)key_code_exact(x[j], s, -128, 127) & 0xffu);
        }
        uint2 w;
        w.x = c[0] | (c[1] << 8) | (c[2] << 16) | (c[3] << 24);
        w.y = c[4] | (c[5] << 8) | (c[6] << 16) | (c[7] << 24);
        st_u2(dst + e, w);
      }
    } else {
      for (int i = threadIdx.x; i < kKElems; i += kThreads) {
        long long e = e0 + i;
        if (e >= n) continue;
        float x = load1(src + e);
        dst[e] = (s == 0.f) ? (int8_t)0 : (int8_t)key_code_exact(x, s, -128, 127);
      }
    }
    return;
  }

  // ---- block32: one fp16 scale per 32 contiguous elements (q8_0) ----
  __half* bsc = a.k_bscale[layer];
  if (a.vec_ok) {
#pragma unroll
    for (int i = 0; i < kKElems / (kThreads * 8); ++i) {
      long long e = e0 + ((long long)i * kThreads + threadIdx.x) * 8;
      const bool valid = e < n;
      float x[8];
      if (valid) {
        load8(src + e, x);
      } else {
#pragma unroll
        for (int j = 0; j < 8; ++j) x[j] = 0.f;
      }
      uint32_t m = 0;
#pragma unroll
      for (int j = 0; j < 8; ++j) m = max(m, abs_bits(x[j]));
      // 4 consecutive lanes hold one 32-element block
      m = max(m, __shfl_xor_sync(0xffffffffu, m, 1));
      m = max(m, __shfl_xor_sync(0xffffffffu, m, 2));
      if (!valid) continue;
      const bool nonfinite = m >= 0x7f800000u;
      const float peak = __uint_as_float(m);
      const float s32 = peak / 127.0f;
      __half s16 = __float2half_rn(s32);
      uint16_t s16b = __half_as_ushort(s16);
      bool overflow = false;
      if (nonfinite) {
        s16b = 0;
      } else if (m == 0) {
        s16b = 0;
      } else if ((s16b & 0x7fffu) >= 0x7c00u) {
        overflow = true;
        s16b = 0;
      } else if (s16b == 0) {
        s16b = 1;  // peak > 0 but the scale underflows fp16: smallest subnormal
      }
      const float s = __half2float(__ushort_as_half(s16b));
      if ((threadIdx.x & 3) == 0) {
        bsc[e >> 5] = __ushort_as_half(s16b);
        if (nonfinite) atomicOr(&a.status[layer], PKV_FLAG_K_NONFINITE);
        if (overflow) atomicOr(&a.status[layer], PKV_FLAG_K_SCALE_OVERFLOW);
      }
      const float rcp = 1.0f / s;
      bool near = !(s >= 1e-30f);
      uint32_t c[8];
#pragma unroll
      for (int j = 0; j < 8; ++j) c[j] = key_code_fast(x[j], rcp, true, near);
      if (near) {
#pragma unroll
        for (int j = 0; j < 8; ++j)
          c[j] = (s == 0.f) ? 0u : ((uint32_t)key_code_exact(x[j], s, -127, 127) & 0xffu);
      }
      uint2 w;
      w.x = c[0] | (c[1] << 8) | (c[2] << 16) | (c[3] << 24);
      w.y = c[4] | (c[5] << 8) | (c[6] << 16) | (c[7] << 24);
      st_u2(dst + e, w);
    }
  } else {
    // scalar path: one thread per 32-element block
    const long long nb = (n + 31) / 32;
    for (int bi = threadIdx.x; bi < kKElems / 32; bi += kThreads) {
      long long b = e0 / 32 + bi;
      if (b >= nb) continue;
      long long lo = b * 32, hi = min(lo + 32, n);
      uint32_t m = 0;
      for (long long e = lo; e < hi; ++e) m = max(m, abs_bits(load1(src + e)));
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
__device__ void v_replay(const EncodeArgs& a, int layer, long long v, double* R, uint8_t* C) {
  const int lane = threadIdx.x & 31;
  const TIn* p = static_cast<const TIn*>(a.v_in[layer]) + v * D;
  for (int i = lane; i < D; i += 32) {
    double x = (double)load1(p + i);
    if (a.use_sign && sign_bit(a.sign_bits, i)) x = -x;  // vals * sign_diagonal
    R[i] = x;
  }
  __syncwarp();
  for (int h = 1; h < D; h <<= 1) {  // fwht.py:31-39, in f64
    for (int q = lane; q < D / 2; q += 32) {
      int i = (q / h) * 2 * h + (q % h);
      double lo = R[i], hi = R[i + h];
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
    double mean = pairwise_sumsq(R, D) / (double)D;  // np.mean(np.square(rot))
    rms = sqrt(mean);
  }
  rms = __shfl_sync(0xffffffffu, rms, 0);
  const float scale = (float)rms;
  const double den = rms > 0.0 ? rms : 1.0;
  for (int i = lane; i < D; i += 32) {
    double z = R[i] / den;
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

// Per-warp shared memory for the value kernels.
template <int D>
struct VSmem {
  uint32_t stage[VG<D>::VPW][VG<D>::W + 1];  // packed-word transpose
  double R[D];                               // replay scratch
  uint8_t C[D];
};

template <int D, typename TIn>
__device__ void v_encode_item(const EncodeArgs& a, int layer, int item, VSmem<D>* sm_all) {
  using G = VG<D>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int vw = lane / G::TPV, s = lane % G::TPV;
  VSmem<D>& sm = sm_all[warp];
  const TIn* src = static_cast<const TIn*>(a.v_in[layer]);
  uint8_t* packed = a.v_packed[layer];
  float* scales = a.v_scales[layer];
  const long long vbase = (long long)item * VItem<D>::VECS;
  const float delta = a.delta;

  for (int it = 0; it < VItem<D>::ITERS; ++it) {
    const long long v = vbase + (long long)it * G::VPI + warp * G::VPW + vw;
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
    if (a.use_sign) {
#pragma unroll
      for (int c = 0; c < G::NCH; ++c)
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (sign_bit(a.sign_bits, 8 * (s + G::TPV * c) + e)) x[c * 8 + e] = -x[c * 8 + e];
    }
    // squared norm in fp64 from the inputs (the rotation is orthogonal):
    // every x^2 is exact in fp64, the sum is good to ~D*2^-53 relative.
    double S = 0.0;
#pragma unroll
    for (int i = 0; i < G::CPT; ++i) S = fma((double)x[i], (double)x[i], S);
#pragma unroll
    for (int lb = 0; lb < G::LB; ++lb) S += __shfl_xor_sync(0xffffffffu, S, 1 << lb);

    fwht_lanes<D>(x, s);

    bool replay = false, nonfinite = false, zero = false;
    float scale = 0.f, inv = 0.f;
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
      inv = (float)rsqrt(S);  // 1/||x||; z = U/||x|| with U the unnormalised FWHT
    }

    uint32_t words[G::NCH];
    const float* m = a.cb.mid32;
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
        replay |= (fabsf(z - m[3]) < delta) | (fabsf(z - t2) < delta) | (fabsf(z - t3) < delta);
        const uint32_t code = (p1 ? 4u : 0u) | (p2 ? 2u : 0u) | (p3 ? 1u : 0u);
        w |= code << (3 * e);
      }
      words[c] = w;
    }
    if (zero || nonfinite) {
#pragma unroll
      for (int c = 0; c < G::NCH; ++c) words[c] = 0;
      scale = 0.f;
    }
    // all lanes of a vector agree on replay/nonfinite
#pragma unroll
    for (int lb = 0; lb < G::LB; ++lb) {
      replay |= __shfl_xor_sync(0xffffffffu, (int)replay, 1 << lb) != 0;
    }
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
      const long long rv = vbase + (long long)it * G::VPI + warp * G::VPW + src_lane / G::TPV;
      v_replay<D, TIn>(a, layer, rv, sm.R, sm.C);
    }
  }
}

// ---------------------------------------------------------------------------
// persistent encode kernel with ticketed work items
// ---------------------------------------------------------------------------
// Items are ordered in rounds r = 0..L: round r holds the absmax items of
// layer r, the value items of layer r and the key-encode items of layer r-1
// (interleaved). A key-encode item waits for its layer's absmax to be
// complete; all those items hold smaller tickets and never wait, so the
// schedule is deadlock-free, and layer r-1's keys are re-read from L2.
struct ItemRef {
  int kind;  // 0 absmax, 1 key encode, 2 value encode
  int layer;
  int idx;
};

__device__ __forceinline__ ItemRef decode_ticket(const EncodeArgs& a, long long t) {
  const long long nA = a.a_items, nE = a.e_items, nV = a.v_items;
  const int L = a.num_layers;
  const long long s0 = nA + nV, sm = nA + nV + nE;
  int r;
  long long off;
  if (t < s0) {
    r = 0;
    off = t;
  } else {
    long long tt = t - s0;
    if (L > 1 && tt < (long long)(L - 1) * sm) {
      r = 1 + (int)(tt / sm);
      off = tt % sm;
    } else {
      r = L;
      off = tt - (long long)(L - 1) * sm;
    }
  }
  ItemRef it;
  if (r < L) {
    if (off < nA) {
      it.kind = 0; it.layer = r; it.idx = (int)off;
      return it;
    }
    off -= nA;
    const long long nE_r = (r >= 1) ? nE : 0;
    // interleave value items of layer r with key-encode items of layer r-1
    const long long both = 2 * min(nV, nE_r);
    if (off < both) {
      if ((off & 1) == 0) { it.kind = 2; it.layer = r; it.idx = (int)(off >> 1); }
      else { it.kind = 1; it.layer = r - 1; it.idx = (int)(off >> 1); }
      return it;
    }
    off -= both;
    if (nV > nE_r) { it.kind = 2; it.layer = r; it.idx = (int)(min(nV, nE_r) + off); }
    else { it.kind = 1; it.layer = r - 1; it.idx = (int)(min(nV, nE_r) + off); }
    return it;
  }
  it.kind = 1; it.layer = L - 1; it.idx = (int)off;
  return it;
}

template <int D, typename TIn>
__global__ void __launch_bounds__(kThreads, 2) encode_kernel(const __grid_constant__ EncodeArgs a) {
  __shared__ VSmem<D> vsm[kThreads / 32];
  __shared__ uint32_t red[kThreads / 32 + 2];
  __shared__ long long ticket_sh;
  for (;;) {
    if (threadIdx.x == 0) ticket_sh = (long long)atomicAdd(a.ws, 1u);
    __syncthreads();
    const long long t = ticket_sh;
    __syncthreads();
    if (t >= a.total_items) break;
    const ItemRef it = decode_ticket(a, t);
    if (it.kind == 0) {
      k_absmax_item<TIn>(a, it.layer, it.idx, red);
    } else if (it.kind == 1) {
      k_encode_item<TIn>(a, it.layer, it.idx, red);
    } else {
      v_encode_item<D, TIn>(a, it.layer, it.idx, vsm);
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// decode (materialise) kernel
// ---------------------------------------------------------------------------

// int8 code -> exact f32 via the 2^23 magic (no I2F on the conversion pipe)
__device__ __forceinline__ float i8_to_f32(uint32_t word, int byte) {
  uint32_t b = (word >> (8 * byte)) & 0xffu;
  return __uint_as_float(0x4B000000u | (b ^ 0x80u)) - 8388736.0f;
}

template <typename TOut>
__device__ void k_decode_item(const DecodeArgs& a, int layer, int item) {
  const int8_t* codes = a.k_codes[layer];
  TOut* out = static_cast<TOut*>(a.k_out[layer]);
  const long long e0 = (long long)item * kKElems;
  const long long n = a.nelem;
  const bool tensor = a.k_mode == PKV_K_TENSOR;
  const float ts = tensor ? __ldg(a.k_scale[layer]) : 0.f;
  if (a.vec_ok) {
#pragma unroll
    for (int i = 0; i < kKElems / (kThreads * 8); ++i) {
      long long e = e0 + ((long long)i * kThreads + threadIdx.x) * 8;
      if (e >= n) continue;
      const uint2 w = ld_stream_u2(codes + e);
      const float s = tensor ? ts : __half2float(__ldg(a.k_bscale[layer] + (e >> 5)));
      float y[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) y[j] = i8_to_f32(w.x, j) * s;
#pragma unroll
      for (int j = 0; j < 4; ++j) y[4 + j] = i8_to_f32(w.y, j) * s;
      store8(out + e, y);
    }
  } else {
    for (int i = threadIdx.x; i < kKElems; i += kThreads) {
      long long e = e0 + i;
      if (e >= n) continue;
      const float s = tensor ? ts : __half2float(__ldg(a.k_bscale[layer] + (e >> 5)));
      store1(out + e, (float)codes[e] * s);
    }
  }
}

template <int D, typename TOut>
__device__ void v_decode_item(const DecodeArgs& a, int layer, int item, uint32_t* stage_all,
                              float* tbl) {
  using G = VG<D>;
  const int warp = threadIdx.x >> 5, lane = threadIdx.x & 31;
  const int vw = lane / G::TPV, s = lane % G::TPV;
  uint32_t(*stage)[G::W + 1] =
      reinterpret_cast<uint32_t(*)[G::W + 1]>(stage_all + warp * G::VPW * (G::W + 1));
  const uint8_t* packed = a.v_packed[layer];
  const float* scales = a.v_scales[layer];
  TOut* out = static_cast<TOut*>(a.v_out[layer]);
  const long long vbase = (long long)item * VItem<D>::VECS;
  const float sqd = a.sqrt_d32;

  for (int itr = 0; itr < VItem<D>::ITERS; ++itr) {
    const long long v = vbase + (long long)itr * G::VPI + warp * G::VPW + vw;
    const bool valid = v < a.nvec;
    // each lane fetches its Q contiguous packed words, then a warp transpose
    // hands every lane the words of its own chunks
    uint32_t q[G::Q];
    if (valid) {
      const uint8_t* p = packed + v * G::PACKED_BYTES + s * 3 * G::Q;
      if constexpr (G::Q == 8) {
        const uint2 u0 = ld_stream_u2(p), u1 = ld_stream_u2(p + 8), u2 = ld_stream_u2(p + 16);
        const uint32_t u[6] = {u0.x, u0.y, u1.x, u1.y, u2.x, u2.y};
        q[0] = u[0] & 0xffffffu;
        q[1] = ((u[0] >> 24) | (u[1] << 8)) & 0xffffffu;
        q[2] = ((u[1] >> 16) | (u[2] << 16)) & 0xffffffu;
        q[3] = u[2] >> 8;
        q[4] = u[3] & 0xffffffu;
        q[5] = ((u[3] >> 24) | (u[4] << 8)) & 0xffffffu;
        q[6] = ((u[4] >> 16) | (u[5] << 16)) & 0xffffffu;
        q[7] = u[5] >> 8;
      } else if constexpr (G::Q == 4) {
        const uint32_t* w = reinterpret_cast<const uint32_t*>(p);
        const uint32_t u0 = __ldg(w), u1 = __ldg(w + 1), u2 = __ldg(w + 2);
        q[0] = u0 & 0xffffffu;
        q[1] = ((u0 >> 24) | (u1 << 8)) & 0xffffffu;
        q[2] = ((u1 >> 16) | (u2 << 16)) & 0xffffffu;
        q[3] = u2 >> 8;
      } else {
#pragma unroll
        for (int j = 0; j < G::Q; ++j)
          q[j] = (uint32_t)p[3 * j] | ((uint32_t)p[3 * j + 1] << 8) | ((uint32_t)p[3 * j + 2] << 16);
      }
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
      for (int e = 0; e < 8; ++e)
        x[c * 8 + e] = tbl[((words[c] >> (3 * e)) & 7u) * kThreads + threadIdx.x];

    fwht_lanes<D>(x, s);

#pragma unroll
    for (int i = 0; i < G::CPT; ++i) x[i] = x[i] / sqd;  // IEEE division (fwht.py:50)
    if (a.use_sign) {
#pragma unroll
      for (int c = 0; c < G::NCH; ++c)
#pragma unroll
        for (int e = 0; e < 8; ++e)
          if (sign_bit(a.sign_bits, 8 * (s + G::TPV * c) + e)) x[c * 8 + e] = -x[c * 8 + e];
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
  }
}

template <int D, typename TOut>
__global__ void __launch_bounds__(kThreads, 2) decode_kernel(const __grid_constant__ DecodeArgs a) {
  __shared__ uint32_t stage[kThreads / VG<D>::TPV * (VG<D>::W + 1)];
  __shared__ float tbl[8 * kThreads];
  const long long per_layer = (long long)a.k_items + a.v_items;
  for (long long t = blockIdx.x; t < a.total_items; t += gridDim.x) {
    const int layer = (int)(t / per_layer);
    long long off = t % per_layer;
    // interleave key and value items so memory- and ALU-heavy work overlap
    const long long both = 2 * (long long)min(a.k_items, a.v_items);
    int kind, idx;
    if (off < both) {
      kind = (off & 1) ? 1 : 0;
      idx = (int)(off >> 1);
    } else {
      off -= both;
      kind = a.k_items > a.v_items ? 0 : 1;
      idx = (int)(min(a.k_items, a.v_items) + off);
    }
    if (kind == 0) k_decode_item<TOut>(a, layer, idx);
    else v_decode_item<D, TOut>(a, layer, idx, stage, tbl);
  }
}

// ---------------------------------------------------------------------------
// canonical codes <-> packed payload
// ---------------------------------------------------------------------------
__global__ void unpack_kernel(const uint8_t* __restrict__ packed, long long count,
                              uint8_t* __restrict__ codes) {
  const long long groups = (count + 7) / 8;
  for (long long g = blockIdx.x * (long long)blockDim.x + threadIdx.x; g < groups;
       g += (long long)gridDim.x * blockDim.x) {
    uint32_t w = (uint32_t)packed[3 * g] | ((uint32_t)packed[3 * g + 1] << 8) |
                 ((uint32_t)packed[3 * g + 2] << 16);
    for (int e = 0; e < 8; ++e) {
      long long i = 8 * g + e;
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
      long long i = 8 * g + e;
      uint32_t c = i < count ? codes[i] : 0u;
      oob |= c > 7u;
      w |= (c & 7u) << (3 * e);
    }
    if (oob && bad) atomicOr(bad, 0x8u);
    packed[3 * g] = (uint8_t)(w & 0xff);
    packed[3 * g + 1] = (uint8_t)((w >> 8) & 0xff);
    packed[3 * g + 2] = (uint8_t)((w >> 16) & 0xff);
  }
}

}  // namespace pkv

// ===========================================================================
// host side: C ABI
// ===========================================================================
namespace {

using namespace pkv;

bool pinned_midpoints(const double* c, double* mid) {
  for (int i = 0; i < 8; ++i)
    if (!std::isfinite(c[i])) return false;
  for (int i = 0; i < 7; ++i) {
    if (!(c[i + 1] > c[i])) return false;
    // largest double not above the exact rational midpoint
    // (valuequant.py:62-71): TwoSum gives the exact a+b = s + e.
    const double a = c[i], b = c[i + 1];
    const double s = a + b;
    const double bb = s - a;
    const double e = (a - (s - bb)) + (b - bb);
    double m = s * 0.5;
    if (e < 0.0) m = std::nextafter(m, -INFINITY);
    mid[i] = m;
  }
  return true;
}

bool fill_codebook(const double* centroids, Codebook3& cb) {
  if (!centroids) return false;
  if (!pinned_midpoints(centroids, cb.mid64)) return false;
  for (int i = 0; i < 7; ++i) cb.mid32[i] = (float)cb.mid64[i];
  for (int i = 0; i < 8; ++i) cb.cent32[i] = (float)centroids[i];
  return true;
}

int log2i(int d) {
  int l = 0;
  while ((1 << l) < d) ++l;
  return l;
}

// Proven bound on |z32 - z_exact| for the fp32 fast path plus the error of
// the f32 thresholds, with a 1.5x margin.
float guard_delta(int d) {
  const double u = std::ldexp(1.0, -24);
  return (float)(1.5 * u * (log2i(d) * std::sqrt((double)d) + 6.0) + 1e-12);
}

bool aligned16(const void* p) { return (reinterpret_cast<uintptr_t>(p) & 15u) == 0; }

int occupancy_grid(const void* fn, int smem) {
  int dev = 0, sms = 148, per_sm = 1;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm, fn, kThreads, smem) != cudaSuccess ||
      per_sm < 1)
    per_sm = 1;
  return sms * per_sm;
}

template <int D, typename TIn>
int launch_encode(EncodeArgs& a, cudaStream_t st) {
  const void* fn = (const void*)encode_kernel<D, TIn>;
  int grid = occupancy_grid(fn, 0);
  if ((long long)grid > a.total_items) grid = (int)a.total_items;
  if (grid < 1) return PKV_OK;
  encode_kernel<D, TIn><<<grid, kThreads, 0, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? PKV_OK : PKV_ERR_CUDA;
}

template <typename TIn>
int dispatch_encode(EncodeArgs& a, cudaStream_t st) {
  switch (a.do_v ? a.head_dim : 128) {
    case 8: return launch_encode<8, TIn>(a, st);
    case 16: return launch_encode<16, TIn>(a, st);
    case 32: return launch_encode<32, TIn>(a, st);
    case 64: return launch_encode<64, TIn>(a, st);
    case 128: return launch_encode<128, TIn>(a, st);
    case 256: return launch_encode<256, TIn>(a, st);
    default: return PKV_ERR_UNSUPPORTED_HEAD_DIM;
  }
}

template <int D, typename TOut>
int launch_decode(DecodeArgs& a, cudaStream_t st) {
  const void* fn = (const void*)decode_kernel<D, TOut>;
  long long grid = occupancy_grid(fn, 0);
  if (grid > a.total_items) grid = a.total_items;
  if (grid < 1) return PKV_OK;
  decode_kernel<D, TOut><<<(int)grid, kThreads, 0, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? PKV_OK : PKV_ERR_CUDA;
}

template <typename TOut>
int dispatch_decode(DecodeArgs& a, cudaStream_t st) {
  switch (a.do_v ? a.head_dim : 128) {
    case 8: return launch_decode<8, TOut>(a, st);
    case 16: return launch_decode<16, TOut>(a, st);
    case 32: return launch_decode<32, TOut>(a, st);
    case 64: return launch_decode<64, TOut>(a, st);
    case 128: return launch_decode<128, TOut>(a, st);
    case 256: return launch_decode<256, TOut>(a, st);
    default: return PKV_ERR_UNSUPPORTED_HEAD_DIM;
  }
}

void fill_sign(const uint32_t* sign_bits_host, int d, uint32_t* dst, int* use) {
  std::memset(dst, 0, 8 * sizeof(uint32_t));
  *use = 0;
  if (!sign_bits_host) return;
  const int words = (d + 31) / 32;
  for (int i = 0; i < words && i < 8; ++i) dst[i] = sign_bits_host[i];
  if (d % 32) dst[words - 1] &= (1u << (d % 32)) - 1u;
  *use = 1;
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

}  // namespace

extern "C" {

int pkv_abi_version(void) { return PKV_ABI_VERSION; }

const char* pkv_status_string(int status) {
  switch (status) {
    case PKV_OK: return "ok";
    case PKV_ERR_INVALID_ARG: return "invalid argument";
    case PKV_ERR_UNSUPPORTED_HEAD_DIM: return "head_dim not supported by the value kernels (8..256, power of two)";
    case PKV_ERR_CUDA: return "CUDA launch error";
    case PKV_ERR_WORKSPACE: return "workspace too small";
    case PKV_ERR_ALIGNMENT: return "misaligned pointer";
    case PKV_ERR_UNSUPPORTED_CODEBOOK: return "codebook must have 8 strictly increasing finite centroids";
    default: return "unknown status";
  }
}

int pkv_v_head_dim_supported(int d) {
  return d == 8 || d == 16 || d == 32 || d == 64 || d == 128 || d == 256;
}

size_t pkv_encode_workspace_bytes(int num_layers) {
  if (num_layers < 0) return 0;
  const int l = std::min(num_layers, (int)PKV_MAX_LAYERS_PER_LAUNCH);
  return (size_t)(1 + 2 * l) * sizeof(uint32_t);
}

int pkv_encode(int num_layers, int64_t num_vectors, int head_dim, int in_dtype,
               const void* const* k_in, const void* const* v_in, int k_mode,
               int8_t* const* k_codes, float* const* k_scale, uint16_t* const* k_bscale,
               uint8_t* const* v_packed, float* const* v_scales, const double* centroids_host,
               const uint32_t* sign_bits_host, uint32_t* status, uint32_t* replay_count,
               void* workspace, size_t workspace_bytes, void* stream) {
  if (num_layers < 0 || num_vectors < 0 || head_dim < 1) return PKV_ERR_INVALID_ARG;
  if (in_dtype != PKV_F32 && in_dtype != PKV_BF16) return PKV_ERR_INVALID_ARG;
  if (k_mode != PKV_K_TENSOR && k_mode != PKV_K_BLOCK32) return PKV_ERR_INVALID_ARG;
  if (!status) return PKV_ERR_INVALID_ARG;
  const bool do_k = k_in != nullptr, do_v = v_in != nullptr;
  if (num_layers == 0 || num_vectors == 0 || (!do_k && !do_v)) return PKV_OK;
  if (do_v && !pkv_v_head_dim_supported(head_dim)) return PKV_ERR_UNSUPPORTED_HEAD_DIM;
  if (workspace_bytes < pkv_encode_workspace_bytes(num_layers) || !workspace) return PKV_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int elt = in_dtype == PKV_F32 ? 4 : 2;
  const long long nelem = (long long)num_vectors * head_dim;

  for (int l0 = 0; l0 < num_layers; l0 += PKV_MAX_LAYERS_PER_LAUNCH) {
    const int L = std::min(num_layers - l0, (int)PKV_MAX_LAYERS_PER_LAUNCH);
    EncodeArgs a;
    std::memset(&a, 0, sizeof(a));
    a.num_layers = L;
    a.head_dim = head_dim;
    a.k_mode = k_mode;
    a.do_k = do_k;
    a.do_v = do_v;
    a.nvec = num_vectors;
    a.nelem = nelem;
    a.delta = guard_delta(head_dim);
    fill_sign(sign_bits_host, head_dim, a.sign_bits, &a.use_sign);
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
        ok = ok && aligned16(a.k_in[l]) && (reinterpret_cast<uintptr_t>(a.k_codes[l]) & 7u) == 0;
      }
      if (do_v) {
        a.v_in[l] = v_in[l0 + l];
        a.v_packed[l] = v_packed ? v_packed[l0 + l] : nullptr;
        a.v_scales[l] = v_scales ? v_scales[l0 + l] : nullptr;
        if (!a.v_in[l] || !a.v_packed[l] || !a.v_scales[l]) return PKV_ERR_INVALID_ARG;
        // the value kernels use 16 B chunk loads and word-aligned packed stores
        if (!aligned16(a.v_in[l]) || (reinterpret_cast<uintptr_t>(a.v_packed[l]) & 7u) ||
            (reinterpret_cast<uintptr_t>(a.v_scales[l]) & 3u))
          return PKV_ERR_ALIGNMENT;
      }
    }
    (void)elt;
    a.vec_ok = ok ? 1 : 0;
    const int k_items = do_k ? (int)((nelem + kKElems - 1) / kKElems) : 0;
    a.e_items = k_items;
    a.a_items = (do_k && k_mode == PKV_K_TENSOR) ? k_items : 0;
    a.v_items = do_v ? v_items_dispatch(head_dim, num_vectors) : 0;
    a.total_items = (long long)L * (a.a_items + a.e_items + a.v_items);
    if (cudaMemsetAsync(workspace, 0, pkv_encode_workspace_bytes(L), st) != cudaSuccess)
      return PKV_ERR_CUDA;
    const int rc = in_dtype == PKV_F32 ? dispatch_encode<float>(a, st)
                                       : dispatch_encode<__nv_bfloat16>(a, st);
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
  for (int l0 = 0; l0 < num_layers; l0 += PKV_MAX_LAYERS_PER_LAUNCH) {
    const int L = std::min(num_layers - l0, (int)PKV_MAX_LAYERS_PER_LAUNCH);
    DecodeArgs a;
    std::memset(&a, 0, sizeof(a));
    a.num_layers = L;
    a.head_dim = head_dim;
    a.k_mode = k_mode;
    a.do_k = do_k;
    a.do_v = do_v;
    a.nvec = num_vectors;
    a.nelem = nelem;
    a.sqrt_d32 = (float)std::sqrt((double)head_dim);  // np.float32(np.sqrt(d))
    fill_sign(sign_bits_host, head_dim, a.sign_bits, &a.use_sign);
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
        if (!a.k_codes[l] || !a.k_out[l] ||
            (k_mode == PKV_K_TENSOR ? !a.k_scale[l] : !a.k_bscale[l]))
          return PKV_ERR_INVALID_ARG;
        ok = ok && (reinterpret_cast<uintptr_t>(a.k_codes[l]) & 7u) == 0 && aligned16(a.k_out[l]);
      }
      if (do_v) {
        a.v_packed[l] = v_packed[l0 + l];
        a.v_scales[l] = v_scales ? v_scales[l0 + l] : nullptr;
        a.v_out[l] = v_out[l0 + l];
        if (!a.v_packed[l] || !a.v_scales[l] || !a.v_out[l]) return PKV_ERR_INVALID_ARG;
        if (!aligned16(a.v_out[l]) || (reinterpret_cast<uintptr_t>(a.v_packed[l]) & 7u))
          return PKV_ERR_ALIGNMENT;
      }
    }
    a.vec_ok = ok ? 1 : 0;
    a.k_items = do_k ? (int)((nelem + kKElems - 1) / kKElems) : 0;
    a.v_items = do_v ? v_items_dispatch(head_dim, num_vectors) : 0;
    a.total_items = (long long)L * (a.k_items + a.v_items);
    const int rc = out_dtype == PKV_F32 ? dispatch_decode<float>(a, st)
                                        : dispatch_decode<__nv_bfloat16>(a, st);
    if (rc != PKV_OK) return rc;
  }
  return PKV_OK;
}

int pkv_unpack_codes(const uint8_t* packed, int64_t count, uint8_t* codes, void* stream) {
  if (count < 0 || (count > 0 && (!packed || !codes))) return PKV_ERR_INVALID_ARG;
  if (count == 0) return PKV_OK;
  const long long groups = (count + 7) / 8;
  int grid = (int)std::min<long long>((groups + 255) / 256, 148LL * 16);
  unpack_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(packed, count, codes);
  return cudaGetLastError() == cudaSuccess ? PKV_OK : PKV_ERR_CUDA;
}

int pkv_pack_codes(const uint8_t* codes, int64_t count, uint8_t* packed, uint32_t* bad_code,
                   void* stream) {
  if (count < 0 || (count > 0 && (!packed || !codes))) return PKV_ERR_INVALID_ARG;
  if (count == 0) return PKV_OK;
  const long long groups = (count + 7) / 8;
  int grid = (int)std::min<long long>((groups + 255) / 256, 148LL * 16);
  pack_kernel<<<grid, 256, 0, static_cast<cudaStream_t>(stream)>>>(codes, count, packed, bad_code);
  return cudaGetLastError() == cudaSuccess ? PKV_OK : PKV_ERR_CUDA;
}

}  // extern "C"
