// GQA decode attention that reads the packed SharedKVPool directly.
//
// Replaces, for one layer, the eager/SDPA attention that the reference runs
// over a per-agent materialised DynamicCache (kvbridge/hfcache.py:58-67 ->
// transformers LlamaAttention.forward, modeling_llama.py:251-290, eager path
// :199-230 with repeat_kv :187): softmax(q k^T * scale) v, where k and v are
// the pool's dequantised keys and values.
//
// Layout of the work:
//   * all agents' query rows that share a KV head (rows = agents * group) are
//     processed together, so each pool tile is read from HBM once per step;
//   * the prefix is cut into whole-tile splits, ~2 CTAs per SM (8 for
//     16-row tiles at d=64), one CTA per (kv head, split,
//     64-row tile); a CTA walks its split in 64-token tiles, converting each
//     K tile (int8 codes * scale, exactly the reference dequant) to f32 in
//     shared memory and each V tile to the *rotated* domain
//     y = table[code] * rms (valuequant.py:232-234), and runs register-tiled
//     fp32 S = Q K / P Y products with an online (flash) softmax;
//   * a combine kernel merges the tiles with log-sum-exp weights, applies
//     ONE inverse FWHT / sqrt(d) (and the sign diagonal) per output vector —
//     valid because H is linear — and folds in the agent's private bf16
//     tail (tokens appended after the shared prefix).
#include <algorithm>
#include <cmath>
#include <cstdlib>
#include <cstring>

#include "../../include/polykv.h"
#include "pkv_common.cuh"
#include "tuning.h"

namespace pkv {
namespace attn {

constexpr float kLog2e = 1.4426950408889634f;

struct Args {
  int rows;        // agents * group
  int kv_heads, group, head_dim;
  long long T;
  int q_dtype, out_dtype, k_mode;
  int use_sign;
  int splits;      // ceil(T / TT)
  float qscale;    // softmax_scale * log2(e)
  uint32_t sign_bits[8];
  float cent32[8];
  const void* q;
  const int8_t* k_codes;
  const float* k_scale;
  const __half* k_bscale;
  const uint8_t* v_packed;
  const float* v_scales;
  const void* tail_k;
  const void* tail_v;
  const int32_t* tail_len;
  int tail_cap;
  float* part;     // [kv_heads][splits][rows][D + 4]: acc[D], m, l, pad (16 B rows)
  void* out;
};

__device__ __forceinline__ float ldq(const Args& a, long long i) {
  return a.q_dtype == PKV_F32 ? static_cast<const float*>(a.q)[i]
                              : __bfloat162float(static_cast<const __nv_bfloat16*>(a.q)[i]);
}

// ---------------------------------------------------------------------------
// prefix kernel: register-tiled fp32 attention over one split of the prefix
// ---------------------------------------------------------------------------
// CTA = (kv head h, split sp, row tile). The split covers a contiguous token
// range, walked in tiles of TT2 tokens with an online (flash) softmax, so
// partials are written once per split. Per tile:
//   Ks[d][t]  = k code * key scale (dequantize_k, keyquant.py:71), f32
//   Ys[t][d]  = table[code] * rms  (rotated-domain V, valuequant.py:232-234)
//   S = Q Ks (16 x 16 threads, TR rows x 4 tokens each), P = exp2(S - m)
//   O += P Ys (16 x 16 threads, TR rows x D/16 columns each)
// The pool's per-tensor key scale and log2(e)*softmax_scale are applied in
// fp32 exactly like the reference path: s = (q * qscale) . k_deq.
constexpr int TT2 = 64;
#ifndef PKV_ATTN_THREADS
#define PKV_ATTN_THREADS 128  // 8x8 register tiles: C3 attention step 1.80 -> 1.59 ms, C2 0.89 -> 0.62 ms vs 256
#endif
constexpr int kAttnThreads2 = PKV_ATTN_THREADS;  // 16 column groups x (threads / 16) row groups

template <int D, int RT>
struct AttnTile {
  static constexpr int TR = RT / (kAttnThreads2 / 16);  // rows per thread
  static constexpr int TD = D / 16;        // output columns per thread
  static constexpr int Q_FLOATS = D * RT;  // Qs[d][r]
  static constexpr int K_FLOATS = D * TT2; // Ks[d][t]
  static constexpr int P_FLOATS = TT2 * RT;// Ps[t][r]
  static constexpr int Y_FLOATS = TT2 * D; // Ys[t][d]
  static_assert(P_FLOATS <= K_FLOATS, "P overlays the consumed K tile");
  // raw (packed) tile staged by cp.async while the previous tile computes
  static constexpr int RAW_K = TT2 * D;            // int8 codes
  static constexpr int RAW_V = TT2 * 3 * D / 8;    // packed values
  static constexpr int RAW_S = TT2 * 4;            // f32 scales
  static constexpr int RAW = RAW_K + RAW_V + RAW_S;
  static constexpr size_t SMEM = sizeof(float) * (size_t)(Q_FLOATS + K_FLOATS + Y_FLOATS) + RAW;
};

__device__ __forceinline__ void cp_async16(void* smem, const void* gmem) {
  asm volatile("cp.async.cg.shared.global [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async4(void* smem, const void* gmem) {
  asm volatile("cp.async.ca.shared.global [%0], [%1], 4;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)), "l"(gmem)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_async_wait_all() { asm volatile("cp.async.wait_group 0;" ::: "memory"); }

template <int N>
__device__ __forceinline__ void lds_vec(const float* p, float (&v)[N]) {
  if constexpr (N == 4) {
    const float4 t = *reinterpret_cast<const float4*>(p);
    v[0] = t.x; v[1] = t.y; v[2] = t.z; v[3] = t.w;
  } else if constexpr (N == 8) {
    const float4 t0 = *reinterpret_cast<const float4*>(p), t1 = *reinterpret_cast<const float4*>(p + 4);
    v[0] = t0.x; v[1] = t0.y; v[2] = t0.z; v[3] = t0.w; v[4] = t1.x; v[5] = t1.y; v[6] = t1.z; v[7] = t1.w;
  } else {
#pragma unroll
    for (int i = 0; i < N; ++i) v[i] = p[i];
  }
}

template <int D, int RT>
__global__ void __launch_bounds__(kAttnThreads2, 2) prefix_kernel2(const __grid_constant__ Args a) {
  using AT = AttnTile<D, RT>;
  constexpr int TR = AT::TR, TD = AT::TD;
  extern __shared__ __align__(16) float sm2[];
  float* Qs = sm2;
  float* Ks = Qs + AT::Q_FLOATS;
  float* Ps = Ks;  // P overlays K once S = Q K is done
  float* Ys = Ks + AT::K_FLOATS;
  __shared__ float cent[8];

  const int h = blockIdx.y;
  const int sp = blockIdx.x;
  const int r0 = blockIdx.z * RT;
  // splits start on tile boundaries (whole tiles per split, see attn_splits)
  const long long tiles = (a.T + TT2 - 1) / TT2;
  const long long per = (tiles + a.splits - 1) / a.splits * TT2;
  const long long t_begin = (long long)sp * per, t_end = min(a.T, t_begin + per);
  const int tid = threadIdx.x;
  const int rg = tid >> 4, cg = tid & 15;  // row group, column (token / d) group
  if (tid < 8) cent[tid] = a.cent32[tid];

  // ---- Q row tile, pre-scaled by softmax_scale * log2(e): Qs[d][r] ----
  // (8 consecutive d per thread: one 16-byte load for bf16 queries)
  // (consecutive threads take consecutive rows: the transposed stores
  // Qs[d][r] are bank-conflict free)
  for (int i = tid; i < RT * D / 8; i += kAttnThreads2) {
    const int r = i % RT, d0 = (i / RT) * 8;
    const int row = r0 + r;
    float qv[8];
    if (row < a.rows) {
      const int agent = row / a.group, g = row % a.group;
      const long long off = (((long long)agent * a.kv_heads + h) * a.group + g) * D + d0;
      if (a.q_dtype == PKV_BF16) {
        const uint4 w = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.q) + off);
        qv[0] = bf16lo(w.x); qv[1] = bf16hi(w.x); qv[2] = bf16lo(w.y); qv[3] = bf16hi(w.y);
        qv[4] = bf16lo(w.z); qv[5] = bf16hi(w.z); qv[6] = bf16lo(w.w); qv[7] = bf16hi(w.w);
      } else {
        const float4 x0 = *reinterpret_cast<const float4*>(static_cast<const float*>(a.q) + off);
        const float4 x1 = *reinterpret_cast<const float4*>(static_cast<const float*>(a.q) + off + 4);
        qv[0] = x0.x; qv[1] = x0.y; qv[2] = x0.z; qv[3] = x0.w; qv[4] = x1.x; qv[5] = x1.y; qv[6] = x1.z; qv[7] = x1.w;
      }
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) qv[j] = 0.f;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) Qs[(d0 + j) * RT + r] = qv[j] * a.qscale;
  }

  float m_run[TR], l_run[TR];
  float2 acc[TR][TD / 2];  // column pairs, updated with FFMA2
#pragma unroll
  for (int i = 0; i < TR; ++i) {
    m_run[i] = -INFINITY;
    l_run[i] = 0.f;
#pragma unroll
    for (int j = 0; j < TD / 2; ++j) acc[i][j] = make_float2(0.f, 0.f);
  }
  const float ts = a.k_mode == PKV_K_TENSOR ? __ldg(a.k_scale) : 0.f;

  uint8_t* raw = reinterpret_cast<uint8_t*>(Ys + AT::Y_FLOATS);
  int8_t* rk = reinterpret_cast<int8_t*>(raw);
  uint8_t* rv = raw + AT::RAW_K;
  float* rs = reinterpret_cast<float*>(raw + AT::RAW_K + AT::RAW_V);
  // stage the packed tile [t0, t0 + nt) of head h into raw shared memory
  auto stage = [&](long long t0, int nt) {
    const int8_t* gk = a.k_codes + ((long long)h * a.T + t0) * D;
    // 16-byte chunk c of token t lands in slot c ^ (t % (D/16)) of its row, so
    // the dequant's column reads (consecutive tokens, one chunk) are
    // bank-conflict free
    for (int i = tid; i < nt * D / 16; i += kAttnThreads2) {
      const int t = i / (D / 16), c = i % (D / 16);
      cp_async16(rk + t * D + ((c ^ (t % (D / 16))) * 16), gk + i * 16);
    }
    const uint8_t* gv = a.v_packed + ((long long)h * a.T + t0) * (3 * D / 8);
    for (int i = tid; i < nt * (3 * D / 8) / 4; i += kAttnThreads2) cp_async4(rv + i * 4, gv + i * 4);
    const float* gs = a.v_scales + (long long)h * a.T + t0;
    for (int i = tid; i < nt; i += kAttnThreads2) cp_async4(rs + i, gs + i);
    cp_async_commit();
  };
  if (t_begin < t_end) stage(t_begin, (int)min((long long)TT2, t_end - t_begin));

  for (long long t0 = t_begin; t0 < t_end; t0 += TT2) {
    const int nt = (int)min((long long)TT2, t_end - t0);
    cp_async_wait_all();
    __syncthreads();  // raw tile landed; previous tile's Ks / Ys / Ps are consumed
    // ---- K tile -> Ks[d][t] (f32 dequant); 8 lanes read one token's 128 B ----
    // (consecutive threads take consecutive tokens: the transposed stores
    // Ks[d][t] are bank-conflict free; the swizzled raw rows keep the loads so)
    for (int i = tid; i < TT2 * (D / 16); i += kAttnThreads2) {
      const int t = i % TT2, d0 = (i / TT2) * 16;
      float kv[16];
      if (t < nt) {
        const uint4 w = *reinterpret_cast<const uint4*>(rk + t * D + (((d0 >> 4) ^ (t % (D / 16))) * 16));
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
        const float s = a.k_mode == PKV_K_TENSOR ? ts
                                                 : __half2float(a.k_bscale[(((long long)h * a.T + t0 + t) * D + d0) >> 5]);
#pragma unroll
        for (int j = 0; j < 16; ++j) kv[j] = (float)(int)(int8_t)((ww[j >> 2] >> (8 * (j & 3))) & 0xffu) * s;
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) kv[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) Ks[(d0 + j) * TT2 + t] = kv[j];
    }
    // ---- V tile -> Ys[t][d] = table[code] * rms ----
    for (int i = tid; i < TT2 * (D / 8); i += kAttnThreads2) {
      const int t = i / (D / 8), w8 = i % (D / 8);
      float y[8];
      if (t < nt) {
        const uint8_t* p = rv + t * (3 * D / 8) + 3 * w8;
        const uint32_t word = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16);
        const float rms = rs[t];
#pragma unroll
        for (int e = 0; e < 8; ++e) y[e] = cent[(word >> (3 * e)) & 7u] * rms;
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) y[e] = 0.f;
      }
      float4* dst = reinterpret_cast<float4*>(Ys + t * D + 8 * w8);
      dst[0] = make_float4(y[0], y[1], y[2], y[3]);
      dst[1] = make_float4(y[4], y[5], y[6], y[7]);
    }
    __syncthreads();  // raw buffer free: prefetch the next tile while this one computes
    if (t0 + TT2 < t_end) stage(t0 + TT2, (int)min((long long)TT2, t_end - t0 - TT2));

    // ---- S = Q K: thread (rg, cg) -> rows rg*TR.., tokens cg*4.. ----
    // paired fp32 FMAs (FFMA2): token pairs (k_j, k_j+1) x broadcast q_i
    float2 sc2[TR][2];
#pragma unroll
    for (int i = 0; i < TR; ++i) sc2[i][0] = sc2[i][1] = make_float2(0.f, 0.f);
#pragma unroll 4
    for (int d = 0; d < D; ++d) {
      float qa[TR];
      lds_vec<TR>(Qs + d * RT + rg * TR, qa);
      const float4 kb = *reinterpret_cast<const float4*>(Ks + d * TT2 + cg * 4);
      const float2 k01 = make_float2(kb.x, kb.y), k23 = make_float2(kb.z, kb.w);
#pragma unroll
      for (int i = 0; i < TR; ++i) {
        sc2[i][0] = __ffma2_rn(make_float2(qa[i], qa[i]), k01, sc2[i][0]);
        sc2[i][1] = __ffma2_rn(make_float2(qa[i], qa[i]), k23, sc2[i][1]);
      }
    }
    float sc[TR][4];
#pragma unroll
    for (int i = 0; i < TR; ++i) {
      sc[i][0] = sc2[i][0].x; sc[i][1] = sc2[i][0].y; sc[i][2] = sc2[i][1].x; sc[i][3] = sc2[i][1].y;
    }
    __syncthreads();  // every thread is done reading Ks (P overwrites it)
    // ---- online softmax over this tile (16 threads share a row group) ----
#pragma unroll
    for (int i = 0; i < TR; ++i) {
      float m = -INFINITY;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (cg * 4 + j >= nt) sc[i][j] = -INFINITY;
        m = fmaxf(m, sc[i][j]);
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      const float m_new = fmaxf(m_run[i], m);
      const float corr = exp2f(m_run[i] - m_new);  // 0 on the first tile
      float l = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float p = exp2f(sc[i][j] - m_new);
        sc[i][j] = p;
        l += p;
      }
#pragma unroll
      for (int o = 8; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
      l_run[i] = l_run[i] * corr + l;
      m_run[i] = m_new;
#pragma unroll
      for (int j = 0; j < TD / 2; ++j) acc[i][j] = __fmul2_rn(acc[i][j], make_float2(corr, corr));
#pragma unroll
      for (int j = 0; j < 4; ++j) Ps[(cg * 4 + j) * RT + rg * TR + i] = sc[i][j];
    }
    __syncthreads();
    // ---- O += P Y: thread (rg, cg) -> rows rg*TR.., columns cg*TD.. ----
#pragma unroll 4
    for (int t = 0; t < TT2; ++t) {
      float pa[TR], yb[TD];
      lds_vec<TR>(Ps + t * RT + rg * TR, pa);
      lds_vec<TD>(Ys + t * D + cg * TD, yb);
#pragma unroll
      for (int i = 0; i < TR; ++i)
#pragma unroll
        for (int j = 0; j < TD / 2; ++j)
          acc[i][j] = __ffma2_rn(make_float2(pa[i], pa[i]), make_float2(yb[2 * j], yb[2 * j + 1]), acc[i][j]);
    }
  }
  // ---- partial: [h][split][row][0..D) acc, D: m, D+1: l ----
#pragma unroll
  for (int i = 0; i < TR; ++i) {
    const int row = r0 + rg * TR + i;
    if (row >= a.rows) continue;
    float* dst = a.part + (((long long)h * a.splits + sp) * a.rows + row) * (D + 4);
#pragma unroll
    for (int j = 0; j < TD / 2; ++j) {
      dst[cg * TD + 2 * j] = acc[i][j].x;
      dst[cg * TD + 2 * j + 1] = acc[i][j].y;
    }
    if (cg == 0) {
      dst[D] = m_run[i];
      dst[D + 1] = l_run[i];
    }
  }
}

// One CTA of kCombineWarps warps per (row, kv head): the warps merge
// interleaved subsets of the splits, warp 0 folds their results, then
// inverse-rotates and adds the private tail.
constexpr int kCombineWarps = 4;
template <int D>
__global__ void __launch_bounds__(32 * kCombineWarps) combine_kernel(const __grid_constant__ Args a) {
  constexpr int EPL = D / 32;  // coordinates per lane: lane holds [EPL*lane, EPL*lane+EPL)
  __shared__ float s_acc[kCombineWarps][D];
  __shared__ float s_ml[kCombineWarps][2];
  const int wid = threadIdx.x >> 5;
  const int lane = threadIdx.x & 31;
  const int row = blockIdx.x / a.kv_heads;
  const int h = blockIdx.x % a.kv_heads;
  const int agent = row / a.group, g = row % a.group;

  const long long stride = (long long)a.rows * (D + 4);  // between splits
  const float* base = a.part + ((long long)h * a.splits * a.rows + row) * (D + 4);
  // this warp's splits (wid, wid + W, ...), CH at a time: the CH partials'
  // loads are all issued before any is used (one L2 round trip per chunk),
  // then folded with an online max
  constexpr int CH = 8;
  float M = -INFINITY, L = 0.f;
  float acc[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) acc[j] = 0.f;
  for (int s0 = wid; s0 < a.splits; s0 += kCombineWarps * CH) {
    float mv[CH], lv[CH], vv[CH][EPL];
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const int sidx = s0 + c * kCombineWarps;
      if (sidx < a.splits) {
        const float* src = base + sidx * stride;
        mv[c] = src[D];
        lv[c] = src[D + 1];
        if constexpr (EPL == 4) {
          const float4 t = *reinterpret_cast<const float4*>(src + 4 * lane);
          vv[c][0] = t.x; vv[c][1] = t.y; vv[c][2] = t.z; vv[c][3] = t.w;
        } else {
#pragma unroll
          for (int j = 0; j < EPL; ++j) vv[c][j] = src[EPL * lane + j];
        }
      } else {
        mv[c] = -INFINITY;
        lv[c] = 0.f;
#pragma unroll
        for (int j = 0; j < EPL; ++j) vv[c][j] = 0.f;
      }
    }
    float mc = M;
#pragma unroll
    for (int c = 0; c < CH; ++c) mc = fmaxf(mc, mv[c]);
    if (mc == -INFINITY) continue;  // no tokens in these splits
    const float r = exp2f(M - mc);   // M = -inf: 0 (acc and L are 0 then)
    L *= r;
#pragma unroll
    for (int j = 0; j < EPL; ++j) acc[j] *= r;
#pragma unroll
    for (int c = 0; c < CH; ++c) {
      const float w = exp2f(mv[c] - mc);  // an empty split (-inf) weighs 0
      L = fmaf(w, lv[c], L);
#pragma unroll
      for (int j = 0; j < EPL; ++j) acc[j] = fmaf(w, vv[c][j], acc[j]);
    }
    M = mc;
  }
#pragma unroll
  for (int j = 0; j < EPL; ++j) s_acc[wid][EPL * lane + j] = acc[j];
  if (lane == 0) {
    s_ml[wid][0] = M;
    s_ml[wid][1] = L;
  }
  __syncthreads();
  if (wid != 0) return;
  {
    float Mg = -INFINITY;
#pragma unroll
    for (int w = 0; w < kCombineWarps; ++w) Mg = fmaxf(Mg, s_ml[w][0]);
    L = 0.f;
#pragma unroll
    for (int j = 0; j < EPL; ++j) acc[j] = 0.f;
#pragma unroll
    for (int w = 0; w < kCombineWarps; ++w) {
      const float mw = s_ml[w][0];
      const float c = mw == -INFINITY ? 0.f : exp2f(mw - Mg);  // a warp without splits contributes nothing
      L = fmaf(c, s_ml[w][1], L);
#pragma unroll
      for (int j = 0; j < EPL; ++j) acc[j] = fmaf(c, s_acc[w][EPL * lane + j], acc[j]);
    }
    M = Mg;
  }
  // inverse rotation of the merged rotated-domain accumulator:
  // in-lane stages over the low log2(EPL) bits, shuffles over the lane bits
#pragma unroll
  for (int hh = 1; hh < EPL; hh <<= 1) {
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      if (e & hh) continue;
      const float x0 = acc[e], x1 = acc[e + hh];
      acc[e] = x0 + x1;
      acc[e + hh] = x0 - x1;
    }
  }
#pragma unroll
  for (int lb = 0; lb < 5; ++lb) {
    const float sg = ((lane >> lb) & 1) ? -1.f : 1.f;
#pragma unroll
    for (int e = 0; e < EPL; ++e) {
      const float p = __shfl_xor_sync(0xffffffffu, acc[e], 1 << lb);
      acc[e] = fmaf(sg, acc[e], p);
    }
  }
  const float inv_sqrt_d = rsqrtf((float)D);
#pragma unroll
  for (int e = 0; e < EPL; ++e) {
    acc[e] *= inv_sqrt_d;
    if (a.use_sign && sign_bit(a.sign_bits, EPL * lane + e)) acc[e] = -acc[e];
  }

  // private tail (bf16), online-merged in the original domain
  // clamped: a tail_len past the buffer (e.g. a graph replayed beyond its
  // capacity) must not read out of bounds
  const int tl = a.tail_len ? max(0, min(a.tail_len[agent], a.tail_cap)) : 0;
  if (tl > 0) {
    const __nv_bfloat16* tk = static_cast<const __nv_bfloat16*>(a.tail_k);
    const __nv_bfloat16* tv = static_cast<const __nv_bfloat16*>(a.tail_v);
    float qv[EPL];
#pragma unroll
    for (int e = 0; e < EPL; ++e)
      qv[e] = ldq(a, (((long long)agent * a.kv_heads + h) * a.group + g) * D + EPL * lane + e) *
              a.qscale;
    for (int j = 0; j < tl; ++j) {
      const long long base = (((long long)agent * a.kv_heads + h) * a.tail_cap + j) * D;
      float sdot = 0.f;
#pragma unroll
      for (int e = 0; e < EPL; ++e) sdot = fmaf(qv[e], __bfloat162float(tk[base + EPL * lane + e]), sdot);
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) sdot += __shfl_xor_sync(0xffffffffu, sdot, o);
      const float Mn = fmaxf(M, sdot);
      const float c_old = exp2f(M - Mn), p = exp2f(sdot - Mn);
      L = L * c_old + p;
#pragma unroll
      for (int e = 0; e < EPL; ++e)
        acc[e] = fmaf(acc[e], c_old, p * __bfloat162float(tv[base + EPL * lane + e]));
      M = Mn;
    }
  }
  const float invL = 1.f / L;
  const long long ob = (((long long)agent * a.kv_heads + h) * a.group + g) * D + EPL * lane;
  if (a.out_dtype == PKV_F32) {
    float* o = static_cast<float*>(a.out) + ob;
#pragma unroll
    for (int e = 0; e < EPL; ++e) o[e] = acc[e] * invL;
  } else {
    __nv_bfloat16* o = static_cast<__nv_bfloat16*>(a.out) + ob;
#pragma unroll
    for (int e = 0; e < EPL; ++e) o[e] = __float2bfloat16_rn(acc[e] * invL);
  }
}

// splits per head: about `per_sm` CTAs per SM (co-resident CTAs hide each
// other's tile loads), each split at least one tile. 64-row tiles fit two
// CTAs per SM (shared memory); the 16-row tile (rows <= 16) fits more at d=64.
// PKV_ATTN_CTAS_PER_SM overrides (tuning only).
#ifndef PKV_ATTN_SMALL_PER_SM
#define PKV_ATTN_SMALL_PER_SM 8  // d=64 (C2, 5 rows per head): 0.58 -> 0.49 ms per 24-layer step vs 2
#endif
inline int attn_splits(int kv_heads, long long T, int rows, int head_dim) {
  const int env_per_sm = tuning().attn_ctas_per_sm;
  const int rt = rows <= 16 ? 16 : 64;
  const int row_tiles = (rows + rt - 1) / rt;
  const int per_sm = env_per_sm > 0 ? env_per_sm : (rt == 16 && head_dim == 64 ? PKV_ATTN_SMALL_PER_SM : 2);
  // (16-row tiles at d=128 fill shared memory at two CTAs per SM as well)
  int dev = 0, sms = 148;
  cudaGetDevice(&dev);
  cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long den = (long long)kv_heads * row_tiles;
  const long long want = std::max(1LL, ((long long)per_sm * sms + den - 1) / den);
  // whole tiles per split (a ragged split costs a full tile step), then the
  // fewest splits of that length
  const long long tiles = (T + TT2 - 1) / TT2;
  const long long per = (tiles + want - 1) / want;
  return (int)((tiles + per - 1) / per);
}

template <int D, int RTILE>
int launch_rt(Args& a, cudaStream_t st) {
  using AT = AttnTile<D, RTILE>;
  if (cudaFuncSetAttribute(prefix_kernel2<D, RTILE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)AT::SMEM) != cudaSuccess)
    return PKV_ERR_CUDA;
  const int row_tiles = (a.rows + RTILE - 1) / RTILE;
  dim3 grid(a.splits, a.kv_heads, row_tiles);
  prefix_kernel2<D, RTILE><<<grid, kAttnThreads2, AT::SMEM, st>>>(a);
  if (cudaGetLastError() != cudaSuccess) return PKV_ERR_CUDA;
  combine_kernel<D><<<a.rows * a.kv_heads, 32 * kCombineWarps, 0, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? PKV_OK : PKV_ERR_CUDA;
}

template <int D>
int launch(Args& a, cudaStream_t st) {
  return a.rows <= 16 ? launch_rt<D, 16>(a, st) : launch_rt<D, 64>(a, st);
}

}  // namespace attn
}  // namespace pkv

extern "C" {

size_t pkv_attention_workspace_bytes(int num_rows, int kv_heads, int group, int head_dim,
                                     int64_t seq_len) {
  if (num_rows < 1 || kv_heads < 1 || group < 1 || head_dim < 1 || seq_len < 1) return 0;
  const int rows = num_rows * group;
  const int splits = pkv::attn::attn_splits(kv_heads, seq_len, rows, head_dim);
  return sizeof(float) * (size_t)kv_heads * (size_t)splits * (size_t)rows * (size_t)(head_dim + 4);
}

int pkv_decode_attention(int num_rows, int kv_heads, int group, int head_dim, int64_t seq_len,
                         int q_dtype, const void* q, int k_mode, const int8_t* k_codes,
                         const float* k_scale, const uint16_t* k_bscale, const uint8_t* v_packed,
                         const float* v_scales, const double* centroids_host,
                         const uint32_t* sign_bits_host, const void* tail_k, const void* tail_v,
                         const int32_t* tail_len, int tail_cap, float softmax_scale,
                         int out_dtype, void* out, void* workspace, size_t workspace_bytes,
                         void* stream) {
  using namespace pkv::attn;
  if (num_rows < 1 || kv_heads < 1 || group < 1 || seq_len < 1) return PKV_ERR_INVALID_ARG;
  if (head_dim != 64 && head_dim != 128) return PKV_ERR_UNSUPPORTED_HEAD_DIM;
  if ((q_dtype != PKV_F32 && q_dtype != PKV_BF16) || (out_dtype != PKV_F32 && out_dtype != PKV_BF16))
    return PKV_ERR_INVALID_ARG;
  if (k_mode != PKV_K_TENSOR && k_mode != PKV_K_BLOCK32) return PKV_ERR_INVALID_ARG;
  if (!q || !k_codes || !v_packed || !v_scales || !out || !centroids_host) return PKV_ERR_INVALID_ARG;
  if (k_mode == PKV_K_TENSOR ? !k_scale : !k_bscale) return PKV_ERR_INVALID_ARG;
  if (tail_len && (!tail_k || !tail_v || tail_cap < 1)) return PKV_ERR_INVALID_ARG;
  if ((reinterpret_cast<uintptr_t>(k_codes) & 15u) != 0) return PKV_ERR_ALIGNMENT;
  const size_t need = pkv_attention_workspace_bytes(num_rows, kv_heads, group, head_dim, seq_len);
  if (!workspace || workspace_bytes < need) return PKV_ERR_WORKSPACE;
  for (int i = 0; i < 8; ++i)
    if (!std::isfinite(centroids_host[i])) return PKV_ERR_UNSUPPORTED_CODEBOOK;

  Args a;
  std::memset(&a, 0, sizeof(a));
  a.rows = num_rows * group;
  a.kv_heads = kv_heads;
  a.group = group;
  a.head_dim = head_dim;
  a.T = seq_len;
  a.q_dtype = q_dtype;
  a.out_dtype = out_dtype;
  a.k_mode = k_mode;
  a.splits = attn_splits(kv_heads, seq_len, a.rows, head_dim);
  a.qscale = softmax_scale * kLog2e;
  for (int i = 0; i < 8; ++i) a.cent32[i] = (float)centroids_host[i];
  if (sign_bits_host) {
    a.use_sign = 1;
    for (int i = 0; i < (head_dim + 31) / 32; ++i) a.sign_bits[i] = sign_bits_host[i];
  }
  a.q = q;
  a.k_codes = k_codes;
  a.k_scale = k_scale;
  a.k_bscale = reinterpret_cast<const __half*>(k_bscale);
  a.v_packed = v_packed;
  a.v_scales = v_scales;
  a.tail_k = tail_k;
  a.tail_v = tail_v;
  a.tail_len = tail_len;
  a.tail_cap = tail_cap;
  a.part = static_cast<float*>(workspace);
  a.out = out;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return head_dim == 64 ? launch<64>(a, st) : launch<128>(a, st);
}

}  // extern "C"
