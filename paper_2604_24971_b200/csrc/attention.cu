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
#include "diag.h"
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
  int q_len;       // query positions per agent (rows of an agent: group = G * q_len, position = g % q_len)
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
__device__ __forceinline__ void cp_async_wait_one() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

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

// ---------------------------------------------------------------------------
// prefix kernel, tensor-core version (mma.sync m16n8k16, f16 in / f32 acc)
// ---------------------------------------------------------------------------
// Same split / partial layout as prefix_kernel2 (the combine kernel is
// shared), but S = Q K^T and O += P Y run on the tensor cores. Precision:
//   * K codes are integers |c| <= 128: exact in f16; the per-tensor key
//     scale is applied to S in f32 after the MMA (block32: f16(code * s16));
//   * Q (pre-scaled by softmax_scale * log2 e) is split hi + lo in f16
//     (two MMAs, ~2^-22 relative), so large logits keep f32-like accuracy;
//   * the rotated-domain values Y = centroid[code] * rms are factored:
//     rms scales P (per token, f32) and the centroids are split hi + lo in
//     f16 (two MMAs): the centroid rounding is systematic across tokens and
//     would not average out;
//   * P' = p * rms is rounded to f16 (random per token).
// CTA = 4 warps; WR warps along rows (16 rows each), 4 / WR along the
// tokens of each 64-token tile (rows <= 16: WR = 1, the four warps split
// the tile and merge their online-softmax states at the end).
namespace mma {

__device__ __forceinline__ void ldsm_x4(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void ldsm_x4_t(uint32_t addr, uint32_t (&r)[4]) {
  asm volatile("ldmatrix.sync.aligned.m8n8.x4.trans.shared.b16 {%0,%1,%2,%3}, [%4];"
               : "=r"(r[0]), "=r"(r[1]), "=r"(r[2]), "=r"(r[3])
               : "r"(addr));
}
__device__ __forceinline__ void mma16816(float (&c)[4], const uint32_t (&a)[4], uint32_t b0, uint32_t b1) {
  asm volatile("mma.sync.aligned.m16n8k16.row.col.f32.f16.f16.f32 {%0,%1,%2,%3}, {%4,%5,%6,%7}, {%8,%9}, "
               "{%0,%1,%2,%3};"
               : "+f"(c[0]), "+f"(c[1]), "+f"(c[2]), "+f"(c[3])
               : "r"(a[0]), "r"(a[1]), "r"(a[2]), "r"(a[3]), "r"(b0), "r"(b1));
}
__device__ __forceinline__ uint32_t h2u(__half2 h) { return *reinterpret_cast<uint32_t*>(&h); }
__device__ __forceinline__ __half2 u2h(uint32_t u) { return *reinterpret_cast<__half2*>(&u); }
// f32 pair -> (hi, lo) f16 pairs with hi + lo == x to ~2^-22
__device__ __forceinline__ void split2(float x, float y, uint32_t& hi, uint32_t& lo) {
  const __half2 h = __floats2half2_rn(x, y);
  const float2 hf = __half22float2(h);
  hi = h2u(h);
  lo = h2u(__floats2half2_rn(x - hf.x, y - hf.y));
}
// byte offset of 16-byte chunk c of row r in a [rows][D] f16 tile, XOR-swizzled
// so that ldmatrix reads of 8 consecutive rows hit 8 distinct chunk slots
template <int D>
__device__ __forceinline__ uint32_t sw(int r, int c) {
  return (uint32_t)(r * (2 * D) + ((c ^ (r & 7)) << 4));
}

template <int D, int WR>
struct MmaTile {
  static constexpr int RT = 16 * WR;            // rows per CTA
  static constexpr int WT = 4 / WR;             // warps along tokens
  static constexpr int TT = 64;                 // tokens per tile
  static constexpr int TW = TT / WT;            // tokens per warp per tile
  static constexpr int Q_BYTES = RT * D * 2;    // one f16 Q tile (hi or lo)
  static constexpr int T_BYTES = TT * D * 2;    // one f16 K / Y tile
  static constexpr int RAW = TT * D + TT * 3 * D / 8 + TT * 4;
  static constexpr int MERGE = WT > 1 ? 4 * 16 * (D + 2) * 4 : 0;  // every warp's 16-row state
  static constexpr int MAIN = 2 * Q_BYTES + 3 * T_BYTES + TT * 4 + 2 * RAW;  // raw tiles double-buffered
  static constexpr int SMEM = (MAIN > MERGE ? MAIN : MERGE) + 128 * 8 * 4 + 128;
};

}  // namespace mma

template <int D, int WR>
__global__ void __launch_bounds__(128) prefix_mma(const __grid_constant__ Args a) {
  using namespace mma;
  using MT = MmaTile<D, WR>;
  constexpr int RT = MT::RT, WT = MT::WT, TT = MT::TT, TW = MT::TW;
  constexpr int NB = TW / 8;   // S n-blocks (8 tokens) per warp per tile
  constexpr int KS = D / 16;   // k-steps of S
  constexpr int ND = D / 8;    // O n-blocks (8 dims)
  extern __shared__ __align__(128) uint8_t smm[];
  uint8_t* qhi = smm;
  uint8_t* qlo = qhi + MT::Q_BYTES;
  uint8_t* kh = qlo + MT::Q_BYTES;
  uint8_t* yhi = kh + MT::T_BYTES;
  uint8_t* ylo = yhi + MT::T_BYTES;
  float* rms_s = reinterpret_cast<float*>(ylo + MT::T_BYTES);
  uint8_t* raw0 = reinterpret_cast<uint8_t*>(rms_s + TT);  // two raw (packed) tile buffers
  // per-thread (conflict-free) table: code -> (centroid hi, centroid lo) f16 bits
  uint32_t* ctab = reinterpret_cast<uint32_t*>(smm + (MT::MAIN > MT::MERGE ? MT::MAIN : MT::MERGE));

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int wr = warp % WR, wt = warp / WR;  // row block, token slice
  const int h = blockIdx.y, sp = blockIdx.x, r0 = blockIdx.z * RT;
  const long long tiles = (a.T + TT - 1) / TT;
  const long long per = (tiles + a.splits - 1) / a.splits * TT;
  const long long t_begin = (long long)sp * per, t_end = min(a.T, t_begin + per);
#pragma unroll
  for (int k = 0; k < 8; ++k) {
    const __half hc = __float2half_rn(a.cent32[k]);
    const __half lc = __float2half_rn(a.cent32[k] - __half2float(hc));
    ctab[k * 128 + tid] = (uint32_t)__half_as_ushort(hc) | ((uint32_t)__half_as_ushort(lc) << 16);
  }
  const float ts = a.k_mode == PKV_K_TENSOR ? __ldg(a.k_scale) : 1.f;
  // raw tile layout: int8 codes [TT][D] | packed values [TT][3D/8] | f32 scales [TT]
  auto stage = [&](long long t0, int nt, uint8_t* buf) {
    const int8_t* gk = a.k_codes + ((long long)h * a.T + t0) * D;
    for (int i = tid; i < nt * D / 16; i += 128) cp_async16(buf + i * 16, gk + i * 16);
    const uint8_t* gv = a.v_packed + ((long long)h * a.T + t0) * (3 * D / 8);
    uint8_t* bv = buf + TT * D;
    for (int i = tid; i < nt * (3 * D / 8) / 4; i += 128) cp_async4(bv + i * 4, gv + i * 4);
    const float* gs = a.v_scales + (long long)h * a.T + t0;
    float* bs = reinterpret_cast<float*>(buf + TT * D + TT * 3 * D / 8);
    for (int i = tid; i < nt; i += 128) cp_async4(bs + i, gs + i);
    cp_async_commit();
  };
  // two tiles in flight: tile i + 1 loads while tile i converts and computes
  if (t_begin < t_end) stage(t_begin, (int)min((long long)TT, t_end - t_begin), raw0);
  if (t_begin + TT < t_end) stage(t_begin + TT, (int)min((long long)TT, t_end - t_begin - TT), raw0 + MT::RAW);
  // (Q is loaded while the first two tiles are in flight)
  // ---- Q tile (x qscale), split hi / lo, f16 swizzled [RT][D] ----
  for (int i = tid; i < RT * D / 8; i += 128) {
    const int r = i / (D / 8), c = i % (D / 8);
    const int row = r0 + r;
    float qv[8];
    if (row < a.rows) {
      const int agent = row / a.group, g = row % a.group;
      const long long off = (((long long)agent * a.kv_heads + h) * a.group + g) * D + c * 8;
      if (a.q_dtype == PKV_BF16) {
        const uint4 w = *reinterpret_cast<const uint4*>(static_cast<const __nv_bfloat16*>(a.q) + off);
        qv[0] = bf16lo(w.x); qv[1] = bf16hi(w.x); qv[2] = bf16lo(w.y); qv[3] = bf16hi(w.y);
        qv[4] = bf16lo(w.z); qv[5] = bf16hi(w.z); qv[6] = bf16lo(w.w); qv[7] = bf16hi(w.w);
      } else {
        const float4 x0 = *reinterpret_cast<const float4*>(static_cast<const float*>(a.q) + off);
        const float4 x1 = *reinterpret_cast<const float4*>(static_cast<const float*>(a.q) + off + 4);
        qv[0] = x0.x; qv[1] = x0.y; qv[2] = x0.z; qv[3] = x0.w; qv[4] = x1.x; qv[5] = x1.y; qv[6] = x1.z; qv[7] = x1.w;
      }
#pragma unroll
      for (int j = 0; j < 8; ++j) qv[j] *= a.qscale;
    } else {
#pragma unroll
      for (int j = 0; j < 8; ++j) qv[j] = 0.f;
    }
    uint32_t hi[4], lo[4];
#pragma unroll
    for (int j = 0; j < 4; ++j) split2(qv[2 * j], qv[2 * j + 1], hi[j], lo[j]);
    *reinterpret_cast<uint4*>(qhi + sw<D>(r, c)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
    *reinterpret_cast<uint4*>(qlo + sw<D>(r, c)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
  }

  float o[ND][4];
#pragma unroll
  for (int j = 0; j < ND; ++j) o[j][0] = o[j][1] = o[j][2] = o[j][3] = 0.f;
  float m_run[2] = {-INFINITY, -INFINITY}, l_run[2] = {0.f, 0.f};  // rows g, g + 8
  const int g = lane >> 2, t4 = lane & 3;
  const uint32_t qhi_s = (uint32_t)__cvta_generic_to_shared(qhi), qlo_s = (uint32_t)__cvta_generic_to_shared(qlo);
  const uint32_t kh_s = (uint32_t)__cvta_generic_to_shared(kh);
  const uint32_t yhi_s = (uint32_t)__cvta_generic_to_shared(yhi), ylo_s = (uint32_t)__cvta_generic_to_shared(ylo);
  const int qrow = wr * 16;

  int it = 0;
  for (long long t0 = t_begin; t0 < t_end; t0 += TT, ++it) {
    const int nt = (int)min((long long)TT, t_end - t0);
    uint8_t* raw = raw0 + (it & 1) * MT::RAW;
    const int8_t* rk = reinterpret_cast<const int8_t*>(raw);
    const uint8_t* rv = raw + TT * D;
    const float* rs = reinterpret_cast<const float*>(raw + TT * D + TT * 3 * D / 8);
    if (t0 + TT < t_end) cp_async_wait_one();  // this tile landed (the next may still be in flight)
    else cp_async_wait_all();
    __syncthreads();  // raw tile landed; every warp is done with the previous K / Y tiles
    // ---- K: int8 codes -> f16 (exact; block32: x f16 scale), 16 codes per thread-step ----
#ifndef PKV_ATTN_SKIP_K  // (timing experiment)
    for (int i = tid; i < TT * D / 16; i += 128) {
      const int t = i / (D / 16), c = i % (D / 16);
      uint4 w = make_uint4(0x80808080u, 0x80808080u, 0x80808080u, 0x80808080u);  // code 0
      __half2 sc2 = __float2half2_rn(1.f);
      if (t < nt) {
        w = *reinterpret_cast<const uint4*>(rk + t * D + c * 16);
        w.x ^= 0x80808080u; w.y ^= 0x80808080u; w.z ^= 0x80808080u; w.w ^= 0x80808080u;
        if (a.k_mode != PKV_K_TENSOR)
          sc2 = __half2half2(a.k_bscale[(((long long)h * a.T + t0 + t) * D + c * 16) >> 5]);
      }
      const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
      const __half2 bias = __float2half2_rn(1152.f);  // 1024 + 128
      uint32_t hv[8];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        __half2 lo2 = __hsub2(u2h(__byte_perm(ww[j], 0x64646464u, 0x5140)), bias);
        __half2 hi2 = __hsub2(u2h(__byte_perm(ww[j], 0x64646464u, 0x7362)), bias);
        if (a.k_mode != PKV_K_TENSOR) {
          lo2 = __hmul2(lo2, sc2);
          hi2 = __hmul2(hi2, sc2);
        }
        hv[2 * j] = h2u(lo2);
        hv[2 * j + 1] = h2u(hi2);
      }
      *reinterpret_cast<uint4*>(kh + sw<D>(t, 2 * c)) = make_uint4(hv[0], hv[1], hv[2], hv[3]);
      *reinterpret_cast<uint4*>(kh + sw<D>(t, 2 * c + 1)) = make_uint4(hv[4], hv[5], hv[6], hv[7]);
    }
#endif
    // ---- V: 3-bit codes -> centroid hi / lo f16 tiles; rms per token ----
#ifndef PKV_ATTN_SKIP_V  // (timing experiment: PKV_ATTN_SKIP_V=1 leaves the V tiles unconverted)
    // (four packed 24-bit words = 32 codes per step, read as three aligned
    // 32-bit words instead of twelve bytes)
    for (int i = tid; i < TT * D / 32; i += 128) {
      const int t = i / (D / 32), cg = i % (D / 32);
      uint32_t wd[4] = {0, 0, 0, 0};
      if (t < nt) {
        const uint32_t* p = reinterpret_cast<const uint32_t*>(rv + t * (3 * D / 8) + 12 * cg);
        const uint32_t u0 = p[0], u1 = p[1], u2 = p[2];
        wd[0] = u0 & 0xffffffu;
        wd[1] = __funnelshift_r(u0, u1, 24) & 0xffffffu;
        wd[2] = __funnelshift_r(u1, u2, 16) & 0xffffffu;
        wd[3] = u2 >> 8;
      }
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        uint32_t hi[4] = {0, 0, 0, 0}, lo[4] = {0, 0, 0, 0};
        if (t < nt) {
#pragma unroll
          for (int e = 0; e < 8; e += 2) {
            const uint32_t x0 = ctab[((wd[q] >> (3 * e)) & 7u) * 128 + tid];
            const uint32_t x1 = ctab[((wd[q] >> (3 * e + 3)) & 7u) * 128 + tid];
            hi[e / 2] = __byte_perm(x0, x1, 0x5410);
            lo[e / 2] = __byte_perm(x0, x1, 0x7632);
          }
        }
        *reinterpret_cast<uint4*>(yhi + sw<D>(t, 4 * cg + q)) = make_uint4(hi[0], hi[1], hi[2], hi[3]);
        *reinterpret_cast<uint4*>(ylo + sw<D>(t, 4 * cg + q)) = make_uint4(lo[0], lo[1], lo[2], lo[3]);
      }
    }
#endif
    for (int i = tid; i < TT; i += 128) rms_s[i] = i < nt ? rs[i] : 0.f;
    __syncthreads();  // tiles converted; this raw buffer is free for tile i + 2
    if (t0 + 2 * TT < t_end) stage(t0 + 2 * TT, (int)min((long long)TT, t_end - t0 - 2 * TT), raw);

    // ---- S = Q K^T over this warp's TW tokens ----
    const int tw0 = wt * TW;
    float s[NB][4];
#pragma unroll
    for (int n = 0; n < NB; ++n) s[n][0] = s[n][1] = s[n][2] = s[n][3] = 0.f;
#pragma unroll
    for (int k = 0; k < KS; ++k) {
      uint32_t ah[4], al[4];
      const int ar = qrow + (lane & 7) + 8 * ((lane >> 3) & 1), ac = 2 * k + (lane >> 4);
      ldsm_x4(qhi_s + sw<D>(ar, ac), ah);
      ldsm_x4(qlo_s + sw<D>(ar, ac), al);
      uint32_t b[NB / 2][4];
#pragma unroll
      for (int n = 0; n < NB; n += 2) {
        const int br = tw0 + n * 8 + (lane & 7) + 8 * (lane >> 4), bc = 2 * k + ((lane >> 3) & 1);
        ldsm_x4(kh_s + sw<D>(br, bc), b[n / 2]);
      }
      // the hi and lo products of one accumulator are NB MMAs apart (no
      // back-to-back dependent MMAs)
#pragma unroll
      for (int n = 0; n < NB; n += 2) {
        mma16816(s[n], ah, b[n / 2][0], b[n / 2][1]);
        mma16816(s[n + 1], ah, b[n / 2][2], b[n / 2][3]);
      }
#pragma unroll
      for (int n = 0; n < NB; n += 2) {
        mma16816(s[n], al, b[n / 2][0], b[n / 2][1]);
        mma16816(s[n + 1], al, b[n / 2][2], b[n / 2][3]);
      }
    }
    // ---- online softmax (rows g and g + 8 of this warp's 16) ----
    float mx[2] = {-INFINITY, -INFINITY};
#pragma unroll
    for (int n = 0; n < NB; ++n)
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const int tok = tw0 + n * 8 + 2 * t4 + (j & 1);
        s[n][j] = tok < nt ? s[n][j] * ts : -INFINITY;
        mx[j >> 1] = fmaxf(mx[j >> 1], s[n][j]);
      }
    float corr[2];
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      mx[rr] = fmaxf(mx[rr], __shfl_xor_sync(0xffffffffu, mx[rr], 1));
      mx[rr] = fmaxf(mx[rr], __shfl_xor_sync(0xffffffffu, mx[rr], 2));
      const float m_new = fmaxf(m_run[rr], mx[rr]);
      // a slice with no tokens yet (m_new = -inf) keeps everything at 0
      corr[rr] = m_new == -INFINITY ? 1.f : exp2f(m_run[rr] - m_new);
      m_run[rr] = m_new;
    }
    float lsum[2] = {0.f, 0.f};
    uint32_t pa[NB][2];  // P' = p * rms as f16 pairs: [n][row g / g + 8]
#pragma unroll
    for (int n = 0; n < NB; ++n) {
      const int tok = tw0 + n * 8 + 2 * t4;
      const float2 rm = *reinterpret_cast<const float2*>(rms_s + tok);
      float p[4];
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float m = m_run[j >> 1];
        p[j] = m == -INFINITY ? 0.f : exp2f(s[n][j] - m);
        lsum[j >> 1] += p[j];
      }
      pa[n][0] = h2u(__floats2half2_rn(p[0] * rm.x, p[1] * rm.y));
      pa[n][1] = h2u(__floats2half2_rn(p[2] * rm.x, p[3] * rm.y));
    }
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      lsum[rr] += __shfl_xor_sync(0xffffffffu, lsum[rr], 1);
      lsum[rr] += __shfl_xor_sync(0xffffffffu, lsum[rr], 2);
      l_run[rr] = l_run[rr] * corr[rr] + lsum[rr];
    }
#pragma unroll
    for (int j = 0; j < ND; ++j) {
      float2 lo = __fmul2_rn(make_float2(o[j][0], o[j][1]), make_float2(corr[0], corr[0]));
      float2 hi = __fmul2_rn(make_float2(o[j][2], o[j][3]), make_float2(corr[1], corr[1]));
      o[j][0] = lo.x; o[j][1] = lo.y; o[j][2] = hi.x; o[j][3] = hi.y;
    }
    // ---- O += P' (Y_hi + Y_lo) over the warp's tokens, 16 tokens per k-step ----
#pragma unroll
    for (int kk = 0; kk < TW / 16; ++kk) {
      const uint32_t af[4] = {pa[2 * kk][0], pa[2 * kk][1], pa[2 * kk + 1][0], pa[2 * kk + 1][1]};
      const int br = tw0 + kk * 16 + (lane & 7) + 8 * ((lane >> 3) & 1);
#pragma unroll
      for (int j = 0; j < ND; j += 2) {
        uint32_t bh[4];
        ldsm_x4_t(yhi_s + sw<D>(br, j + (lane >> 4)), bh);
        mma16816(o[j], af, bh[0], bh[1]);
        mma16816(o[j + 1], af, bh[2], bh[3]);
      }
#pragma unroll
      for (int j = 0; j < ND; j += 2) {
        uint32_t bl[4];
        ldsm_x4_t(ylo_s + sw<D>(br, j + (lane >> 4)), bl);
        mma16816(o[j], af, bl[0], bl[1]);
        mma16816(o[j + 1], af, bl[2], bl[3]);
      }
    }
  }

  // let the combine kernel's launch start while this grid finishes
  asm volatile("griddepcontrol.launch_dependents;" ::: "memory");
  // ---- partials: [h][split][row][0..D) acc, D: m, D+1: l ----
  if constexpr (WT > 1) {
    __syncthreads();  // tiles no longer needed: reuse shared memory to merge the token slices
    float* mrg = reinterpret_cast<float*>(smm);
    float* mine = mrg + (wt * WR + wr) * 16 * (D + 2);  // [token slice][row block][16 rows][D + 2]
#pragma unroll
    for (int j = 0; j < ND; ++j) {
      const int c = j * 8 + 2 * t4;
      mine[g * (D + 2) + c] = o[j][0];
      mine[g * (D + 2) + c + 1] = o[j][1];
      mine[(g + 8) * (D + 2) + c] = o[j][2];
      mine[(g + 8) * (D + 2) + c + 1] = o[j][3];
    }
    if (t4 == 0) {
      mine[g * (D + 2) + D] = m_run[0];
      mine[g * (D + 2) + D + 1] = l_run[0];
      mine[(g + 8) * (D + 2) + D] = m_run[1];
      mine[(g + 8) * (D + 2) + D + 1] = l_run[1];
    }
    __syncthreads();
    // 128 threads: thread -> (row of the RT-row tile, column)
    for (int i = tid; i < RT * (D + 2); i += 128) {
      const int r = i / (D + 2), c = i % (D + 2);
      const int row = r0 + r;
      if (row >= a.rows || c == D + 1) continue;
      const float* st = mrg + ((r >> 4) * 16 + (r & 15)) * (D + 2);  // slice 0, row block r / 16
      constexpr int SL = WR * 16 * (D + 2);                          // stride between token slices
      float M = -INFINITY;
#pragma unroll
      for (int w = 0; w < WT; ++w) M = fmaxf(M, st[w * SL + D]);
      float* dst = a.part + (((long long)h * a.splits + sp) * a.rows + row) * (D + 4);
      float v = 0.f;
#pragma unroll
      for (int w = 0; w < WT; ++w) {
        const float mw = st[w * SL + D];
        v += mw == -INFINITY ? 0.f : exp2f(mw - M) * st[w * SL + (c == D ? D + 1 : c)];
      }
      if (c == D) {
        dst[D] = M;
        dst[D + 1] = v;
      } else {
        dst[c] = v;
      }
    }
  } else {
#pragma unroll
    for (int rr = 0; rr < 2; ++rr) {
      const int row = r0 + qrow + g + 8 * rr;
      if (row >= a.rows) continue;
      float* dst = a.part + (((long long)h * a.splits + sp) * a.rows + row) * (D + 4);
#pragma unroll
      for (int j = 0; j < ND; ++j)
        *reinterpret_cast<float2*>(dst + j * 8 + 2 * t4) = make_float2(o[j][2 * rr], o[j][2 * rr + 1]);
      if (t4 == 0) {
        dst[D] = m_run[rr];
        dst[D + 1] = l_run[rr];
      }
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
  // launched as a programmatic dependent of the prefix kernel (tensor-core
  // path): wait here until the prefix grid has completed and its partials are
  // visible; the launch itself overlapped the prefix kernel's tail
  asm volatile("griddepcontrol.wait;" ::: "memory");
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
  // causal over a multi-token step: position i of q_len sees the tail up to
  // its own token (the tail already holds all q_len new tokens)
  const int pos = g % a.q_len;
  const int tl = a.tail_len ? max(0, min(a.tail_len[agent] - (a.q_len - 1 - pos), a.tail_cap)) : 0;
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
  if (!tuning().attn_simt) {
    // tensor-core prefix: ~2 resident CTAs per SM (shared memory), and at
    // least `min_tiles` tiles per split (double-buffered tile loads)
    const int per_sm = env_per_sm > 0 ? env_per_sm : 2;
    // (C3: 2 -> 0.66 ms per 32-layer step, 3-4 -> 0.80, 8 -> 1.31)
    const int min_tiles = tuning().attn_min_tiles > 0 ? tuning().attn_min_tiles : 2;
    const int rt = rows <= 16 ? 16 : rows <= 32 ? 32 : 64;
    const int row_tiles = (rows + rt - 1) / rt;
    int dev = 0, sms = 148;
    cudaGetDevice(&dev);
    cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
    const long long den = (long long)kv_heads * row_tiles;
    const long long tiles = (T + TT2 - 1) / TT2;
    long long want = std::max(1LL, ((long long)per_sm * sms + den - 1) / den);
    want = std::max(1LL, std::min(want, tiles / min_tiles));
    const long long per = (tiles + want - 1) / want;
    return (int)((tiles + per - 1) / per);
  }
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
  if (!pkv::cuda_ok(cudaFuncSetAttribute(prefix_kernel2<D, RTILE>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                         (int)AT::SMEM),
                    "cudaFuncSetAttribute"))
    return PKV_ERR_CUDA;
  const int row_tiles = (a.rows + RTILE - 1) / RTILE;
  dim3 grid(a.splits, a.kv_heads, row_tiles);
  prefix_kernel2<D, RTILE><<<grid, kAttnThreads2, AT::SMEM, st>>>(a);
  if (!pkv::cuda_ok(cudaGetLastError(), "kernel launch")) return PKV_ERR_CUDA;
  combine_kernel<D><<<a.rows * a.kv_heads, 32 * kCombineWarps, 0, st>>>(a);
  return pkv::cuda_ok(cudaGetLastError(), "kernel launch") ? PKV_OK : PKV_ERR_CUDA;
}

template <int D, int WR>
int launch_mma(Args& a, cudaStream_t st) {
  using MT = mma::MmaTile<D, WR>;
  if (!pkv::cuda_ok(cudaFuncSetAttribute(prefix_mma<D, WR>, cudaFuncAttributeMaxDynamicSharedMemorySize, MT::SMEM),
                    "cudaFuncSetAttribute"))
    return PKV_ERR_CUDA;
  const int row_tiles = (a.rows + MT::RT - 1) / MT::RT;
  dim3 grid(a.splits, a.kv_heads, row_tiles);
  prefix_mma<D, WR><<<grid, 128, MT::SMEM, st>>>(a);
  if (!pkv::cuda_ok(cudaGetLastError(), "kernel launch")) return PKV_ERR_CUDA;
  // combine as a programmatic dependent launch (PDL): it may start launching
  // before the prefix grid ends and waits on griddepcontrol.wait
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = dim3(a.rows * a.kv_heads);
  cfg.blockDim = dim3(32 * kCombineWarps);
  cfg.dynamicSmemBytes = 0;
  cfg.stream = st;
  cudaLaunchAttribute attr[1];
  attr[0].id = cudaLaunchAttributeProgrammaticStreamSerialization;
  attr[0].val.programmaticStreamSerializationAllowed = 1;
  cfg.attrs = attr;
  cfg.numAttrs = 1;
  if (!pkv::cuda_ok(cudaLaunchKernelEx(&cfg, combine_kernel<D>, a), "cudaLaunchKernelEx")) return PKV_ERR_CUDA;
  return pkv::cuda_ok(cudaGetLastError(), "kernel launch") ? PKV_OK : PKV_ERR_CUDA;
}

template <int D>
int launch(Args& a, cudaStream_t st) {
  if (!tuning().attn_simt) {  // tensor-core prefix (default)
    if (a.rows <= 16) return launch_mma<D, 1>(a, st);
    if (a.rows <= 32) return launch_mma<D, 2>(a, st);
    return launch_mma<D, 4>(a, st);
  }
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
                         const int32_t* tail_len, int tail_cap, int q_len, float softmax_scale,
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
  if (q_len < 1 || group % q_len != 0) return PKV_ERR_INVALID_ARG;
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
  a.q_len = q_len;
  a.part = static_cast<float*>(workspace);
  a.out = out;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  return head_dim == 64 ? launch<64>(a, st) : launch<128>(a, st);
}

}  // extern "C"
