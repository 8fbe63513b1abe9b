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
//   * the prefix is split into 128-token tiles, one CTA per (kv head, tile);
//     a CTA converts its K tile (int8 codes * scale, exactly the reference
//     dequant) to f32 in shared memory and its V tile to the *rotated*
//     domain y = table[code] * rms (valuequant.py:232-234), then computes
//     scores, a tile-local softmax (max, sum) and sum_t p_t * y_t;
//   * a combine kernel merges the tiles with log-sum-exp weights, applies
//     ONE inverse FWHT / sqrt(d) (and the sign diagonal) per output vector —
//     valid because H is linear — and folds in the agent's private bf16
//     tail (tokens appended after the shared prefix).
#include <algorithm>
#include <cmath>
#include <cstring>

#include "../../include/polykv.h"
#include "pkv_common.cuh"

namespace pkv {
namespace attn {

constexpr int TT = 128;        // prefix tokens per CTA
constexpr int RT = 64;         // query rows per row tile (8 warps x 8 rows)
constexpr int kAttnThreads = 256;
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
  float* part;     // [kv_heads][splits][rows][D + 2]
  void* out;
};

__device__ __forceinline__ float ldq(const Args& a, long long i) {
  return a.q_dtype == PKV_F32 ? static_cast<const float*>(a.q)[i]
                              : __bfloat162float(static_cast<const __nv_bfloat16*>(a.q)[i]);
}

// smem: Kt[D][TT] f32 | Y[TT][D] f32 | Q[RT][D] f32 | P[RT][TT] f32
template <int D>
__global__ void __launch_bounds__(kAttnThreads, 1) prefix_kernel(const __grid_constant__ Args a) {
  extern __shared__ __align__(16) float sm[];
  float* Kt = sm;
  float* Y = Kt + D * TT;
  float* Q = Y + TT * D;
  float* P = Q + RT * D;
  __shared__ float cent[8];

  const int h = blockIdx.y;
  const int sidx = blockIdx.x;
  const long long t0 = (long long)sidx * TT;
  const int nt = (int)min((long long)TT, a.T - t0);
  const int tid = threadIdx.x, warp = tid >> 5, lane = tid & 31;
  if (tid < 8) cent[tid] = a.cent32[tid];
  __syncthreads();

  // ---- K tile -> f32, transposed (Kt[d][t]) ----
  {
    const int t = tid % TT;
    const long long tok = t0 + t;
    for (int d0 = (tid / TT) * 16; d0 < D; d0 += (kAttnThreads / TT) * 16) {
      float kv[16];
      if (t < nt) {
        const long long base = ((long long)h * a.T + tok) * D + d0;
        const uint4 w = *reinterpret_cast<const uint4*>(a.k_codes + base);
        const uint32_t ww[4] = {w.x, w.y, w.z, w.w};
#pragma unroll
        for (int j = 0; j < 16; ++j) {
          const int c = (int)(int8_t)((ww[j >> 2] >> (8 * (j & 3))) & 0xffu);
          const float s = a.k_mode == PKV_K_TENSOR ? __ldg(a.k_scale)
                                                   : __half2float(a.k_bscale[(base + j) >> 5]);
          kv[j] = (float)c * s;  // dequantize_k: code * scale in f32
        }
      } else {
#pragma unroll
        for (int j = 0; j < 16; ++j) kv[j] = 0.f;
      }
#pragma unroll
      for (int j = 0; j < 16; ++j) Kt[(d0 + j) * TT + t] = kv[j];
    }
  }
  // ---- V tile -> rotated-domain values Y[t][d] = table[code] * rms ----
  {
    constexpr int W = D / 8;
    for (int i = tid; i < TT * W; i += kAttnThreads) {
      const int t = i / W, w = i % W;
      float y[8];
      if (t < nt) {
        const long long v = (long long)h * a.T + t0 + t;
        const uint8_t* p = a.v_packed + v * (3 * D / 8) + 3 * w;
        const uint32_t word = (uint32_t)p[0] | ((uint32_t)p[1] << 8) | ((uint32_t)p[2] << 16);
        const float rms = a.v_scales[v];
#pragma unroll
        for (int e = 0; e < 8; ++e) y[e] = cent[(word >> (3 * e)) & 7u] * rms;
      } else {
#pragma unroll
        for (int e = 0; e < 8; ++e) y[e] = 0.f;
      }
      float4* dst = reinterpret_cast<float4*>(Y + t * D + 8 * w);
      dst[0] = make_float4(y[0], y[1], y[2], y[3]);
      dst[1] = make_float4(y[4], y[5], y[6], y[7]);
    }
  }

  constexpr int DPL = D / 32;  // output columns per lane in the PV product
  for (int r0 = 0; r0 < a.rows; r0 += RT) {
    __syncthreads();
    // ---- Q row tile (pre-scaled by softmax_scale * log2 e) ----
    for (int i = tid; i < RT * D; i += kAttnThreads) {
      const int r = i / D, d = i % D;
      const int row = r0 + r;
      float qv = 0.f;
      if (row < a.rows) {
        const int agent = row / a.group, g = row % a.group;
        qv = ldq(a, (((long long)agent * a.kv_heads + h) * a.group + g) * D + d) * a.qscale;
      }
      Q[r * D + d] = qv;
    }
    __syncthreads();

    // ---- scores: warp -> 8 rows, lane -> 4 tokens ----
    float s[8][4];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < 4; ++j) s[i][j] = 0.f;
    const float* qrow = Q + (warp * 8) * D;
#pragma unroll 2
    for (int d = 0; d < D; d += 4) {
      float4 kk[4];
#pragma unroll
      for (int dd = 0; dd < 4; ++dd) kk[dd] = *reinterpret_cast<const float4*>(Kt + (d + dd) * TT + 4 * lane);
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 qq = *reinterpret_cast<const float4*>(qrow + i * D + d);
        s[i][0] = fmaf(qq.x, kk[0].x, s[i][0]); s[i][1] = fmaf(qq.x, kk[0].y, s[i][1]);
        s[i][2] = fmaf(qq.x, kk[0].z, s[i][2]); s[i][3] = fmaf(qq.x, kk[0].w, s[i][3]);
        s[i][0] = fmaf(qq.y, kk[1].x, s[i][0]); s[i][1] = fmaf(qq.y, kk[1].y, s[i][1]);
        s[i][2] = fmaf(qq.y, kk[1].z, s[i][2]); s[i][3] = fmaf(qq.y, kk[1].w, s[i][3]);
        s[i][0] = fmaf(qq.z, kk[2].x, s[i][0]); s[i][1] = fmaf(qq.z, kk[2].y, s[i][1]);
        s[i][2] = fmaf(qq.z, kk[2].z, s[i][2]); s[i][3] = fmaf(qq.z, kk[2].w, s[i][3]);
        s[i][0] = fmaf(qq.w, kk[3].x, s[i][0]); s[i][1] = fmaf(qq.w, kk[3].y, s[i][1]);
        s[i][2] = fmaf(qq.w, kk[3].z, s[i][2]); s[i][3] = fmaf(qq.w, kk[3].w, s[i][3]);
      }
    }
    // ---- tile softmax: row max, p = 2^(s - m), row sum ----
    float mrow[8], lrow[8];
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      float m = -INFINITY;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        if (4 * lane + j >= nt) s[i][j] = -INFINITY;
        m = fmaxf(m, s[i][j]);
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) m = fmaxf(m, __shfl_xor_sync(0xffffffffu, m, o));
      float l = 0.f;
#pragma unroll
      for (int j = 0; j < 4; ++j) {
        const float p = exp2f(s[i][j] - m);
        s[i][j] = p;
        l += p;
      }
#pragma unroll
      for (int o = 16; o > 0; o >>= 1) l += __shfl_xor_sync(0xffffffffu, l, o);
      mrow[i] = m;
      lrow[i] = l;
      *reinterpret_cast<float4*>(P + (warp * 8 + i) * TT + 4 * lane) =
          make_float4(s[i][0], s[i][1], s[i][2], s[i][3]);
    }
    __syncwarp();  // each warp only reads back its own P rows

    // ---- PV in the rotated domain: warp -> 8 rows, lane -> DPL columns ----
    float acc[8][DPL];
#pragma unroll
    for (int i = 0; i < 8; ++i)
#pragma unroll
      for (int j = 0; j < DPL; ++j) acc[i][j] = 0.f;
    const float* prow = P + (warp * 8) * TT;
    for (int t = 0; t < nt; t += 4) {
      float yv[4][DPL];
#pragma unroll
      for (int tt = 0; tt < 4; ++tt)
#pragma unroll
        for (int j = 0; j < DPL; ++j) yv[tt][j] = Y[(t + tt) * D + lane * DPL + j];
#pragma unroll
      for (int i = 0; i < 8; ++i) {
        const float4 pp = *reinterpret_cast<const float4*>(prow + i * TT + t);
#pragma unroll
        for (int j = 0; j < DPL; ++j) {
          acc[i][j] = fmaf(pp.x, yv[0][j], acc[i][j]);
          acc[i][j] = fmaf(pp.y, yv[1][j], acc[i][j]);
          acc[i][j] = fmaf(pp.z, yv[2][j], acc[i][j]);
          acc[i][j] = fmaf(pp.w, yv[3][j], acc[i][j]);
        }
      }
    }
    // ---- partial: [h][split][row][0..D) acc, D: m, D+1: l ----
#pragma unroll
    for (int i = 0; i < 8; ++i) {
      const int row = r0 + warp * 8 + i;
      if (row >= a.rows) continue;
      float* dst = a.part + (((long long)h * a.splits + sidx) * a.rows + row) * (D + 2);
#pragma unroll
      for (int j = 0; j < DPL; ++j) dst[lane * DPL + j] = acc[i][j];
      if (lane == 0) {
        dst[D] = mrow[i];
        dst[D + 1] = lrow[i];
      }
    }
  }
}

// One warp per (row, kv head): merge tiles, inverse-rotate, add the tail.
template <int D>
__global__ void combine_kernel(const __grid_constant__ Args a) {
  constexpr int EPL = D / 32;  // coordinates per lane: lane holds [EPL*lane, EPL*lane+EPL)
  const int warp_global = (blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (warp_global >= a.rows * a.kv_heads) return;
  const int row = warp_global / a.kv_heads;
  const int h = warp_global % a.kv_heads;
  const int agent = row / a.group, g = row % a.group;

  float M = -INFINITY;
  for (int sidx = 0; sidx < a.splits; ++sidx) {
    const float* src = a.part + (((long long)h * a.splits + sidx) * a.rows + row) * (D + 2);
    M = fmaxf(M, src[D]);
  }
  float L = 0.f;
  float acc[EPL];
#pragma unroll
  for (int j = 0; j < EPL; ++j) acc[j] = 0.f;
  for (int sidx = 0; sidx < a.splits; ++sidx) {
    const float* src = a.part + (((long long)h * a.splits + sidx) * a.rows + row) * (D + 2);
    const float w = exp2f(src[D] - M);
    L += w * src[D + 1];
#pragma unroll
    for (int j = 0; j < EPL; ++j) acc[j] = fmaf(w, src[EPL * lane + j], acc[j]);
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
  const int tl = a.tail_len ? a.tail_len[agent] : 0;
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

template <int D>
size_t smem_bytes() {
  return sizeof(float) * (size_t)(D * TT + TT * D + RT * D + RT * TT);
}

template <int D>
int launch(Args& a, cudaStream_t st) {
  const size_t smem = smem_bytes<D>();
  if (cudaFuncSetAttribute(prefix_kernel<D>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                           (int)smem) != cudaSuccess)
    return PKV_ERR_CUDA;
  dim3 grid(a.splits, a.kv_heads);
  prefix_kernel<D><<<grid, kAttnThreads, smem, st>>>(a);
  if (cudaGetLastError() != cudaSuccess) return PKV_ERR_CUDA;
  const int warps = a.rows * a.kv_heads;
  combine_kernel<D><<<(warps + 7) / 8, 256, 0, st>>>(a);
  return cudaGetLastError() == cudaSuccess ? PKV_OK : PKV_ERR_CUDA;
}

}  // namespace attn
}  // namespace pkv

extern "C" {

size_t pkv_attention_workspace_bytes(int num_rows, int kv_heads, int group, int head_dim,
                                     int64_t seq_len) {
  if (num_rows < 1 || kv_heads < 1 || group < 1 || head_dim < 1 || seq_len < 1) return 0;
  const long long splits = (seq_len + pkv::attn::TT - 1) / pkv::attn::TT;
  return sizeof(float) * (size_t)kv_heads * (size_t)splits * (size_t)num_rows * (size_t)group *
         (size_t)(head_dim + 2);
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
  a.splits = (int)((seq_len + TT - 1) / TT);
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
