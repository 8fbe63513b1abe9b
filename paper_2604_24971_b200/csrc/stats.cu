// Build statistics of a pool (LayerStats, kvpool/pool.py:274-288 and
// metrics.py:166-222) as one fused, deterministic error reduction (sm_100a).
//
// Per layer: k_err = dequant(K) - K and v_err = dequant(V) - V in f64 (the
// reference's float64 arithmetic: the difference of two f32 values is exact
// in f64), reduced to  sum k_err^2, max |k_err|, sum v_err^2, sum V^2.
// The dequantised tensors come from pkv_decode at 32 bits (bit-identical to
// the reference's dequantize_k / dequantize_v). One read of the four tensors,
// f64 accumulation, a fixed reduction tree (run-to-run identical results):
// block partials land in the workspace, one warp per layer folds them in
// order. HBM-bound: 2 x (in + 4) bytes per element and per tensor.
#include <algorithm>

#include "../../include/polykv.h"
#include "diag.h"
#include "pkv_common.cuh"

namespace pkv {
namespace {

constexpr int kStatThreads = 256;

struct StatArgs {
  const void* k_in[kMaxLayers];
  const void* v_in[kMaxLayers];
  const float* k_dec[kMaxLayers];
  const float* v_dec[kMaxLayers];
  long long count;  // elements per tensor
  int bf16;
  int vec;          // 16-byte aligned tensors and count % 8 == 0
  int blocks;       // blocks per layer
  double* part;     // [L][blocks][4]
  double* out;      // [L][4]
};

__device__ __forceinline__ void load_in8(const void* base, long long e, bool bf16, float (&x)[8]) {
  if (bf16) load8(static_cast<const __nv_bfloat16*>(base) + e, x);
  else load8(static_cast<const float*>(base) + e, x);
}
__device__ __forceinline__ float load_in1(const void* base, long long e, bool bf16) {
  return bf16 ? load1(static_cast<const __nv_bfloat16*>(base) + e) : load1(static_cast<const float*>(base) + e);
}

__global__ void __launch_bounds__(kStatThreads) stats_partial(const __grid_constant__ StatArgs a) {
  const int layer = blockIdx.y;
  double sk = 0.0, kmax = 0.0, sv = 0.0, sp = 0.0;
  const long long stride = (long long)a.blocks * kStatThreads;
  const long long tid = (long long)blockIdx.x * kStatThreads + threadIdx.x;
  const float* kd = a.k_dec[layer];
  const float* vd = a.v_dec[layer];
  if (a.vec) {
    for (long long u = tid; u * 8 < a.count; u += stride) {
      const long long e = u * 8;
      float ki[8], vi[8], kq[8], vq[8];
      load_in8(a.k_in[layer], e, a.bf16, ki);
      load_in8(a.v_in[layer], e, a.bf16, vi);
      load8(kd + e, kq);
      load8(vd + e, vq);
#pragma unroll
      for (int j = 0; j < 8; ++j) {
        const double dk = (double)kq[j] - (double)ki[j];
        const double dv = (double)vq[j] - (double)vi[j];
        sk = __dadd_rn(sk, __dmul_rn(dk, dk));
        kmax = fmax(kmax, fabs(dk));
        sv = __dadd_rn(sv, __dmul_rn(dv, dv));
        sp = __dadd_rn(sp, __dmul_rn((double)vi[j], (double)vi[j]));
      }
    }
  } else {
    for (long long e = tid; e < a.count; e += stride) {
      const double ki = load_in1(a.k_in[layer], e, a.bf16), vi = load_in1(a.v_in[layer], e, a.bf16);
      const double dk = (double)kd[e] - ki, dv = (double)vd[e] - vi;
      sk = __dadd_rn(sk, __dmul_rn(dk, dk));
      kmax = fmax(kmax, fabs(dk));
      sv = __dadd_rn(sv, __dmul_rn(dv, dv));
      sp = __dadd_rn(sp, __dmul_rn(vi, vi));
    }
  }
  // fixed-order block reduction
  __shared__ double red[4][kStatThreads];
  red[0][threadIdx.x] = sk;
  red[1][threadIdx.x] = kmax;
  red[2][threadIdx.x] = sv;
  red[3][threadIdx.x] = sp;
  __syncthreads();
  for (int h = kStatThreads / 2; h > 0; h >>= 1) {
    if (threadIdx.x < h) {
      red[0][threadIdx.x] = __dadd_rn(red[0][threadIdx.x], red[0][threadIdx.x + h]);
      red[1][threadIdx.x] = fmax(red[1][threadIdx.x], red[1][threadIdx.x + h]);
      red[2][threadIdx.x] = __dadd_rn(red[2][threadIdx.x], red[2][threadIdx.x + h]);
      red[3][threadIdx.x] = __dadd_rn(red[3][threadIdx.x], red[3][threadIdx.x + h]);
    }
    __syncthreads();
  }
  if (threadIdx.x < 4) a.part[((long long)layer * a.blocks + blockIdx.x) * 4 + threadIdx.x] = red[threadIdx.x][0];
}

__global__ void stats_final(const __grid_constant__ StatArgs a) {
  const int layer = blockIdx.x;
  if (threadIdx.x != 0) return;
  double s[4] = {0.0, 0.0, 0.0, 0.0};
  for (int b = 0; b < a.blocks; ++b) {
    const double* p = a.part + ((long long)layer * a.blocks + b) * 4;
    s[0] = __dadd_rn(s[0], p[0]);
    s[1] = fmax(s[1], p[1]);
    s[2] = __dadd_rn(s[2], p[2]);
    s[3] = __dadd_rn(s[3], p[3]);
  }
  for (int i = 0; i < 4; ++i) a.out[layer * 4 + i] = s[i];
}

int blocks_for(long long count, int layers) {
  int sms = 148, dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  const long long want = (count / 8 + kStatThreads - 1) / kStatThreads;
  return (int)std::max(1LL, std::min(want, (long long)std::max(1, 8 * sms / std::max(1, layers))));
}

}  // namespace
}  // namespace pkv

extern "C" size_t pkv_layer_stats_workspace_bytes(int num_layers, int64_t count) {
  const int L = std::min(std::max(num_layers, 1), pkv::kMaxLayers);
  return (size_t)L * pkv::blocks_for(count, L) * 4 * sizeof(double);
}

extern "C" int pkv_layer_stats(int num_layers, int64_t count, int in_dtype, const void* const* k_in,
                               const void* const* v_in, const float* const* k_dec, const float* const* v_dec,
                               double* out, void* workspace, size_t workspace_bytes, void* stream) {
  using namespace pkv;
  if (num_layers < 0 || count < 0 || !out) return PKV_ERR_INVALID_ARG;
  if (in_dtype != PKV_F32 && in_dtype != PKV_BF16) return PKV_ERR_INVALID_ARG;
  if (num_layers == 0) return PKV_OK;
  if (!workspace || workspace_bytes < pkv_layer_stats_workspace_bytes(num_layers, count)) return PKV_ERR_WORKSPACE;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  const int eb = in_dtype == PKV_F32 ? 4 : 2;
  for (int l0 = 0; l0 < num_layers; l0 += kMaxLayers) {
    const int L = std::min(num_layers - l0, kMaxLayers);
    StatArgs a;
    a.count = count;
    a.bf16 = eb == 2;
    a.vec = count % 8 == 0;
    a.blocks = blocks_for(count, L);
    a.part = static_cast<double*>(workspace);
    a.out = out + 4 * l0;
    for (int l = 0; l < L; ++l) {
      a.k_in[l] = k_in[l0 + l];
      a.v_in[l] = v_in[l0 + l];
      a.k_dec[l] = k_dec[l0 + l];
      a.v_dec[l] = v_dec[l0 + l];
      if (!a.k_in[l] || !a.v_in[l] || !a.k_dec[l] || !a.v_dec[l]) return PKV_ERR_INVALID_ARG;
      for (const void* p : {a.k_in[l], a.v_in[l], (const void*)a.k_dec[l], (const void*)a.v_dec[l]})
        if (reinterpret_cast<uintptr_t>(p) % 16) a.vec = 0;
    }
    if (count == 0) {
      if (!pkv::cuda_ok(cudaMemsetAsync(a.out, 0, sizeof(double) * 4 * L, st), "cudaMemsetAsync")) return PKV_ERR_CUDA;
      continue;
    }
    stats_partial<<<dim3(a.blocks, L), kStatThreads, 0, st>>>(a);
    stats_final<<<L, 32, 0, st>>>(a);
    if (!pkv::cuda_ok(cudaGetLastError(), "kernel launch")) return PKV_ERR_CUDA;
  }
  return PKV_OK;
}
