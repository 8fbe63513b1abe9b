// Per-layer max|K| for the head-sharded pool (sm_100a).
//
// kvpool's per-tensor key scale is f32(max|K| / 127) over the WHOLE layer
// (keyquant.py:55-60). When a layer's KV heads are split across GPUs
// (parallel.build_pool_head_sharded) every rank computes the
// max over its heads here, the ranks MAX-reduce the 32-bit patterns (|x| bit
// patterns order like the floats, NaN above +inf), and pkv_encode takes the
// reduced maxima through its k_layer_max argument, so each rank's key codes
// equal the single-GPU build's codes for its heads.
//
// HBM-bound streaming reduction: 16-byte loads, a grid of whole waves over
// the 148 SMs, one atomicMax per CTA and layer.
#include <algorithm>

#include "../../include/polykv.h"
#include "diag.h"
#include "pkv_common.cuh"

namespace pkv {
namespace {

constexpr int kAbsThreads = 512;

__device__ __forceinline__ uint32_t absmax_u4(uint4 w, bool bf16) {
  if (bf16) {
    uint32_t m = __vmaxu2(__vmaxu2(w.x & 0x7fff7fffu, w.y & 0x7fff7fffu), __vmaxu2(w.z & 0x7fff7fffu, w.w & 0x7fff7fffu));
    m = max(m & 0xffffu, m >> 16);
    return m << 16;  // bf16 -> f32 bit pattern
  }
  return max(max(w.x & 0x7fffffffu, w.y & 0x7fffffffu), max(w.z & 0x7fffffffu, w.w & 0x7fffffffu));
}

struct AbsArgs {
  const void* k_in[kMaxLayers];
  long long count;  // elements per layer
  int bf16;
  int vec;  // every layer 16-byte aligned and a whole number of 16-byte units
  uint32_t* out;
};

__global__ void __launch_bounds__(kAbsThreads) absmax_kernel(const __grid_constant__ AbsArgs a) {
  const int layer = blockIdx.y;
  uint32_t m = 0;
  if (a.vec) {
    const uint4* p = static_cast<const uint4*>(a.k_in[layer]);
    const long long units = a.count * (a.bf16 ? 2 : 4) / 16;
    const long long stride = (long long)gridDim.x * kAbsThreads;
    long long i = (long long)blockIdx.x * kAbsThreads + threadIdx.x;
    // four loads in flight per thread
    for (; i + 3 * stride < units; i += 4 * stride) {
      const uint4 w0 = ld_stream_u4(p + i), w1 = ld_stream_u4(p + i + stride);
      const uint4 w2 = ld_stream_u4(p + i + 2 * stride), w3 = ld_stream_u4(p + i + 3 * stride);
      m = max(max(m, max(absmax_u4(w0, a.bf16), absmax_u4(w1, a.bf16))),
              max(absmax_u4(w2, a.bf16), absmax_u4(w3, a.bf16)));
    }
    for (; i < units; i += stride) m = max(m, absmax_u4(ld_stream_u4(p + i), a.bf16));
  } else {
    for (long long i = (long long)blockIdx.x * kAbsThreads + threadIdx.x; i < a.count;
         i += (long long)gridDim.x * kAbsThreads) {
      const float x = a.bf16 ? load1(static_cast<const __nv_bfloat16*>(a.k_in[layer]) + i)
                             : load1(static_cast<const float*>(a.k_in[layer]) + i);
      m = max(m, __float_as_uint(x) & 0x7fffffffu);
    }
  }
#pragma unroll
  for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
  __shared__ uint32_t wm[kAbsThreads / 32];
  if ((threadIdx.x & 31) == 0) wm[threadIdx.x >> 5] = m;
  __syncthreads();
  if (threadIdx.x < 32) {
    m = threadIdx.x < kAbsThreads / 32 ? wm[threadIdx.x] : 0u;
#pragma unroll
    for (int o = 16; o > 0; o >>= 1) m = max(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (threadIdx.x == 0 && m) atomicMax(a.out + layer, m);
  }
}

}  // namespace
}  // namespace pkv

extern "C" int pkv_k_absmax(int num_layers, int64_t count, int in_dtype, const void* const* k_in,
                            uint32_t* max_bits, void* stream) {
  using namespace pkv;
  if (num_layers < 0 || count < 0 || !max_bits) return PKV_ERR_INVALID_ARG;
  if (in_dtype != PKV_F32 && in_dtype != PKV_BF16) return PKV_ERR_INVALID_ARG;
  cudaStream_t st = static_cast<cudaStream_t>(stream);
  if (num_layers == 0) return PKV_OK;
  if (!pkv::cuda_ok(cudaMemsetAsync(max_bits, 0, sizeof(uint32_t) * num_layers, st), "cudaMemsetAsync")) return PKV_ERR_CUDA;
  if (count == 0) return PKV_OK;
  const int eb = in_dtype == PKV_F32 ? 4 : 2;
  int sms = 148;
  int dev = 0;
  if (cudaGetDevice(&dev) == cudaSuccess) cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, dev);
  for (int l0 = 0; l0 < num_layers; l0 += kMaxLayers) {
    const int L = std::min(num_layers - l0, kMaxLayers);
    AbsArgs a;
    a.count = count;
    a.bf16 = eb == 2;
    a.out = max_bits + l0;
    a.vec = (count * eb) % 16 == 0;
    for (int l = 0; l < L; ++l) {
      a.k_in[l] = k_in[l0 + l];
      if (!a.k_in[l]) return PKV_ERR_INVALID_ARG;
      if (reinterpret_cast<uintptr_t>(a.k_in[l]) % 16) a.vec = 0;
    }
    // ~4 resident 512-thread CTAs per SM in total, spread over the layers
    const long long units = a.vec ? count * eb / 16 : count;
    const long long want = (units + 4LL * kAbsThreads - 1) / (4LL * kAbsThreads);
    const int per_layer = (int)std::max(1LL, std::min(want, (long long)std::max(1, 4 * sms / L)));
    absmax_kernel<<<dim3(per_layer, L), kAbsThreads, 0, st>>>(a);
    if (!pkv::cuda_ok(cudaGetLastError(), "kernel launch")) return PKV_ERR_CUDA;
  }
  return PKV_OK;
}
