// Internal interface between the C ABI (codec.cu) and the TMA-streamed
// kernels (stream_codec.cu). Not part of include/polykv.h.
#pragma once

#include <cuda_runtime.h>
#include <stdint.h>

#include "codec_common.cuh"

namespace pkv {
namespace stream {

struct EncodeRequest {
  int num_layers;  // <= kMaxLayers
  long long num_vectors;
  int head_dim, in_dtype, k_mode;
  const void* const* k_in;  // null: no keys
  const void* const* v_in;  // null: no values
  int8_t* const* k_codes;
  float* const* k_scale;
  uint16_t* const* k_bscale;
  uint8_t* const* v_packed;
  float* const* v_scales;
  Codebook3 cb;
  uint32_t sign_bits[8];
  bool sign;
  uint32_t* status;
  uint32_t* replay_count;
  const uint32_t* k_max_ext;  // per-tensor keys: external max|K| bits per layer (null: own absmax pass)
  void* ws;  // workspace_bytes(num_layers, num_vectors, head_dim)
  size_t ws_bytes;
};

struct DecodeRequest {
  int num_layers;
  long long num_vectors;
  int head_dim, out_dtype, k_mode;
  const int8_t* const* k_codes;  // null: no keys
  const float* const* k_scale;
  const uint16_t* const* k_bscale;
  void* const* k_out;
  const uint8_t* const* v_packed;  // null: no values
  const float* const* v_scales;
  void* const* v_out;
  float cent32[8];
  uint32_t sign_bits[8];
  bool sign;
};

bool head_dim_streamable(int d);
// device scratch the streamed encoder needs for one launch of <= kMaxLayers layers
size_t workspace_bytes(int num_layers, long long num_vectors, int head_dim);
// PKV_OK, or a PKV_ERR_* code; PKV_ERR_ALIGNMENT / PKV_ERR_UNSUPPORTED_HEAD_DIM
// mean "use the warp-granular kernels" and leave the stream untouched.
int encode(const EncodeRequest& r, cudaStream_t st);
int decode(const DecodeRequest& r, cudaStream_t st);

}  // namespace stream
}  // namespace pkv
