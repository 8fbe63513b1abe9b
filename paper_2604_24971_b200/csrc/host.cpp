// Host-side helpers of libpolykv.so.
//
// 64-bit FNV-1a (kvpool/checksum.py:13-14, 44-52) fingerprints the decoded
// tensors of an injection transcript (kvpool/pool.py:239-255). FNV-1a is
// byte-serial, so it runs on the CPU over the device->host copy.
#include <stddef.h>
#include <stdint.h>

#include <atomic>
#include <cstdio>
#include <cstdlib>
#include <cstring>
#include <mutex>

#include "../../include/polykv.h"
#include "diag.h"
#include "tuning.h"

namespace pkv {
namespace {
Tuning read_env() {
  Tuning t;
  if (const char* e = std::getenv("PKV_CODEC_PATH")) t.codec_warp = std::strcmp(e, "warp") == 0;
  if (const char* e = std::getenv("PKV_DBG_ENC")) t.dbg_enc = std::atoi(e);
  if (const char* e = std::getenv("PKV_KEY_LAG")) t.key_lag = std::atoi(e);
  if (const char* e = std::getenv("PKV_ABSMAX_ROLE")) t.abs_on_values = std::strcmp(e, "values") == 0;
  if (const char* e = std::getenv("PKV_ENC_ROLES")) t.enc_co = std::strcmp(e, "co") == 0;
  if (const char* e = std::getenv("PKV_KEY_SM_FRACTION")) t.key_sm_fraction = std::atof(e);
  if (const char* e = std::getenv("PKV_DEC_KEY_FRACTION")) t.dec_key_fraction = std::atof(e);
  if (const char* e = std::getenv("PKV_ATTN_CTAS_PER_SM")) t.attn_ctas_per_sm = std::atoi(e);
  if (const char* e = std::getenv("PKV_ATTN_PATH")) t.attn_simt = std::strcmp(e, "simt") == 0;
  if (const char* e = std::getenv("PKV_ATTN_MIN_TILES")) t.attn_min_tiles = std::atoi(e);
  return t;
}
std::mutex g_reload;
std::atomic<const Tuning*> g_tuning{nullptr};
}  // namespace

const Tuning& tuning() {
  const Tuning* t = g_tuning.load(std::memory_order_acquire);
  if (t) return *t;
  reload_tuning();
  return *g_tuning.load(std::memory_order_acquire);
}

void reload_tuning() {
  std::lock_guard<std::mutex> lk(g_reload);
  // snapshots are immutable and never freed: a launch that read the previous
  // one on another thread keeps a valid reference (reloads are rare)
  g_tuning.store(new Tuning(read_env()), std::memory_order_release);
}
}  // namespace pkv

extern "C" int pkv_reload_tuning(void) {
  pkv::reload_tuning();
  return PKV_OK;
}

namespace pkv {
CudaFailure& last_cuda_failure() {
  static thread_local CudaFailure f;
  return f;
}
}  // namespace pkv

extern "C" const char* pkv_last_cuda_error(void) {
  static thread_local char buf[256];
  const pkv::CudaFailure& f = pkv::last_cuda_failure();
  if (f.err == 0) return "";
  if (f.driver)
    std::snprintf(buf, sizeof(buf), "%s: CUresult %d", f.what, f.err);
  else
    std::snprintf(buf, sizeof(buf), "%s: %s (%s)", f.what, cudaGetErrorName((cudaError_t)f.err),
                  cudaGetErrorString((cudaError_t)f.err));
  return buf;
}

namespace {
constexpr uint64_t kFnvOffset = 0xcbf29ce484222325ull;
constexpr uint64_t kFnvPrime = 0x100000001b3ull;
}  // namespace

extern "C" uint64_t pkv_fnv1a64(const void* data_host, size_t n) {
  const unsigned char* p = static_cast<const unsigned char*>(data_host);
  uint64_t h = kFnvOffset;
  for (size_t i = 0; i < n; ++i) {
    h ^= p[i];
    h *= kFnvPrime;
  }
  return h;
}

// bf16 value b has the f32 image (b << 16): little-endian bytes 0, 0, lo, hi.
extern "C" uint64_t pkv_fnv1a64_bf16_as_f32(const uint16_t* data_host, size_t count) {
  uint64_t h = kFnvOffset;
  for (size_t i = 0; i < count; ++i) {
    const uint16_t b = data_host[i];
    h *= kFnvPrime;  // byte 0 == 0: h ^= 0
    h *= kFnvPrime;  // byte 1 == 0
    h ^= (uint64_t)(b & 0xffu);
    h *= kFnvPrime;
    h ^= (uint64_t)(b >> 8);
    h *= kFnvPrime;
  }
  return h;
}
