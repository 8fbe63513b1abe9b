// Host-side helpers of libpolykv.so.
//
// 64-bit FNV-1a (kvpool/checksum.py:13-14, 44-52) fingerprints the decoded
// tensors of an injection transcript (kvpool/pool.py:239-255). FNV-1a is
// byte-serial, so it runs on the CPU over the device->host copy.
#include <stddef.h>
#include <stdint.h>

#include "../../include/polykv.h"

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
