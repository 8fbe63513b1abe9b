// The last failing CUDA call of the calling host thread, reported by
// pkv_last_cuda_error() (include/polykv.h). Every PKV_ERR_CUDA return of the
// library goes through cuda_ok()/cuda_fail(), so a caller can tell which
// runtime / driver call failed and with what error, not just "CUDA error".
#pragma once
#include <cuda_runtime.h>

namespace pkv {

struct CudaFailure {
  int err = 0;           // cudaError_t (or a CUresult for driver calls)
  const char* what = "";  // the failing call
  bool driver = false;    // err is a CUresult
};

// thread-local record (host.cpp)
CudaFailure& last_cuda_failure();

inline bool cuda_ok(cudaError_t e, const char* what) {
  if (e == cudaSuccess) return true;
  CudaFailure& f = last_cuda_failure();
  f.err = (int)e;
  f.what = what;
  f.driver = false;
  return false;
}

inline void driver_fail(int cu_result, const char* what) {
  CudaFailure& f = last_cuda_failure();
  f.err = cu_result;
  f.what = what;
  f.driver = true;
}

}  // namespace pkv
