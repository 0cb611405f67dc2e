// Host-side status/error helpers shared by the C-ABI entry points.
#pragma once
#include <cstdio>
#include <cuda_runtime.h>

#include "../../include/kvmix_b200.h"

namespace kvmix {
// thread-local message of the last failure (kvmix_last_error)
void set_error(const char* msg);
inline int fail(int code, const char* msg) {
  set_error(msg);
  return code;
}
inline int check_launch(const char* what) {
  cudaError_t e = cudaGetLastError();
  if (e != cudaSuccess) {
    char buf[256];
    snprintf(buf, sizeof(buf), "%s: %s", what, cudaGetErrorString(e));
    set_error(buf);
    return KVMIX_ECUDA;
  }
  return KVMIX_OK;
}
}  // namespace kvmix
