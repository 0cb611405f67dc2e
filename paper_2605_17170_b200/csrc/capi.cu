// Library-level C ABI: version string and per-thread error message.
#include <cstring>

#include <cuda_runtime.h>

#include "launch.h"

namespace kvmix {
static thread_local char g_err[512] = "";
void set_error(const char* msg) {
  strncpy(g_err, msg, sizeof(g_err) - 1);
  g_err[sizeof(g_err) - 1] = 0;
}
}  // namespace kvmix

extern "C" const char* kvmix_version(void) { return "kvmix_b200 0.1.0 sm_100a"; }
extern "C" const char* kvmix_last_error(void) { return kvmix::g_err; }
extern "C" int kvmix_stream_sync(void* stream) {
  const cudaError_t e = cudaStreamSynchronize((cudaStream_t)stream);
  if (e != cudaSuccess) {
    kvmix::set_error(cudaGetErrorString(e));
    return KVMIX_ECUDA;
  }
  return KVMIX_OK;
}
