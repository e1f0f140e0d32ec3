// Library-level host entry points: version, error state, device info.
#include "common.cuh"

namespace nk {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

const char* get_error() { return g_err; }

}  // namespace nk

extern "C" int nk_version(void) { return 10000; /* 1.0.0 */ }

extern "C" const char* nk_last_error(void) { return nk::get_error(); }

extern "C" int nk_order_range(int* nmin, int* nmax) {
  if (nmin) *nmin = NK_MIN_ORDER;
  if (nmax) *nmax = NK_MAX_ORDER;
  return NK_OK;
}

extern "C" int nk_device_info(int* sm_count, int64_t* l2_bytes, int* cc_major, int* cc_minor) {
  int dev = 0;
  cudaError_t e = cudaGetDevice(&dev);
  cudaDeviceProp p;
  if (e == cudaSuccess) e = cudaGetDeviceProperties(&p, dev);
  if (e != cudaSuccess) {
    nk::set_error("device_info: %s", cudaGetErrorString(e));
    return NK_ERR_CUDA;
  }
  if (sm_count) *sm_count = p.multiProcessorCount;
  if (l2_bytes) *l2_bytes = p.l2CacheSize;
  if (cc_major) *cc_major = p.major;
  if (cc_minor) *cc_minor = p.minor;
  return NK_OK;
}
