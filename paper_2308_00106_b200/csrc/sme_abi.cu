// sme_abi.cu — error reporting, version and device queries of the C-ABI.
#include <cstdarg>
#include <cstdio>

#include "common.cuh"

namespace sme {

static thread_local char g_err[1024] = "";

void set_error(const char* fmt, ...) {
  va_list ap;
  va_start(ap, fmt);
  vsnprintf(g_err, sizeof(g_err), fmt, ap);
  va_end(ap);
}

int sm_count() {
  // cached per device (at most 64 devices per process)
  static int cache[64] = {0};
  int dev = 0;
  if (cudaGetDevice(&dev) != cudaSuccess || dev < 0 || dev >= 64) return 148;
  if (cache[dev] == 0) {
    int n = 0;
    if (cudaDeviceGetAttribute(&n, cudaDevAttrMultiProcessorCount, dev) != cudaSuccess || n <= 0)
      n = 148;
    cache[dev] = n;
  }
  return cache[dev];
}

}  // namespace sme

SME_API const char* sme_last_error(void) { return sme::g_err; }

SME_API int sme_version(void) { return 1; }

SME_API int sme_device_sm_count(void) { return sme::sm_count(); }
