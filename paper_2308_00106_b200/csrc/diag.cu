// diag.cu — microbenchmarks that set the roofline of the gather-bound SpMV.
//
// A CSR SpMV with randomly permuted columns performs one random 8-byte x
// gather per nonzero.  Each gather is (at least) one 32-byte L2 sector access,
// so beside the HBM byte roofline the kernel is bounded by the device's random
// sector-gather rate.  k_diag_gather measures that rate for an x of a given
// size: every thread gathers `per_thread` pseudo-random elements (index from a
// hash, no index stream) and writes one sum.
#include "common.cuh"

namespace sme {

__device__ __forceinline__ uint32_t hash32(uint32_t a) {
  a ^= a >> 16; a *= 0x7feb352dU; a ^= a >> 15; a *= 0x846ca68bU; a ^= a >> 16;
  return a;
}

template <int UNROLL>
__global__ void __launch_bounds__(256) k_diag_gather(const double* __restrict__ x, uint32_t n, int per_thread,
                                                     int keep, double* __restrict__ out) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint64_t pol = keep ? policy_evict_last() : policy_evict_first();
  double acc = 0.0;
  for (int i = 0; i < per_thread; i += UNROLL) {
    double v[UNROLL];
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) {
      const uint32_t h = hash32(tid * 0x9E3779B1u + (uint32_t)(i + u) * 0x85EBCA77u);
      const uint32_t idx = (uint32_t)(((uint64_t)h * n) >> 32);
      v[u] = ld_keep(x + idx, pol);
    }
#pragma unroll
    for (int u = 0; u < UNROLL; ++u) acc += v[u];
  }
  out[tid] = acc;
}

}  // namespace sme

using namespace sme;

// Launches blocks x 256 threads, each gathering per_thread elements of x[n].
SME_API int sme_diag_gather(const double* x, int64_t n, int32_t blocks, int32_t per_thread, int32_t keep,
                            double* out, sme_stream_t stream) {
  SME_REQUIRE(n >= 1 && n < (1ll << 32), "n out of range");
  SME_REQUIRE(per_thread % 8 == 0 && blocks >= 1, "per_thread must be a multiple of 8");
  k_diag_gather<8><<<blocks, 256, 0, as_stream(stream)>>>(x, (uint32_t)n, per_thread, keep, out);
  SME_CHECK_LAUNCH("k_diag_gather");
  return SME_OK;
}

namespace sme {
// Lazy module loading (CUDA 12 default) loads this file's module on the first launch of
// any of its kernels, ~10-20 ms each; sme_preload() does it ahead of time.
int preload_diag() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)k_diag_gather<8>) == cudaSuccess ? 0 : -1;
}
}  // namespace sme
