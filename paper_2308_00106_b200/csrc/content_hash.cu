// content_hash.cu — 64-bit content hash of device arrays (the key of the on-disk
// permuted-CSR cache, cache.py).  h = sum_i mix64(seed' + i * G ^ (w_i * K)) mod 2^64
// over the 32-bit words w_i: every word is tied to its index, and the sum is
// order-free, so the result is deterministic under any grid.  Not cryptographic:
// it keys a cache of matrices the caller built, it does not authenticate them.
#include "common.cuh"

#include "hash.cuh"

namespace sme {

__global__ void k_hash_words(int64_t n, const uint32_t* __restrict__ w, uint64_t seed,
                             unsigned long long* __restrict__ out) {
  uint64_t acc = 0;
  const uint64_t s = mix64(seed ^ 0xC0FFEE5EEDull);
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    acc += mix64((s + (uint64_t)i * 0x9E3779B97F4A7C15ull) ^ ((uint64_t)__ldg(w + i) * 0xD1B54A32D192ED03ull));
  for (int o = 16; o; o >>= 1) acc += __shfl_xor_sync(0xffffffffu, acc, o);
  if ((threadIdx.x & 31) == 0) atomicAdd(out, (unsigned long long)acc);
}

}  // namespace sme

using namespace sme;

SME_API int sme_hash64(const void* d_data, int64_t n_bytes, uint64_t seed, uint64_t* d_out, sme_stream_t stream) {
  SME_REQUIRE(n_bytes >= 0 && n_bytes % 4 == 0, "n_bytes %lld must be a multiple of 4", (long long)n_bytes);
  SME_REQUIRE(n_bytes == 0 || ((uintptr_t)d_data & 3) == 0, "data must be 4-byte aligned");
  cudaStream_t s = as_stream(stream);
  SME_CUDA(cudaMemsetAsync(d_out, 0, 8, s));
  const int64_t n = n_bytes / 4;
  if (n == 0) return SME_OK;
  k_hash_words<<<grid_for(n, 256, 4), 256, 0, s>>>(n, (const uint32_t*)d_data, seed, (unsigned long long*)d_out);
  SME_CHECK_LAUNCH("k_hash_words");
  return SME_OK;
}

namespace sme {
// Lazy module loading (CUDA 12 default) loads this file's module on the first launch of
// any of its kernels, ~10-20 ms each; sme_preload() does it ahead of time.
int preload_content_hash() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)k_hash_words) == cudaSuccess ? 0 : -1;
}
}  // namespace sme
