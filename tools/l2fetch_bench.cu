// l2fetch_bench.cu — random 4-byte gathers from a table larger than L2 (the p_c column
// map of K4, 200 MB at C4) under each cudaLimitMaxL2FetchGranularity, with and without
// an accompanying 12 B/entry stream (the CSR rows K4 reads).  Standalone tool.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o l2fetch_bench l2fetch_bench.cu
//   ./l2fetch_bench [table_mb ...]
#include <cuda_runtime.h>
#include <stdint.h>
#include <stdio.h>
#include <stdlib.h>

#define CK(x)                                                                          \
  do {                                                                                 \
    cudaError_t e = (x);                                                               \
    if (e != cudaSuccess) {                                                            \
      fprintf(stderr, "%s:%d %s: %s\n", __FILE__, __LINE__, #x, cudaGetErrorString(e)); \
      exit(1);                                                                         \
    }                                                                                  \
  } while (0)

__device__ __forceinline__ uint32_t hash32(uint32_t a) {
  a ^= a >> 16; a *= 0x7feb352dU; a ^= a >> 15; a *= 0x846ca68bU; a ^= a >> 16;
  return a;
}

// MODE 0: plain __ldg; 1: ld.global.nc.L1::no_allocate; 2: L2 evict_last hint
template <int MODE, bool STREAM>
__global__ void __launch_bounds__(256) k_gather(const int32_t* __restrict__ t, uint32_t n, int per,
                                                const int4* __restrict__ s, uint64_t s_n4, int32_t* out) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  const uint32_t nt = gridDim.x * blockDim.x;
  uint64_t pol;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(pol));
  uint64_t pol_f;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(pol_f));
  int32_t acc = 0;
  for (int i = 0; i < per; i += 4) {
    int32_t v[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t h = hash32(tid * 0x9E3779B1u + (uint32_t)(i + u) * 0x85EBCA77u);
      const int32_t* p = t + (uint32_t)(((uint64_t)h * n) >> 32);
      if (MODE == 0) v[u] = __ldg(p);
      else if (MODE == 1) asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(v[u]) : "l"(p));
      else asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(v[u]) : "l"(p), "l"(pol));
    }
    if (STREAM) {  // 3 x 16 B per 4 gathers = 12 B per gather, coalesced, evict-first
      uint64_t q = ((uint64_t)(i / 4) * nt + tid) * 3;
#pragma unroll
      for (int u = 0; u < 3; ++u) {
        int4 w;
        const int4* pp = s + ((q + u) % s_n4);
        asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
                     : "=r"(w.x), "=r"(w.y), "=r"(w.z), "=r"(w.w) : "l"(pp), "l"(pol_f));
        acc ^= w.x ^ w.w;
      }
    }
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += v[u];
  }
  out[tid] = acc;
}

template <int MODE, bool STREAM>
float run(const int32_t* t, uint32_t n, const int4* s, uint64_t s_n4, int32_t* out, int blocks, int per) {
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  k_gather<MODE, STREAM><<<blocks, 256>>>(t, n, per, s, s_n4, out);
  CK(cudaEventRecord(a));
  for (int r = 0; r < 3; ++r) k_gather<MODE, STREAM><<<blocks, 256>>>(t, n, per, s, s_n4, out);
  CK(cudaEventRecord(b));
  CK(cudaEventSynchronize(b));
  float ms;
  CK(cudaEventElapsedTime(&ms, a, b));
  return ms / 3;
}

int main(int argc, char** argv) {
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  size_t g0;
  CK(cudaDeviceGetLimit(&g0, cudaLimitMaxL2FetchGranularity));
  printf("default cudaLimitMaxL2FetchGranularity = %zu\n", g0);
  const int blocks = sms * 8, per = 512;
  const double gathers = (double)blocks * 256 * per;
  const uint64_t s_bytes = 4ull << 30;
  int4* s;
  CK(cudaMalloc(&s, s_bytes));
  CK(cudaMemset(s, 1, s_bytes));
  int32_t* out;
  CK(cudaMalloc(&out, blocks * 256 * 4));
  int nt = argc > 1 ? argc - 1 : 4;
  const char* defaults[] = {"50", "100", "200", "400"};
  for (int a = 0; a < nt; ++a) {
    const double mb = atof(argc > 1 ? argv[a + 1] : defaults[a]);
    const uint32_t n = (uint32_t)(mb * 1e6 / 4);
    int32_t* t;
    CK(cudaMalloc(&t, (size_t)n * 4));
    CK(cudaMemset(t, 0, (size_t)n * 4));
    const size_t gr[] = {32, 64, 128};
    for (size_t g : gr) {
      CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g));
      size_t got;
      CK(cudaDeviceGetLimit(&got, cudaLimitMaxL2FetchGranularity));
      float m0 = run<0, false>(t, n, s, s_bytes / 16, out, blocks, per);
      float m1 = run<1, false>(t, n, s, s_bytes / 16, out, blocks, per);
      float m2 = run<2, false>(t, n, s, s_bytes / 16, out, blocks, per);
      float s0 = run<0, true>(t, n, s, s_bytes / 16, out, blocks, per);
      float s2 = run<2, true>(t, n, s, s_bytes / 16, out, blocks, per);
      printf("table %6.0f MB gran %3zu (got %3zu): G/s ldg %6.1f  noalloc %6.1f  evict_last %6.1f | "
             "+12B stream: ldg %6.1f evict_last %6.1f\n",
             mb, g, got, gathers / m0 / 1e6, gathers / m1 / 1e6, gathers / m2 / 1e6, gathers / s0 / 1e6,
             gathers / s2 / 1e6);
    }
    CK(cudaFree(t));
  }
  CK(cudaDeviceSetLimit(cudaLimitMaxL2FetchGranularity, g0));
  return 0;
}
