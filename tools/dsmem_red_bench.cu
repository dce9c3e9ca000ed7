// DSMEM f64 reduction throughput: each thread adds to random words of random CTAs of its cluster.
#include <cstdio>
#include <cstdint>
#include <cooperative_groups.h>
namespace cg = cooperative_groups;

constexpr int NT = 256;
constexpr int WORDS = 24 * 1024;  // 192 KB of f64 per CTA

__device__ __forceinline__ uint32_t rng(uint32_t& s) { s ^= s << 13; s ^= s >> 17; s ^= s << 5; return s; }

template <int MODE>  // 0: remote (cluster) red.f64, 1: local smem red.f64, 2: remote red.f32, 3: local atomicAdd f64 via atomicAdd()
__global__ void k(int iters, double* out) {
  extern __shared__ double sm[];
  cg::cluster_group cl = cg::this_cluster();
  for (int i = threadIdx.x; i < WORDS; i += NT) sm[i] = 0.0;
  cl.sync();
  uint32_t s = 0x9e3779b9u ^ (blockIdx.x * NT + threadIdx.x) * 2654435761u;
  const unsigned nb = cl.num_blocks();
  uint32_t base = (uint32_t)__cvta_generic_to_shared(sm);
  for (int it = 0; it < iters; ++it) {
    uint32_t r = rng(s);
    uint32_t w = r % WORDS;
    uint32_t rank = (r >> 20) % nb;
    if (MODE == 0) {
      uint32_t la = base + w * 8, ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
      asm volatile("red.shared::cluster.add.f64 [%0], %1;" ::"r"(ra), "d"(1.0) : "memory");
    } else if (MODE == 1) {
      uint32_t la = base + w * 8;
      asm volatile("red.shared.add.f64 [%0], %1;" ::"r"(la), "d"(1.0) : "memory");
    } else if (MODE == 2) {
      uint32_t la = base + w * 4, ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
      asm volatile("red.shared::cluster.add.f32 [%0], %1;" ::"r"(ra), "f"(1.0f) : "memory");
    } else {
      uint32_t la = base + w * 8, ra;
      asm volatile("mapa.shared::cluster.u32 %0, %1, %2;" : "=r"(ra) : "r"(la), "r"(rank));
      double v;
      asm volatile("ld.shared::cluster.f64 %0, [%1];" : "=d"(v) : "r"(ra) : "memory");
      if (v == 12345.0) out[0] = v;
    }
  }
  cl.sync();
  if (threadIdx.x == 0) out[blockIdx.x] = sm[5];
}

template <int MODE>
void run(int cluster, const char* name) {
  auto kern = k<MODE>;
  size_t smem = WORDS * 8;
  cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem);
  cudaFuncSetAttribute(kern, cudaFuncAttributeNonPortableClusterSizeAllowed, 1);
  int sms; cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0);
  int grid = (sms / cluster) * cluster;
  double* out; cudaMalloc(&out, grid * 8);
  cudaLaunchConfig_t cfg = {};
  cfg.gridDim = grid; cfg.blockDim = NT; cfg.dynamicSmemBytes = smem;
  cudaLaunchAttribute at[1];
  at[0].id = cudaLaunchAttributeClusterDimension; at[0].val.clusterDim.x = cluster; at[0].val.clusterDim.y = 1; at[0].val.clusterDim.z = 1;
  cfg.attrs = at; cfg.numAttrs = 1;
  int iters = 4096;
  cudaLaunchKernelEx(&cfg, kern, iters, out);
  cudaEvent_t a, b; cudaEventCreate(&a); cudaEventCreate(&b);
  cudaEventRecord(a);
  cudaLaunchKernelEx(&cfg, kern, iters, out);
  cudaEventRecord(b);
  cudaError_t e = cudaEventSynchronize(b);
  float ms; cudaEventElapsedTime(&ms, a, b);
  double ops = (double)grid * NT * iters;
  printf("%-28s cluster=%2d grid=%d: %.3f ms  %.1f G ops/s  %.2f ops/SM/clk@1.9GHz  (%s)\n", name, cluster, grid, ms,
         ops / ms / 1e6, ops / (ms * 1e-3) / grid / 1.9e9, cudaGetErrorString(e));
  cudaFree(out);
}

int main() {
  for (int c : {2, 8, 16}) {
    run<0>(c, "remote red.f64");
    run<2>(c, "remote red.f32");
    run<3>(c, "remote ld.f64");
  }
  run<1>(1, "local red.f64");
  return 0;
}
