// stream_gather_bench.cu — does the chunk stream of a panel pass (12 B/entry from
// DRAM) slow the random x gathers (L2-resident) because both occupy the SM's L1
// miss-tracking, and does moving the stream to the TMA engine (cp.async.bulk into
// a per-warp shared-memory ring) give that capacity back to the gathers?
// Standalone timing tool, C4-pass-shaped: 125M entries, x slice 50 MB.
//   gather : 4 random 8-B gathers per lane per 128-entry chunk, indices hashed (no stream)
//   ldg    : pk (int4) + val (2 x double2) per lane with LDG, then the 4 gathers (the seg probe)
//   tma    : the same chunks via cp.async.bulk into a 4-stage per-warp ring, then the gathers
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o stream_gather_bench stream_gather_bench.cu
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

#ifndef STAGES
#define STAGES 4
#endif
constexpr int NT = 256, CH = 128;

__device__ __forceinline__ uint32_t hash32(uint32_t a) {
  a ^= a >> 16; a *= 0x7feb352dU; a ^= a >> 15; a *= 0x846ca68bU; a ^= a >> 16;
  return a;
}
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_expect(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nW_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra W_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}
__device__ __forceinline__ void bulk(void* dst, const void* src, uint32_t bytes, uint64_t* bar) {
  asm volatile("cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes [%0], [%1], %2, [%3];" ::"r"(
                   smem_u32(dst)),
               "l"(src), "r"(bytes), "r"(smem_u32(bar))
               : "memory");
}

__global__ void k_init(int64_t E, uint32_t* pk, double* val, uint32_t nx, double* x) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t h = hash32((uint32_t)i * 0x9E3779B1u + 7u);
    pk[i] = (uint32_t)(((uint64_t)hash32(h) * nx) >> 32);
    val[i] = (double)(h & 0xFFFF) / 65536.0;
    if (i < nx) x[i] = (double)(h >> 16) / 65536.0;
  }
}

__device__ __forceinline__ void range(int64_t chunks, int64_t& c0, int64_t& c1) {
  const int64_t w = ((int64_t)blockIdx.x * NT + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * NT) >> 5;
  c0 = w * chunks / nw;
  c1 = (w + 1) * chunks / nw;
}

__global__ void __launch_bounds__(NT) k_gather(int64_t chunks, uint32_t nx, const double* __restrict__ x,
                                               double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  int64_t c0, c1;
  range(chunks, c0, c1);
  for (int64_t c = c0; c < c1; ++c) {
    double s = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t h = hash32((uint32_t)(c * CH + 4 * lane + k) * 0x9E3779B1u + 7u);
      s += __ldg(x + (uint32_t)(((uint64_t)hash32(h) * nx) >> 32));
    }
    y[c * 32 + lane] = s;
  }
}

__global__ void __launch_bounds__(NT) k_ldg(int64_t chunks, const uint32_t* __restrict__ pk,
                                            const double* __restrict__ val, const double* __restrict__ x,
                                            double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  int64_t c0, c1;
  range(chunks, c0, c1);
  for (int64_t c = c0; c < c1; ++c) {
    const int64_t e = c * CH + 4 * lane;
    const uint4 q = __ldcs(reinterpret_cast<const uint4*>(pk + e));
    const double2 a = __ldcs(reinterpret_cast<const double2*>(val + e));
    const double2 b = __ldcs(reinterpret_cast<const double2*>(val + e) + 1);
    y[c * 32 + lane] = a.x * __ldg(x + q.x) + a.y * __ldg(x + q.y) + b.x * __ldg(x + q.z) + b.y * __ldg(x + q.w);
  }
}

struct __align__(16) Stage {
  uint32_t pk[CH];
  double val[CH];
};

__global__ void __launch_bounds__(NT) k_tma(int64_t chunks, const uint32_t* __restrict__ pk,
                                            const double* __restrict__ val, const double* __restrict__ x,
                                            double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  Stage* ring = reinterpret_cast<Stage*>(smem) + wib * STAGES;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + sizeof(Stage) * STAGES * (NT / 32)) + wib * STAGES;
  int64_t c0, c1;
  range(chunks, c0, c1);
  if (lane == 0)
    for (int s = 0; s < STAGES; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  auto issue = [&](int64_t c, int s) {
    mbar_expect(&bar[s], sizeof(Stage));
    bulk(ring[s].pk, pk + c * CH, CH * 4, &bar[s]);
    bulk(ring[s].val, val + c * CH, CH * 8, &bar[s]);
  };
  if (lane == 0)
    for (int s = 0; s < STAGES && c0 + s < c1; ++s) issue(c0 + s, s);
  for (int64_t c = c0; c < c1; ++c) {
    const int s = (int)((c - c0) % STAGES);
    const uint32_t parity = (uint32_t)(((c - c0) / STAGES) & 1);
    mbar_wait(&bar[s], parity);
    const uint4 q = *reinterpret_cast<const uint4*>(ring[s].pk + 4 * lane);
    const double2 a = *reinterpret_cast<const double2*>(ring[s].val + 4 * lane);
    const double2 b = *reinterpret_cast<const double2*>(ring[s].val + 4 * lane + 2);
    __syncwarp();
    if (lane == 0 && c + STAGES < c1) {
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(c + STAGES, s);
    }
    y[c * 32 + lane] = a.x * __ldg(x + q.x) + a.y * __ldg(x + q.y) + b.x * __ldg(x + q.z) + b.y * __ldg(x + q.w);
  }
}

// per-CTA ring: a stage = SC consecutive chunks (SC / 8 per warp), two bulk copies per
// stage issued by thread 0; full barrier (tx bytes) and empty barrier (8 warp arrivals)
#ifndef SC
#define SC 16
#endif
struct __align__(16) CStage {
  uint32_t pk[CH * SC];
  double val[CH * SC];
};
constexpr int CSTAGES = 2;

__global__ void __launch_bounds__(NT) k_tma_cta(int64_t chunks, const uint32_t* __restrict__ pk,
                                                const double* __restrict__ val, const double* __restrict__ x,
                                                double* __restrict__ y) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  CStage* ring = reinterpret_cast<CStage*>(smem);
  uint64_t* full = reinterpret_cast<uint64_t*>(smem + sizeof(CStage) * CSTAGES);
  uint64_t* empty = full + CSTAGES;
  // CTA range in whole stages
  const int64_t stages_total = chunks / SC;
  const int64_t s0 = (int64_t)blockIdx.x * stages_total / gridDim.x, s1 = (int64_t)(blockIdx.x + 1) * stages_total / gridDim.x;
  if (threadIdx.x == 0) {
    for (int s = 0; s < CSTAGES; ++s) {
      mbar_init(&full[s], 1);
      mbar_init(&empty[s], NT / 32);
    }
  }
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncthreads();
  auto issue = [&](int64_t st, int s) {
    mbar_expect(&full[s], sizeof(CStage));
    bulk(ring[s].pk, pk + st * SC * CH, SC * CH * 4, &full[s]);
    bulk(ring[s].val, val + st * SC * CH, SC * CH * 8, &full[s]);
  };
  if (threadIdx.x == 0)
    for (int s = 0; s < CSTAGES && s0 + s < s1; ++s) issue(s0 + s, s);
  for (int64_t st = s0; st < s1; ++st) {
    const int s = (int)((st - s0) % CSTAGES);
    const uint32_t parity = (uint32_t)(((st - s0) / CSTAGES) & 1);
    mbar_wait(&full[s], parity);
    for (int j = wib; j < SC; j += NT / 32) {
      const uint4 q = *reinterpret_cast<const uint4*>(ring[s].pk + j * CH + 4 * lane);
      const double2 a = *reinterpret_cast<const double2*>(ring[s].val + j * CH + 4 * lane);
      const double2 b = *reinterpret_cast<const double2*>(ring[s].val + j * CH + 4 * lane + 2);
      y[(st * SC + j) * 32 + lane] =
          a.x * __ldg(x + q.x) + a.y * __ldg(x + q.y) + b.x * __ldg(x + q.z) + b.y * __ldg(x + q.w);
    }
    __syncwarp();
    if (lane == 0) asm volatile("mbarrier.arrive.shared::cta.b64 _, [%0];" ::"r"(smem_u32(&empty[s])) : "memory");
    if (threadIdx.x == 0 && st + CSTAGES < s1) {
      mbar_wait(&empty[s], parity);
      asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
      issue(st + CSTAGES, s);
    }
  }
}

int main() {
  const int64_t E = 125000000 / CH * CH, chunks = E / CH;
  const uint32_t nx = 6250000;
  uint32_t* pk;
  double *val, *x, *y;
  CK(cudaMalloc(&pk, E * 4));
  CK(cudaMalloc(&val, E * 8));
  CK(cudaMalloc(&x, (size_t)nx * 8));
  CK(cudaMalloc(&y, chunks * 32 * 8));
  k_init<<<4096, 256>>>(E, pk, val, nx, x);
  CK(cudaDeviceSynchronize());
  int sms;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  const int smem_tma = (int)(sizeof(Stage) * STAGES * (NT / 32) + 8 * STAGES * (NT / 32));
  CK(cudaFuncSetAttribute(k_tma, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_tma));
  const int smem_cta = (int)(sizeof(CStage) * CSTAGES + 16 * CSTAGES);
  CK(cudaFuncSetAttribute(k_tma_cta, cudaFuncAttributeMaxDynamicSharedMemorySize, smem_cta));
  int oc_c;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc_c, k_tma_cta, NT, smem_cta));
  printf("tma_cta: %d chunks per stage, %d stages, smem %d B, %d CTAs/SM\n", SC, CSTAGES, smem_cta, oc_c);
  int oc_g, oc_l, oc_t;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc_g, k_gather, NT, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc_l, k_ldg, NT, 0));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&oc_t, k_tma, NT, smem_tma));
  printf("entries %.3e, x %.0f MB, occupancy gather %d ldg %d tma %d CTAs/SM (tma smem %d B, %d stages)\n",
         (double)E, nx * 8 / 1e6, oc_g, oc_l, oc_t, smem_tma, STAGES);
  cudaEvent_t a, b;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  for (int per_sm = 2; per_sm <= 8; per_sm *= 2) {
    auto run = [&](const char* name, int occ, auto launch) {
      const int grid = sms * (per_sm < occ ? per_sm : occ);
      float best = 1e9;
      for (int it = 0; it < 6; ++it) {
        CK(cudaEventRecord(a));
        launch(grid);
        CK(cudaEventRecord(b));
        CK(cudaEventSynchronize(b));
        float ms;
        CK(cudaEventElapsedTime(&ms, a, b));
        if (it) best = ms < best ? ms : best;
      }
      CK(cudaGetLastError());
      printf("  %-7s grid %5d: %.3f ms  %.1f G gathers/s\n", name, grid, best, (double)E / best / 1e6);
    };
    printf("CTAs per SM requested: %d\n", per_sm);
    run("gather", oc_g, [&](int g) { k_gather<<<g, NT>>>(chunks, nx, x, y); });
    run("ldg", oc_l, [&](int g) { k_ldg<<<g, NT>>>(chunks, pk, val, x, y); });
    run("tma", oc_t, [&](int g) { k_tma<<<g, NT, smem_tma>>>(chunks, pk, val, x, y); });
    run("tma_cta", oc_c, [&](int g) { k_tma_cta<<<g, NT, smem_cta>>>(chunks, pk, val, x, y); });
  }
  return 0;
}
