// gather_bench.cu — random-gather rate of the B200 through three paths, to pick
// the x-gather mechanism of the panel SpMV (standalone tool, not part of libsme):
//   ldg   : one 8-byte LDG per element (each lane a different 128-B line: one
//           L1tex wavefront per element)
//   g4    : TMA tile::gather4 (4 random 16-byte rows of x viewed as [n/2][2] per
//           instruction, issued by every lane, landing in shared memory on an
//           mbarrier; values then read with LDS)
//   bulk  : per-lane 16-byte cp.async.bulk (non-tensor TMA) into shared memory
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_bench gather_bench.cu -lcuda
//   ./gather_bench [x_mb ...]
#include <cuda.h>
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
__device__ __forceinline__ uint32_t smem_u32(const void* p) { return (uint32_t)__cvta_generic_to_shared(p); }
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes) : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n.reg .pred p;\nWAIT_%=:\nmbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n@!p bra WAIT_%=;\n}\n" ::"r"(
          smem_u32(bar)),
      "r"(parity)
      : "memory");
}

template <int U>
__global__ void __launch_bounds__(256) k_ldg(const double* __restrict__ x, uint32_t n, int per, double* out) {
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  for (int i = 0; i < per; i += U) {
    double v[U];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const uint32_t h = hash32(tid * 0x9E3779B1u + (uint32_t)(i + u) * 0x85EBCA77u);
      v[u] = __ldg(x + (uint32_t)(((uint64_t)h * n) >> 32));
    }
#pragma unroll
    for (int u = 0; u < U; ++u) acc += v[u];
  }
  out[tid] = acc;
}

// every lane issues one gather4 (4 random 16-B rows) per stage; STAGES stages per warp
constexpr int G_ST = 4;
#ifndef LSTRIDE
#define LSTRIDE 16  // doubles between lanes' gather4 destinations (TMA needs 128-B aligned smem)
#endif
__global__ void __launch_bounds__(256) k_g4(const __grid_constant__ CUtensorMap tm, uint32_t nrows, int per,
                                            double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  double* buf = reinterpret_cast<double*>(smem) + (size_t)wib * G_ST * 32 * LSTRIDE;  // stage: 32 lanes x 4 rows x 2 dbl
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8 * 32 * LSTRIDE * 8 * G_ST) + wib * G_ST;
  if (lane == 0)
    for (int s = 0; s < G_ST; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  double acc = 0.0;
  const int steps = per / 4;  // each step: 4 elements per lane
  auto issue = [&](int it) {
    const int s = it % G_ST;
    if (lane == 0) mbar_arrive_expect_tx(&bar[s], 32 * 64);
    __syncwarp();
    uint32_t r[4];
#pragma unroll
    for (int u = 0; u < 4; ++u) {
      const uint32_t h = hash32(tid * 0x9E3779B1u + (uint32_t)(it * 4 + u) * 0x85EBCA77u);
      r[u] = (uint32_t)(((uint64_t)h * nrows) >> 32);
    }
    asm volatile(
        "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, %3, %4, "
        "%5, %6}], [%7];" ::"r"(smem_u32(buf + (size_t)s * 32 * LSTRIDE + lane * LSTRIDE)),
        "l"(&tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(smem_u32(&bar[s]))
        : "memory");
  };
  for (int it = 0; it < G_ST && it < steps; ++it) issue(it);
  for (int it = 0; it < steps; ++it) {
    const int s = it % G_ST;
    mbar_wait(&bar[s], (it / G_ST) & 1);
    const double* b = buf + (size_t)s * 32 * LSTRIDE + lane * LSTRIDE;
#pragma unroll
    for (int u = 0; u < 4; ++u) acc += b[2 * u + (tid & 1)];
    __syncwarp();
    if (it + G_ST < steps) issue(it + G_ST);
  }
  out[tid] = acc;
}

// every lane issues one 16-byte bulk copy per stage (4 stages per lane group of 4 elements)
__global__ void __launch_bounds__(256) k_bulk(const double* __restrict__ x, uint32_t nrows, int per, double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  double* buf = reinterpret_cast<double*>(smem) + (size_t)wib * G_ST * 32 * 2;
  uint64_t* bar = reinterpret_cast<uint64_t*>(smem + 8 * 32 * 2 * 8 * G_ST) + wib * G_ST;
  if (lane == 0)
    for (int s = 0; s < G_ST; ++s) mbar_init(&bar[s], 1);
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
  __syncwarp();
  double acc = 0.0;
  auto issue = [&](int it) {
    const int s = it % G_ST;
    if (lane == 0) mbar_arrive_expect_tx(&bar[s], 32 * 16);
    __syncwarp();
    const uint32_t h = hash32(tid * 0x9E3779B1u + (uint32_t)it * 0x85EBCA77u);
    const uint32_t r = (uint32_t)(((uint64_t)h * nrows) >> 32);
    asm volatile("cp.async.bulk.shared::cta.global.mbarrier::complete_tx::bytes [%0], [%1], 16, [%2];" ::"r"(
                     smem_u32(buf + (size_t)s * 64 + lane * 2)),
                 "l"(x + 2 * (size_t)r), "r"(smem_u32(&bar[s]))
                 : "memory");
  };
  for (int it = 0; it < G_ST && it < per; ++it) issue(it);
  for (int it = 0; it < per; ++it) {
    const int s = it % G_ST;
    mbar_wait(&bar[s], (it / G_ST) & 1);
    acc += buf[(size_t)s * 64 + lane * 2 + (tid & 1)];
    __syncwarp();
    if (it + G_ST < per) issue(it + G_ST);
  }
  out[tid] = acc;
}

typedef CUresult (*EncodeFn)(CUtensorMap*, CUtensorMapDataType, cuuint32_t, void*, const cuuint64_t*,
                             const cuuint64_t*, const cuuint32_t*, const cuuint32_t*, CUtensorMapInterleave,
                             CUtensorMapSwizzle, CUtensorMapL2promotion, CUtensorMapFloatOOBfill);

int main(int argc, char** argv) {
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  void* fn = nullptr;
  cudaDriverEntryPointQueryResult q;
  CK(cudaGetDriverEntryPoint("cuTensorMapEncodeTiled", &fn, cudaEnableDefault, &q));
  EncodeFn encode = (EncodeFn)fn;
  int mbs[16] = {8, 64, 400};
  int nmb = 3;
  if (argc > 1) {
    nmb = 0;
    for (int i = 1; i < argc && nmb < 16; ++i) mbs[nmb++] = atoi(argv[i]);
  }
  const int per = 256;
  for (int occ : {4, 8}) {
    const int blocks = sms * occ;
    double* out;
    CK(cudaMalloc(&out, (size_t)blocks * 256 * 8));
    for (int k = 0; k < nmb; ++k) {
      const size_t n = (size_t)mbs[k] * (1 << 20) / 8;
      double* x;
      CK(cudaMalloc(&x, n * 8));
      CK(cudaMemset(x, 0, n * 8));
      CUtensorMap tm;
      cuuint64_t dims[2] = {2, n / 2};
      cuuint64_t strides[1] = {16};
      cuuint32_t box[2] = {2, 1};
      cuuint32_t es[2] = {1, 1};
      CUresult cr = encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es,
                           CU_TENSOR_MAP_INTERLEAVE_NONE, CU_TENSOR_MAP_SWIZZLE_NONE,
                           CU_TENSOR_MAP_L2_PROMOTION_NONE, CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE);
      if (cr != CUDA_SUCCESS) { fprintf(stderr, "encode failed %d\n", (int)cr); return 1; }
      const size_t g4_smem = 8 * 32 * LSTRIDE * 8 * G_ST + 8 * G_ST * 8;
      const size_t bk_smem = 8 * 32 * 2 * 8 * G_ST + 8 * G_ST * 8;
      CK(cudaFuncSetAttribute(k_g4, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)g4_smem));
      cudaEvent_t e0, e1;
      cudaEventCreate(&e0);
      cudaEventCreate(&e1);
      for (int kind = 0; kind < 3; ++kind) {
        auto launch = [&]() {
          if (kind == 0) k_ldg<8><<<blocks, 256>>>(x, (uint32_t)n, per, out);
          else if (kind == 1) k_g4<<<blocks, 256, g4_smem>>>(tm, (uint32_t)(n / 2), per, out);
          else k_bulk<<<blocks, 256, bk_smem>>>(x, (uint32_t)(n / 2), per, out);
        };
        for (int w = 0; w < 2; ++w) launch();
        CK(cudaGetLastError());
        CK(cudaDeviceSynchronize());
        cudaEventRecord(e0);
        const int reps = 5;
        for (int r = 0; r < reps; ++r) launch();
        cudaEventRecord(e1);
        CK(cudaEventSynchronize(e1));
        float ms = 0;
        cudaEventElapsedTime(&ms, e0, e1);
        ms /= reps;
        const double elems = (double)blocks * 256 * per;
        const char* names[3] = {"ldg", "g4", "bulk16"};
        printf("{\"path\": \"%s\", \"occ_ctas\": %d, \"x_mb\": %d, \"ms\": %.4f, \"gathers_per_s\": %.4g}\n",
               names[kind], occ, mbs[k], ms, elems / (ms * 1e-3));
        fflush(stdout);
      }
      CK(cudaFree(x));
    }
    CK(cudaFree(out));
  }
  return 0;
}
