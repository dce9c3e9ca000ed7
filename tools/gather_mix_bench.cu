// gather_mix_bench.cu — do LDG gathers and TMA tile::gather4 gathers share one
// ceiling?  The seg SpMV is bound by the SM's L1 -> crossbar request port (one LDG
// gather = one request; ~1 per SM clock).  TMA requests are issued by the SM's TMA
// unit.  If that path does not queue behind the L1 port, warps issuing gather4 next
// to warps issuing LDG would add gather rates (standalone tool, not part of libsme).
//
// One kernel, 8 warps per CTA: warps [0, NL) do LDG gathers (per_l per lane), warps
// [NL, 8) do gather4 (per_g per lane, 4 random 16-B rows per instruction).  Each
// (NL, per_l, per_g) point is timed three ways: both roles, LDG role only (per_g = 0),
// gather4 role only (per_l = 0).  Both roles on independent paths => t_mix ~ max.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o gather_mix_bench gather_mix_bench.cu -lcuda
//   ./gather_mix_bench [x_mb]
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

constexpr int G_ST = 4;     // gather4 stages per warp
constexpr int LSTRIDE = 16;  // doubles per lane per stage (128-B aligned destinations)
constexpr int WARPS = 8;
constexpr int G4_MAX = 4;  // gather4 warps per CTA at most (their staging sets the occupancy)

__global__ void __launch_bounds__(256) k_mix(const __grid_constant__ CUtensorMap tm, const double* __restrict__ x,
                                             uint32_t n, int nl, int per_l, int per_g, int lanes_g, double* out) {
  extern __shared__ __align__(128) unsigned char smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const uint32_t tid = blockIdx.x * blockDim.x + threadIdx.x;
  double acc = 0.0;
  if (wib < nl) {
    constexpr int U = 8;
    for (int i = 0; i < per_l; i += U) {
      double v[U];
#pragma unroll
      for (int u = 0; u < U; ++u) {
        const uint32_t h = hash32(tid * 0x9E3779B1u + (uint32_t)(i + u) * 0x85EBCA77u);
        asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];"
                     : "=d"(v[u])
                     : "l"(x + (uint32_t)(((uint64_t)h * n) >> 32)));
      }
#pragma unroll
      for (int u = 0; u < U; ++u) acc += v[u];
    }
  } else {
    const int gw = wib - nl;
    double* buf = reinterpret_cast<double*>(smem) + (size_t)gw * G_ST * 32 * LSTRIDE;
    uint64_t* bar = reinterpret_cast<uint64_t*>(smem + (size_t)(G4_MAX * 32 * LSTRIDE * 8 * G_ST)) + gw * G_ST;
    if (lane == 0)
      for (int s = 0; s < G_ST; ++s) mbar_init(&bar[s], 1);
    asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
    __syncwarp();
    const uint32_t nrows = n / 2;
    const int steps = per_g / 4;
    auto issue = [&](int it) {
      const int s = it % G_ST;
      if (lane == 0) mbar_arrive_expect_tx(&bar[s], lanes_g * 64);
      __syncwarp();
      if (lane < lanes_g) {
        uint32_t r[4];
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const uint32_t h = hash32(tid * 0x9E3779B1u + (uint32_t)(it * 4 + u) * 0x85EBCA77u);
          r[u] = (uint32_t)(((uint64_t)h * nrows) >> 32);
        }
        asm volatile(
            "cp.async.bulk.tensor.2d.shared::cta.global.tile::gather4.mbarrier::complete_tx::bytes [%0], [%1, {%2, "
            "%3, %4, %5, %6}], [%7];" ::"r"(smem_u32(buf + (size_t)s * 32 * LSTRIDE + lane * LSTRIDE)),
            "l"(&tm), "r"(0), "r"(r[0]), "r"(r[1]), "r"(r[2]), "r"(r[3]), "r"(smem_u32(&bar[s]))
            : "memory");
      }
    };
    for (int it = 0; it < G_ST && it < steps; ++it) issue(it);
    for (int it = 0; it < steps; ++it) {
      const int s = it % G_ST;
      mbar_wait(&bar[s], (it / G_ST) & 1);
      if (lane < lanes_g) {
        const double* b = buf + (size_t)s * 32 * LSTRIDE + lane * LSTRIDE;
#pragma unroll
        for (int u = 0; u < 4; ++u) acc += b[2 * u + (tid & 1)];
      }
      __syncwarp();
      if (it + G_ST < steps) issue(it + G_ST);
    }
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
  const int x_mb = argc > 1 ? atoi(argv[1]) : 48;
  const size_t n = (size_t)x_mb * (1 << 20) / 8;
  double* x;
  CK(cudaMalloc(&x, n * 8));
  CK(cudaMemset(x, 0, n * 8));
  CUtensorMap tm;
  cuuint64_t dims[2] = {2, n / 2};
  cuuint64_t strides[1] = {16};
  cuuint32_t box[2] = {2, 1};
  cuuint32_t es[2] = {1, 1};
  if (encode(&tm, CU_TENSOR_MAP_DATA_TYPE_FLOAT64, 2, x, dims, strides, box, es, CU_TENSOR_MAP_INTERLEAVE_NONE,
             CU_TENSOR_MAP_SWIZZLE_NONE, CU_TENSOR_MAP_L2_PROMOTION_NONE,
             CU_TENSOR_MAP_FLOAT_OOB_FILL_NONE) != CUDA_SUCCESS) {
    fprintf(stderr, "encode failed\n");
    return 1;
  }
  const size_t smem = (size_t)G4_MAX * 32 * LSTRIDE * 8 * G_ST + G4_MAX * G_ST * 8;
  CK(cudaFuncSetAttribute(k_mix, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int occ = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, k_mix, 256, smem));
  const int blocks = sms * occ;
  double* out;
  CK(cudaMalloc(&out, (size_t)blocks * 256 * 8));
  cudaEvent_t e0, e1;
  cudaEventCreate(&e0);
  cudaEventCreate(&e1);
  auto time = [&](int nl, int per_l, int per_g, int lanes_g) {
    for (int w = 0; w < 2; ++w) k_mix<<<blocks, 256, smem>>>(tm, x, (uint32_t)n, nl, per_l, per_g, lanes_g, out);
    CK(cudaGetLastError());
    CK(cudaDeviceSynchronize());
    const int reps = 5;
    cudaEventRecord(e0);
    for (int r = 0; r < reps; ++r) k_mix<<<blocks, 256, smem>>>(tm, x, (uint32_t)n, nl, per_l, per_g, lanes_g, out);
    cudaEventRecord(e1);
    CK(cudaEventSynchronize(e1));
    float ms = 0;
    cudaEventElapsedTime(&ms, e0, e1);
    return ms / reps;
  };
  printf("{\"x_mb\": %d, \"ctas_per_sm\": %d, \"blocks\": %d}\n", x_mb, occ, blocks);
  const int per_l = 512;
  // reference rates: pure LDG (8 warps), pure gather4 (8 warps)
  {
    const float tl = time(8, per_l, 0, 32);
    const float tg = time(WARPS - G4_MAX, 0, per_l, 32);
    const double el = (double)blocks * 256 * per_l;
    printf("{\"mode\": \"ldg_8warps\", \"ms\": %.4f, \"gps\": %.4g}\n", tl, el / (tl * 1e-3));
    printf("{\"mode\": \"g4_4warps\", \"ms\": %.4f, \"gps\": %.4g}\n", tg, el / 2 / (tg * 1e-3));
  }
  for (int nl : {7, 6, 5, 4}) {
    for (int lanes_g : {32, 8}) {
      for (int per_g : {64, 128, 256, 512, 1024}) {
        const float tm_ = time(nl, per_l, per_g, lanes_g);
        const float tl = time(nl, per_l, 0, lanes_g);
        const float tg = time(nl, 0, per_g, lanes_g);
        const double gl = (double)blocks * nl * 32 * per_l;
        const double gg = (double)blocks * (WARPS - nl) * lanes_g * per_g;
        printf("{\"nl\": %d, \"lanes_g\": %d, \"per_g\": %d, \"ms_mix\": %.4f, \"ms_ldg_only\": %.4f, \"ms_g4_only\": %.4f, "
               "\"gps_mix\": %.4g, \"gps_ldg_only\": %.4g, \"gps_g4_only\": %.4g}\n",
               nl, lanes_g, per_g, tm_, tl, tg, (gl + gg) / (tm_ * 1e-3), gl / (tl * 1e-3), gg / (tg * 1e-3));
        fflush(stdout);
      }
    }
  }
  return 0;
}
