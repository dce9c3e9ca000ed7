// binned_bench.cu — timing prototype of a two-phase ("binned") SpMV for matrices
// whose x does not fit L2 and whose columns are random (C4).  Standalone tool,
// not part of libsme; synthetic layout with C4's statistics (50M x 50M, ~20
// nonzeros per row), values/indices random.
//
//   phase 1 (expand):  CTA per column block (CB columns, x block staged in smem):
//                      prod[e] = val[e] * xs[coloff[e]]   (elementwise stream,
//                      x gathers from shared memory, no L2 gathers at all)
//   phase 2 (combine): CTA per row bin (RB rows, y block in smem): the bin's cells
//                      (one per column block, cb-major storage) staged in smem in
//                      chunks; a static row-sorted word stream (pos | rowoff)
//                      sums each row's run in order and adds it to y[row]
//                      (deterministic, no atomics).
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o binned_bench binned_bench.cu
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

#ifndef RB
#define RB 8192
#endif
#ifndef CB
#define CB 16384
#endif
#ifndef CELL
#define CELL 54  // entries per cell (C4 mean: RB * CB * 20 / 50M)
#endif
#ifndef KC
#define KC 64  // cells per phase-2 chunk
#endif
#ifndef EXU
#define EXU 2
#endif
#ifndef P1T
#define P1T 1024
#endif
#ifndef P2T
#define P2T 512
#endif
constexpr int CHUNK = KC * CELL;

__device__ __forceinline__ uint32_t hash32(uint32_t a) {
  a ^= a >> 16; a *= 0x7feb352dU; a ^= a >> 15; a *= 0x846ca68bU; a ^= a >> 16;
  return a;
}

__global__ void k_init(int64_t E, double* val, uint16_t* coloff, int64_t n, double* x) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t h = hash32((uint32_t)i * 0x9E3779B1u + (uint32_t)(i >> 32));
    val[i] = (double)(h & 0xFFFF) / 65536.0 - 0.5;
    coloff[i] = (uint16_t)(hash32(h) % CB);
    if (i < n) x[i] = (double)(h >> 16) / 65536.0;
  }
}

// words for every chunk: sorted rows (monotone rowoff), positions a bijection of [0, CHUNK)
__global__ void k_words(int64_t nw, uint32_t* words) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < nw; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t k = (uint32_t)(i % CHUNK);
    const uint32_t pos = (uint32_t)(((uint64_t)k * 2459u) % CHUNK);
    const uint32_t row = (uint32_t)(((uint64_t)k * RB) / CHUNK);
    words[i] = pos | (row << 13);
  }
}

__device__ __forceinline__ double2 ldg_stream_d2(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v2.f64 {%0, %1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ uint4 ldg_stream_u4(const uint4* p) {
  uint4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::256B.v4.u32 {%0, %1, %2, %3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w) : "l"(p));
  return r;
}
__device__ __forceinline__ void st_stream_d2(double2* p, double2 v) {
  asm volatile("st.global.L1::no_allocate.v2.f64 [%0], {%1, %2};" ::"l"(p), "d"(v.x), "d"(v.y) : "memory");
}

// phase 1: one CTA per column block; entries of block cb are [cb * per, (cb + 1) * per)
__global__ void __launch_bounds__(P1T) k_expand(int64_t n_cols, int64_t per, const double* __restrict__ x,
                                               const double* __restrict__ val, const uint16_t* __restrict__ coloff,
                                               double* __restrict__ prod) {
  extern __shared__ double xs[];
  const int cb = blockIdx.x;
  const int64_t c0 = (int64_t)cb * CB;
  for (int i = threadIdx.x; i < CB; i += P1T) xs[i] = c0 + i < n_cols ? x[c0 + i] : 0.0;
  __syncthreads();
  const int64_t e0 = (int64_t)cb * per, e1 = e0 + per;  // per % 8 == 0
  constexpr int U = EXU;
  for (int64_t eb = e0 + 8 * (int64_t)threadIdx.x; eb < e1; eb += 8 * P1T * U) {
    uint4 q[U];
    double2 v[U][4];
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = eb + (int64_t)u * 8 * P1T;
      if (e < e1) {
        q[u] = __ldcs(reinterpret_cast<const uint4*>(coloff + e));
#pragma unroll
        for (int k = 0; k < 4; ++k) v[u][k] = __ldcs(reinterpret_cast<const double2*>(val + e) + k);
      }
    }
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = eb + (int64_t)u * 8 * P1T;
      if (e < e1) {
        const uint32_t w[4] = {q[u].x, q[u].y, q[u].z, q[u].w};
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          double2 p;
          p.x = v[u][k].x * xs[w[k] & 0xFFFF];
          p.y = v[u][k].y * xs[w[k] >> 16];
          __stcs(reinterpret_cast<double2*>(prod + e) + k, p);
        }
      }
    }
  }
}

__device__ __forceinline__ void cp16(void* smem, const void* g) {
  asm volatile("cp.async.cg.shared.global.L2::256B [%0], [%1], 16;" ::"r"((uint32_t)__cvta_generic_to_shared(smem)),
               "l"(g)
               : "memory");
}
__device__ __forceinline__ void cp_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
__device__ __forceinline__ void cp_wait1() { asm volatile("cp.async.wait_group 1;" ::: "memory"); }

// phase 2: one CTA per row bin; chunks double-buffered with cp.async
__global__ void __launch_bounds__(P2T) k_combine(int64_t n_rows, int nrb, int ncb, const double* __restrict__ prod,
                                                const uint32_t* __restrict__ words, double* __restrict__ y) {
  extern __shared__ double sm[];
  double* ys = sm;                                                // RB
  double* buf0 = sm + RB;                                         // 2 x CHUNK
  uint32_t* wb0 = reinterpret_cast<uint32_t*>(buf0 + 2 * CHUNK);  // 2 x CHUNK
  const int rb = blockIdx.x;
  for (int i = threadIdx.x; i < RB; i += P2T) ys[i] = 0.0;
  const int lane = threadIdx.x & 31, wid = threadIdx.x >> 5;
  const int n_chunks = ncb / KC;
  const uint32_t* wrb = words + (int64_t)rb * n_chunks * CHUNK;
  auto stage = [&](int j) {
    double* buf = buf0 + (j & 1) * CHUNK;
    uint32_t* wb = wb0 + (j & 1) * CHUNK;
    for (int c = wid; c < KC; c += P2T / 32) {
      const double* src = prod + ((int64_t)(j * KC + c) * nrb + rb) * CELL;
      for (int k = lane; k < CELL / 2; k += 32) cp16(buf + c * CELL + 2 * k, src + 2 * k);
    }
    const uint32_t* wsrc = wrb + (int64_t)j * CHUNK;
    for (int k = threadIdx.x; k < CHUNK / 4; k += P2T) cp16(wb + 4 * k, wsrc + 4 * k);
  };
  stage(0);
  cp_commit();
  for (int j = 0; j < n_chunks; ++j) {
    if (j + 1 < n_chunks) stage(j + 1);
    cp_commit();
    cp_wait1();
    __syncthreads();
    const double* buf = buf0 + (j & 1) * CHUNK;
    const uint32_t* wb = wb0 + (j & 1) * CHUNK;
    for (int i = threadIdx.x; i < CHUNK; i += P2T) {
      const uint32_t w = wb[i];
      const uint32_t row = w >> 13;
      if (i > 0 && (wb[i - 1] >> 13) == row) continue;
      double s = buf[w & 0x1FFF];
      for (int k = i + 1; k < CHUNK && (wb[k] >> 13) == row; ++k) s += buf[wb[k] & 0x1FFF];
      ys[row] += s;
    }
    __syncthreads();
  }
  const int64_t r0 = (int64_t)rb * RB;
  for (int i = threadIdx.x; i < RB; i += P2T)
    if (r0 + i < n_rows) y[r0 + i] = ys[i];
}

#ifndef BB_NO_MAIN
int main(int argc, char** argv) {
  const int64_t n = argc > 1 ? atoll(argv[1]) : 50000000;
  const int nrb = (int)((n + RB - 1) / RB);
  int ncb = (int)((n + CB - 1) / CB);
  ncb = (ncb + KC - 1) / KC * KC;
  const int64_t per = (int64_t)nrb * CELL;  // entries per column block
  const int64_t E = per * ncb;
  printf("n=%lld RB=%d CB=%d nrb=%d ncb=%d cell=%d chunk=%d entries=%.3e\n", (long long)n, RB, CB, nrb, ncb, CELL, CHUNK,
         (double)E);
  double *val, *prod, *x, *y;
  uint16_t* coloff;
  uint32_t* words;
  CK(cudaMalloc(&val, E * 8));
  CK(cudaMalloc(&prod, E * 8));
  CK(cudaMalloc(&coloff, E * 2));
  CK(cudaMalloc(&words, E * 4));
  CK(cudaMalloc(&x, (int64_t)ncb * CB * 8));
  CK(cudaMalloc(&y, (int64_t)nrb * RB * 8));
  k_init<<<4096, 256>>>(E, val, coloff, (int64_t)ncb * CB, x);
  k_words<<<4096, 256>>>(E, words);
  CK(cudaDeviceSynchronize());
  const int sm1 = CB * 8, sm2 = RB * 8 + CHUNK * 24;
  CK(cudaFuncSetAttribute(k_expand, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1));
  CK(cudaFuncSetAttribute(k_combine, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2));
  int o1 = 0, o2 = 0;
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o1, k_expand, P1T, sm1));
  CK(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o2, k_combine, P2T, sm2));
  printf("occupancy: expand %d CTA/SM (%d B smem), combine %d CTA/SM (%d B smem)\n", o1, sm1, o2, sm2);
  cudaEvent_t a, b, c;
  CK(cudaEventCreate(&a));
  CK(cudaEventCreate(&b));
  CK(cudaEventCreate(&c));
  float t1 = 0, t2 = 0;
  const int iters = 10;
  for (int it = -2; it < iters; ++it) {
    CK(cudaEventRecord(a));
    k_expand<<<ncb, P1T, sm1>>>(n, per, x, val, coloff, prod);
    CK(cudaEventRecord(b));
    k_combine<<<nrb, P2T, sm2>>>(n, nrb, ncb, prod, words, y);
    CK(cudaEventRecord(c));
    CK(cudaEventSynchronize(c));
    float x1, x2;
    CK(cudaEventElapsedTime(&x1, a, b));
    CK(cudaEventElapsedTime(&x2, b, c));
    if (it >= 0) { t1 += x1; t2 += x2; }
  }
  CK(cudaGetLastError());
  t1 /= iters; t2 /= iters;
  const double b1 = (double)E * 18 + ncb * (double)CB * 8, b2 = (double)E * 12 + (double)nrb * RB * 8;
  printf("expand  %.3f ms  %.0f GB/s (%.2f GB)\n", t1, b1 / t1 / 1e6, b1 / 1e9);
  printf("combine %.3f ms  %.0f GB/s (%.2f GB)\n", t2, b2 / t2 / 1e6, b2 / 1e9);
  printf("total   %.3f ms  -> %.1f GFLOP/s at 2*%.3e flops\n", t1 + t2, 2.0 * E / (t1 + t2) / 1e6, (double)E);
  return 0;
}
#endif  // BB_NO_MAIN
