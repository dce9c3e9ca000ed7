// split_bench.cu — can the L2-gather SpMV (request-port bound) and the binned
// expand/combine (HBM bound) run side by side on the same SMs and add up?
// Standalone timing tool: a seg-probe-like pull kernel (12 B/entry stream + one
// random 8-B gather per entry from a 50 MB x slice) and the binned kernels of
// binned_bench.cu, alone and concurrently on two streams.
//
//   nvcc -gencode arch=compute_100a,code=sm_100a -O3 -o split_bench split_bench.cu
#define BB_NO_MAIN
#include "binned_bench.cu"

#ifndef PULL_CTAS
#define PULL_CTAS 3
#endif

__global__ void __launch_bounds__(256) k_pull(int64_t E, const uint32_t* __restrict__ pk, const double* __restrict__ val,
                                              const double* __restrict__ xs, double* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * 256 + threadIdx.x) >> 5, nw = ((int64_t)gridDim.x * 256) >> 5;
  const int64_t chunks = E / 128;
  const int64_t c0 = warp * chunks / nw, c1 = (warp + 1) * chunks / nw;
  for (int64_t c = c0; c < c1; ++c) {
    const int64_t e = c * 128 + 4 * lane;
    const uint4 q = __ldcs(reinterpret_cast<const uint4*>(pk + e));
    const double2 a = __ldcs(reinterpret_cast<const double2*>(val + e));
    const double2 b = __ldcs(reinterpret_cast<const double2*>(val + e) + 1);
    const double s = a.x * __ldg(xs + q.x) + a.y * __ldg(xs + q.y) + b.x * __ldg(xs + q.z) + b.y * __ldg(xs + q.w);
    y[c * 32 + lane] = s;
  }
}

__global__ void k_init_pull(int64_t E, uint32_t* pk, double* val, uint32_t nx) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < E; i += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t h = hash32((uint32_t)i * 0x9E3779B1u + 17u);
    pk[i] = (uint32_t)(((uint64_t)hash32(h) * nx) >> 32);
    val[i] = (double)(h & 0xFFFF) / 65536.0;
  }
}

int main(int argc, char** argv) {
  const double f = argc > 1 ? atof(argv[1]) : 0.4;  // binned fraction of the 1e9 entries
  const int64_t n = 50000000, total = 1000000000;
  const uint32_t nx = 6250000;  // 50 MB x slice
  const int64_t Ep = ((int64_t)((1.0 - f) * total) / 128) * 128;
  // binned part: columns [0, f n)
  const int64_t nb_cols = (int64_t)(f * n);
  const int nrb = (int)((n + RB - 1) / RB);
  int ncb = (int)((nb_cols + CB - 1) / CB);
  ncb = (ncb + KC - 1) / KC * KC;
  const int64_t per = (int64_t)nrb * CELL;
  const int64_t Eb = per * ncb;
  printf("f=%.2f pull entries %.3e, binned entries %.3e (ncb=%d), PULL_CTAS=%d P1T=%d\n", f, (double)Ep, (double)Eb, ncb,
         PULL_CTAS, P1T);
  uint32_t *pk, *words;
  double *pv, *xs, *yp, *val, *prod, *x, *y;
  uint16_t* coloff;
  CK(cudaMalloc(&pk, Ep * 4));
  CK(cudaMalloc(&pv, Ep * 8));
  CK(cudaMalloc(&xs, (int64_t)nx * 8));
  CK(cudaMalloc(&yp, Ep / 4 * 8));
  CK(cudaMalloc(&val, Eb * 8));
  CK(cudaMalloc(&prod, Eb * 8));
  CK(cudaMalloc(&coloff, Eb * 2));
  CK(cudaMalloc(&words, Eb * 4));
  CK(cudaMalloc(&x, (int64_t)ncb * CB * 8));
  CK(cudaMalloc(&y, (int64_t)nrb * RB * 8));
  k_init_pull<<<4096, 256>>>(Ep, pk, pv, nx);
  k_init<<<4096, 256>>>(Eb, val, coloff, (int64_t)ncb * CB, x);
  k_init<<<4096, 256>>>(nx, pv, coloff, nx, xs);  // x slice values (overwrites the first nx of pv/coloff harmlessly)
  k_words<<<4096, 256>>>(Eb, words);
  CK(cudaDeviceSynchronize());
  const int sm1 = CB * 8, sm2 = RB * 8 + CHUNK * 24;
  CK(cudaFuncSetAttribute(k_expand, cudaFuncAttributeMaxDynamicSharedMemorySize, sm1));
  CK(cudaFuncSetAttribute(k_combine, cudaFuncAttributeMaxDynamicSharedMemorySize, sm2));
  int sms = 0;
  CK(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, 0));
  cudaStream_t s1, s2;
  CK(cudaStreamCreateWithFlags(&s1, cudaStreamNonBlocking));
  CK(cudaStreamCreateWithFlags(&s2, cudaStreamNonBlocking));
  cudaEvent_t e0, e1, e2, e3;
  CK(cudaEventCreate(&e0));
  CK(cudaEventCreate(&e1));
  CK(cudaEventCreate(&e2));
  CK(cudaEventCreate(&e3));
  auto pull = [&](cudaStream_t s) { k_pull<<<sms * PULL_CTAS, 256, 0, s>>>(Ep, pk, pv, xs, yp); };
  auto expand = [&](cudaStream_t s) { k_expand<<<ncb, P1T, sm1, s>>>(n, per, x, val, coloff, prod); };
  auto combine = [&](cudaStream_t s) { k_combine<<<nrb, P2T, sm2, s>>>(n, nrb, ncb, prod, words, y); };
  auto timeit = [&](const char* name, auto body) {
    float best = 1e9;
    for (int it = 0; it < 6; ++it) {
      CK(cudaEventRecord(e0, s1));
      CK(cudaStreamWaitEvent(s2, e0));
      body();
      CK(cudaEventRecord(e1, s2));
      CK(cudaStreamWaitEvent(s1, e1));
      CK(cudaEventRecord(e2, s1));
      CK(cudaEventSynchronize(e2));
      float ms;
      CK(cudaEventElapsedTime(&ms, e0, e2));
      if (it >= 2) best = ms < best ? ms : best;
    }
    CK(cudaGetLastError());
    printf("  %-28s %.3f ms\n", name, best);
    return best;
  };
  timeit("pull alone", [&] { pull(s1); });
  timeit("expand alone", [&] { expand(s2); });
  timeit("combine alone", [&] { combine(s2); });
  timeit("expand+combine", [&] { expand(s2); combine(s2); });
  timeit("pull || expand", [&] { pull(s1); expand(s2); });
  timeit("pull || expand+combine", [&] { pull(s1); expand(s2); combine(s2); });
  timeit("expand+combine || pull", [&] { expand(s2); combine(s2); pull(s1); });
  return 0;
}
