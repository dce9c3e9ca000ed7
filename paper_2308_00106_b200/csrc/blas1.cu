// blas1.cu — device vector kernels for the iterative drivers (C5: power
// iteration / CG on the permuted matrix).
//
// Every scalar (dot products, alpha, beta, norms) stays in device memory, so
// one solver iteration is a fixed sequence of launches with no host
// synchronisation and can be captured in a CUDA graph.  Reductions use a fixed
// grid and a fixed combine order: results are deterministic run to run.
#include "common.cuh"

namespace sme {

constexpr int B_NT = 256;
constexpr int B_BLOCKS = 1024;  // fixed reduction grid (deterministic partials)

__device__ __forceinline__ double block_sum(double v) {
  __shared__ double s[B_NT / 32];
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if ((threadIdx.x & 31) == 0) s[threadIdx.x >> 5] = v;
  __syncthreads();
  double t = 0.0;
  if (threadIdx.x == 0)
    for (int w = 0; w < B_NT / 32; ++w) t += s[w];
  __syncthreads();
  return t;  // valid in thread 0
}

// partial[b] = sum over the block's grid-stride share of x[i] * y[i]
template <typename T>
__global__ void __launch_bounds__(B_NT) k_dot_partial(int64_t n, const T* __restrict__ x, const T* __restrict__ y,
                                                      double* __restrict__ partial) {
  double v = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * B_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * B_NT)
    v += (double)x[i] * (double)y[i];
  v = block_sum(v);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
}

// out = sum(partial[0..nb)) in a fixed tree; optional derived scalars:
//  mode 0: out[0] = s
//  mode 1 (CG alpha):  out[0] = s (= p.Ap); alpha = rr / s -> scal[1]
//  mode 2 (CG beta):   rr_new = s; beta = rr_new / rr; rr <- rr_new -> scal[2], scal[0]
//  mode 3 (norm):      out[0] = s; scal[3] = 1 / sqrt(s)
__global__ void __launch_bounds__(B_NT) k_dot_finish(int nb, const double* __restrict__ partial, double* out,
                                                     double* scal, int mode) {
  double v = 0.0;
  for (int i = threadIdx.x; i < nb; i += B_NT) v += partial[i];
  v = block_sum(v);
  if (threadIdx.x == 0) {
    if (out) *out = v;
    if (mode == 1) scal[1] = scal[0] / v;
    if (mode == 2) { scal[2] = v / scal[0]; scal[0] = v; }
    if (mode == 3) scal[3] = 1.0 / sqrt(v);
  }
}

// CG: x += alpha p; r -= alpha Ap; partial r.r (alpha = scal[1])
template <typename T>
__global__ void __launch_bounds__(B_NT) k_cg_xr(int64_t n, T* __restrict__ x, T* __restrict__ r, const T* __restrict__ p,
                                                const T* __restrict__ ap, const double* __restrict__ scal,
                                                double* __restrict__ partial) {
  const double alpha = scal[1];
  double v = 0.0;
  for (int64_t i = (int64_t)blockIdx.x * B_NT + threadIdx.x; i < n; i += (int64_t)gridDim.x * B_NT) {
    x[i] = (T)((double)x[i] + alpha * (double)p[i]);
    const double ri = (double)r[i] - alpha * (double)ap[i];
    r[i] = (T)ri;
    v += ri * ri;
  }
  v = block_sum(v);
  if (threadIdx.x == 0) partial[blockIdx.x] = v;
}

// CG: p = r + beta p (beta = scal[2])
template <typename T>
__global__ void k_cg_p(int64_t n, T* __restrict__ p, const T* __restrict__ r, const double* __restrict__ scal) {
  const double beta = scal[2];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    p[i] = (T)((double)r[i] + beta * (double)p[i]);
}

// y = x * scal[idx]
template <typename T>
__global__ void k_scale(int64_t n, T* __restrict__ y, const T* __restrict__ x, const double* __restrict__ scal, int idx) {
  const double a = scal[idx];
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (T)((double)x[i] * a);
}

// y = a * x + b * y with host scalars
template <typename T>
__global__ void k_axpby(int64_t n, double a, const T* __restrict__ x, double b, T* __restrict__ y) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x)
    y[i] = (T)(a * (double)x[i] + b * (double)y[i]);
}

}  // namespace sme

using namespace sme;

#define DISPATCH_T(dtype, CALL_F64, CALL_F32)                          \
  do {                                                                 \
    if ((dtype) == SME_F64) { CALL_F64; }                              \
    else if ((dtype) == SME_F32) { CALL_F32; }                         \
    else SME_REQUIRE(false, "unknown dtype %d", (int)(dtype));         \
  } while (0)

SME_API int sme_blas_partials(int64_t* n_partials) {
  SME_REQUIRE(n_partials, "null pointer");
  *n_partials = B_BLOCKS;
  return SME_OK;
}

// out[0] = x . y (f64 accumulation; deterministic); `partial` holds B_BLOCKS doubles
SME_API int sme_dot(int dtype, int64_t n, const void* x, const void* y, double* partial, double* out, double* scal,
                    int mode, sme_stream_t stream) {
  SME_REQUIRE(n >= 0 && mode >= 0 && mode <= 3, "bad arguments");
  cudaStream_t s = as_stream(stream);
  DISPATCH_T(dtype,
             (k_dot_partial<double><<<B_BLOCKS, B_NT, 0, s>>>(n, (const double*)x, (const double*)y, partial)),
             (k_dot_partial<float><<<B_BLOCKS, B_NT, 0, s>>>(n, (const float*)x, (const float*)y, partial)));
  SME_CHECK_LAUNCH("k_dot_partial");
  k_dot_finish<<<1, B_NT, 0, s>>>(B_BLOCKS, partial, out, scal, mode);
  SME_CHECK_LAUNCH("k_dot_finish");
  return SME_OK;
}

// CG update: x += alpha p, r -= alpha Ap, rr_new = r.r, beta = rr_new / rr, rr = rr_new
// (scal = [rr, alpha, beta, inv_norm] in device memory), then p = r + beta p.
SME_API int sme_cg_update(int dtype, int64_t n, void* x, void* r, void* p, const void* ap, double* scal,
                          double* partial, sme_stream_t stream) {
  cudaStream_t s = as_stream(stream);
  DISPATCH_T(dtype,
             (k_cg_xr<double><<<B_BLOCKS, B_NT, 0, s>>>(n, (double*)x, (double*)r, (const double*)p,
                                                        (const double*)ap, scal, partial)),
             (k_cg_xr<float><<<B_BLOCKS, B_NT, 0, s>>>(n, (float*)x, (float*)r, (const float*)p, (const float*)ap,
                                                       scal, partial)));
  SME_CHECK_LAUNCH("k_cg_xr");
  k_dot_finish<<<1, B_NT, 0, s>>>(B_BLOCKS, partial, nullptr, scal, 2);
  SME_CHECK_LAUNCH("k_dot_finish");
  DISPATCH_T(dtype, (k_cg_p<double><<<grid_for(n, 256), 256, 0, s>>>(n, (double*)p, (const double*)r, scal)),
             (k_cg_p<float><<<grid_for(n, 256), 256, 0, s>>>(n, (float*)p, (const float*)r, scal)));
  SME_CHECK_LAUNCH("k_cg_p");
  return SME_OK;
}

// y = x * scal[idx]
SME_API int sme_scale(int dtype, int64_t n, void* y, const void* x, const double* scal, int idx,
                      sme_stream_t stream) {
  cudaStream_t s = as_stream(stream);
  DISPATCH_T(dtype, (k_scale<double><<<grid_for(n, 256), 256, 0, s>>>(n, (double*)y, (const double*)x, scal, idx)),
             (k_scale<float><<<grid_for(n, 256), 256, 0, s>>>(n, (float*)y, (const float*)x, scal, idx)));
  SME_CHECK_LAUNCH("k_scale");
  return SME_OK;
}

// y = a x + b y
SME_API int sme_axpby(int dtype, int64_t n, double a, const void* x, double b, void* y, sme_stream_t stream) {
  cudaStream_t s = as_stream(stream);
  DISPATCH_T(dtype, (k_axpby<double><<<grid_for(n, 256), 256, 0, s>>>(n, a, (const double*)x, b, (double*)y)),
             (k_axpby<float><<<grid_for(n, 256), 256, 0, s>>>(n, a, (const float*)x, b, (float*)y)));
  SME_CHECK_LAUNCH("k_axpby");
  return SME_OK;
}

namespace sme {
// Lazy module loading (CUDA 12 default) loads this file's module on the first launch of
// any of its kernels, ~10-20 ms each; sme_preload() does it ahead of time.
int preload_blas1() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)k_dot_finish) == cudaSuccess ? 0 : -1;
}
}  // namespace sme
