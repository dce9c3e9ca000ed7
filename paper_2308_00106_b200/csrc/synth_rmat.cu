// synth_rmat.cu — R-MAT edge generator for C3 (BASELINE.json configs[2]:
// "R-MAT power-law graph 16M rows ~256M nnz fp32 (no dense rows)").
//
// Edge e of a scale-s R-MAT picks, at each of the s levels, one quadrant with
// probabilities (a, b, c, 1-a-b-c) from u = U[0,1)(hash3(seed, e, level)):
// u < a -> (0,0), < a+b -> (0,1), < a+b+c -> (1,0), else (1,1); the row/col
// bits are appended most significant first.  Dedupe and the degree cap run
// through the CSR builder (sme_coo_to_csr_dedup + sme_csr_compact), and values
// are assigned per (row, slot) afterwards (k_row_values).  The numpy
// restatement is oracle.rmat_edges / oracle.row_values.
#include "common.cuh"
#include "hash.cuh"

#include "../../include/sme_synth.h"

namespace sme {

__global__ void k_rmat_edges(int64_t n_edges, int32_t scale, double a, double ab, double abc, uint64_t seed,
                             int32_t* __restrict__ row, int32_t* __restrict__ col) {
  for (int64_t e = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; e < n_edges; e += (int64_t)gridDim.x * blockDim.x) {
    uint32_t r = 0, c = 0;
    for (int lvl = 0; lvl < scale; ++lvl) {
      const double u = unit01(hash3(seed, (uint64_t)e, (uint64_t)lvl));
      const uint32_t rb = u >= ab;                         // quadrants (1,0), (1,1)
      const uint32_t cb = (u >= a && u < ab) || u >= abc;  // quadrants (0,1), (1,1)
      r = (r << 1) | rb;
      c = (c << 1) | cb;
    }
    row[e] = (int32_t)r;
    col[e] = (int32_t)c;
  }
}

// val[k] for the s-th entry of row r = U[-1,1)(hash3(seed ^ VAL_SALT, r, s))
template <typename T>
__global__ void k_row_values(int64_t n_rows, const int32_t* __restrict__ row_ptr, uint64_t seed, T* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_rows; r += n_warps) {
    const int32_t a = row_ptr[r], b = row_ptr[r + 1];
    for (int32_t k = a + lane; k < b; k += 32)
      val[k] = (T)unit_pm1(hash3(seed ^ VAL_SALT, (uint64_t)r, (uint64_t)(k - a)));
  }
}

}  // namespace sme

using namespace sme;

SME_API int sme_synth_rmat_edges(int64_t n_edges, int32_t scale, double a, double b, double c, uint64_t seed,
                                 int32_t* row, int32_t* col, sme_stream_t stream) {
  SME_REQUIRE(scale >= 1 && scale <= 30, "scale must lie in [1, 30]");
  SME_REQUIRE(n_edges >= 0 && n_edges < INT32_MAX, "edge count exceeds int32");
  SME_REQUIRE(a >= 0 && b >= 0 && c >= 0 && a + b + c <= 1.0, "bad R-MAT probabilities");
  if (n_edges == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  k_rmat_edges<<<grid_for(n_edges, 256), 256, 0, s>>>(n_edges, scale, a, a + b, a + b + c, seed, row, col);
  SME_CHECK_LAUNCH("k_rmat_edges");
  return SME_OK;
}

SME_API int sme_synth_row_values(int dtype, int64_t n_rows, const int32_t* row_ptr, uint64_t seed, void* val,
                                 sme_stream_t stream) {
  if (n_rows == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == SME_F64)
    k_row_values<double><<<grid_for(n_rows * 32, 256), 256, 0, s>>>(n_rows, row_ptr, seed, (double*)val);
  else if (dtype == SME_F32)
    k_row_values<float><<<grid_for(n_rows * 32, 256), 256, 0, s>>>(n_rows, row_ptr, seed, (float*)val);
  else
    SME_REQUIRE(false, "unknown dtype %d", dtype);
  SME_CHECK_LAUNCH("k_row_values");
  return SME_OK;
}

namespace sme {
// Lazy module loading (CUDA 12 default) loads this file's module on the first launch of
// any of its kernels, ~10-20 ms each; sme_preload() does it ahead of time.
int preload_synth_rmat() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)k_rmat_edges) == cudaSuccess ? 0 : -1;
}
}  // namespace sme
