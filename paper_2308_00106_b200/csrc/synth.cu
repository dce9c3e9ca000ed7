// synth.cu — deterministic device generators for the BASELINE.json configs
// (SURVEY.md §8d).  These build benchmark/test INPUTS; they are not part of the
// reference's path.  Every generator has a bit-identical numpy restatement in
// paper_2308_00106_b200/synth.py (used for sampled-row checks on the host).
//
//   C2/C5  5-point Laplacian on a g x g grid: diag 4, off-diagonals -1.
//   C4     "random-structured": every row holds k distinct uniformly random
//          columns (first k distinct of a counter-based hash stream), sorted,
//          values U[-1, 1).
#include "common.cuh"

#include "../../include/sme_synth.h"

#include "hash.cuh"

namespace sme {

// row_ptr[r] for the g x g 5-point stencil, r in [0, g*g]
__device__ __forceinline__ int64_t lap_ptr(int64_t g, int64_t r) {
  if (r >= g * g) return 5 * g * g - 4 * g;
  int64_t i = r / g, j = r % g;
  int64_t rows = i * (5 * g - 2) - (i > 0 ? g : 0);
  int64_t per = 5 - (i == 0) - (i == g - 1);
  int64_t within = j * per - (j > 0 ? 1 : 0);
  return rows + within;
}

template <typename T>
__global__ void k_laplacian(int64_t g, int32_t* __restrict__ row_ptr, int32_t* __restrict__ col, T* __restrict__ val) {
  const int64_t n = g * g;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r <= n; r += (int64_t)gridDim.x * blockDim.x) {
    int64_t p = lap_ptr(g, r);
    row_ptr[r] = (int32_t)p;
    if (r == n) continue;
    int64_t i = r / g, j = r % g;
    if (i > 0) { col[p] = (int32_t)(r - g); val[p] = T(-1); ++p; }
    if (j > 0) { col[p] = (int32_t)(r - 1); val[p] = T(-1); ++p; }
    col[p] = (int32_t)r; val[p] = T(4); ++p;
    if (j < g - 1) { col[p] = (int32_t)(r + 1); val[p] = T(-1); ++p; }
    if (i < g - 1) { col[p] = (int32_t)(r + g); val[p] = T(-1); ++p; }
  }
}

// warp per row; k <= 32 distinct columns: the first k distinct values of the
// stream cand(t) = hash3(seed, r, t) -> [0, n_cols), t = 0, 1, 2, ...
// rows != nullptr: output row i is generator row rows[i] (a row shard of the
// permuted matrix generates only the original rows it owns)
template <typename T>
__global__ void k_random_rows(int64_t n_rows, int64_t n_cols, int32_t k, uint64_t seed, const int32_t* __restrict__ rows,
                              int32_t* __restrict__ row_ptr, int32_t* __restrict__ col, T* __restrict__ val) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const unsigned lt = (1u << lane) - 1u;
  for (int64_t i = warp; i < n_rows; i += n_warps) {
    if (row_ptr && lane == 0) row_ptr[i] = (int32_t)(i * k);
    if (row_ptr && i == n_rows - 1 && lane == 0) row_ptr[n_rows] = (int32_t)(n_rows * k);
    const int64_t r = rows ? (int64_t)__ldg(rows + i) : i;
    uint32_t acc = 0xFFFFFFFFu;  // lane a holds accepted[a], a < cnt
    int cnt = 0;
    for (int round = 0; cnt < k; ++round) {
      uint64_t h = hash3(seed, (uint64_t)r, (uint64_t)round * 32 + lane);
      uint32_t cand = (uint32_t)(((h >> 32) * (uint64_t)n_cols) >> 32);
      unsigned same = __match_any_sync(0xffffffffu, cand);
      bool is_new = (same & lt) == 0;  // first occurrence in this round
      for (int a = 0; a < cnt; ++a)
        if (__shfl_sync(0xffffffffu, acc, a) == cand) is_new = false;
      unsigned nm = __ballot_sync(0xffffffffu, is_new);
      int take = min(__popc(nm), k - cnt);
      // lane p in [cnt, cnt+take) receives the (p-cnt)-th new candidate
      int src = 0;
      if (lane >= cnt && lane < cnt + take) {
        unsigned m = nm;
        for (int q = 0; q < lane - cnt; ++q) m &= m - 1u;  // drop the lower new lanes
        src = __ffs(m) - 1;
      }
      uint32_t got = __shfl_sync(0xffffffffu, cand, src);
      if (lane >= cnt && lane < cnt + take) acc = got;
      cnt += take;
    }
    // sort the k accepted columns ascending (pads = 0xFFFFFFFF sort last)
    uint32_t v = acc;
    for (int kk = 2; kk <= 32; kk <<= 1)
      for (int j = kk >> 1; j > 0; j >>= 1) {
        uint32_t o = __shfl_xor_sync(0xffffffffu, v, j);
        bool asc = (lane & kk) == 0, lower = (lane & j) == 0;
        uint32_t mn = min(v, o), mx = max(v, o);
        v = (lower == asc) ? mn : mx;
      }
    if (lane < k) {
      int64_t p = i * k + lane;
      col[p] = (int32_t)v;
      val[p] = (T)unit_pm1(hash3(seed ^ VAL_SALT, (uint64_t)r, (uint64_t)lane));
    }
  }
}

}  // namespace sme

using namespace sme;

SME_API int sme_synth_laplacian5(int dtype, int64_t g, int32_t* row_ptr, int32_t* col, void* val,
                                 sme_stream_t stream) {
  SME_REQUIRE(g >= 1 && 5 * g * g < INT32_MAX, "grid %lld out of range", (long long)g);
  cudaStream_t s = as_stream(stream);
  int blocks = grid_for(g * g + 1, 256);
  if (dtype == SME_F64)
    k_laplacian<double><<<blocks, 256, 0, s>>>(g, row_ptr, col, (double*)val);
  else if (dtype == SME_F32)
    k_laplacian<float><<<blocks, 256, 0, s>>>(g, row_ptr, col, (float*)val);
  else
    SME_REQUIRE(false, "unknown dtype %d", dtype);
  SME_CHECK_LAUNCH("k_laplacian");
  return SME_OK;
}

SME_API int sme_synth_random_rows(int dtype, int64_t n_rows, int64_t n_cols, int32_t k, uint64_t seed,
                                  int32_t* row_ptr, int32_t* col, void* val, sme_stream_t stream) {
  SME_REQUIRE(n_rows >= 1 && n_cols >= 1 && n_cols < INT32_MAX, "bad dimensions");
  SME_REQUIRE(k >= 1 && k <= 32 && k <= n_cols, "k must lie in [1, min(32, n_cols)]");
  SME_REQUIRE(!row_ptr || n_rows * k < INT32_MAX, "nnz exceeds int32 (pass row_ptr = NULL: it is r * k)");
  cudaStream_t s = as_stream(stream);
  int blocks = grid_for(n_rows * 32, 256);
  if (dtype == SME_F64)
    k_random_rows<double><<<blocks, 256, 0, s>>>(n_rows, n_cols, k, seed, nullptr, row_ptr, col, (double*)val);
  else if (dtype == SME_F32)
    k_random_rows<float><<<blocks, 256, 0, s>>>(n_rows, n_cols, k, seed, nullptr, row_ptr, col, (float*)val);
  else
    SME_REQUIRE(false, "unknown dtype %d", dtype);
  SME_CHECK_LAUNCH("k_random_rows");
  return SME_OK;
}

SME_API int sme_synth_random_rows_sel(int dtype, int64_t n_sel, const int32_t* rows, int64_t n_cols, int32_t k,
                                      uint64_t seed, int32_t* row_ptr, int32_t* col, void* val, sme_stream_t stream) {
  SME_REQUIRE(n_sel >= 1 && n_cols >= 1 && n_cols < INT32_MAX && rows != nullptr, "bad dimensions");
  SME_REQUIRE(k >= 1 && k <= 32 && k <= n_cols, "k must lie in [1, min(32, n_cols)]");
  SME_REQUIRE(n_sel * k < INT32_MAX, "nnz exceeds int32");
  cudaStream_t s = as_stream(stream);
  int blocks = grid_for(n_sel * 32, 256);
  if (dtype == SME_F64)
    k_random_rows<double><<<blocks, 256, 0, s>>>(n_sel, n_cols, k, seed, rows, row_ptr, col, (double*)val);
  else if (dtype == SME_F32)
    k_random_rows<float><<<blocks, 256, 0, s>>>(n_sel, n_cols, k, seed, rows, row_ptr, col, (float*)val);
  else
    SME_REQUIRE(false, "unknown dtype %d", dtype);
  SME_CHECK_LAUNCH("k_random_rows");
  return SME_OK;
}

namespace sme {
// Lazy module loading (CUDA 12 default) loads this file's module on the first launch of
// any of its kernels, ~10-20 ms each; sme_preload() does it ahead of time.
int preload_synth() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)k_laplacian<double>) == cudaSuccess ? 0 : -1;
}
}  // namespace sme
