// spmv.cu — CSR SpMV y = A x (K7 in SURVEY.md §2.2) and COO SpMV (K9).
//
// Reference: spmv_csr / _accumulate_rows (kernels.py:59-78): per-row sums of
// values[k] * x[col_idx[k]]; spmv_coo (kernels.py:81-86).
//
// SpMV moves B = nnz*(s_v + s_i) + (M+1)*s_p + N*s_v + M*s_v bytes for 2*nnz
// flops: it is HBM-bound on B200 (0.17 flop/B).  Two kernels:
//
//  * k_spmv_merge — nnz+row balanced ("merge-path") tiles.  A per-matrix plan
//    stores the (row, nnz) split point of every tile on the merge path of
//    row-ends and nonzero positions, so every CTA gets exactly TILE items no
//    matter how ragged the rows are (power-law, empty rows).  Phase A streams
//    the tile's col_idx / values with 128-bit L1-bypassing evict-first loads,
//    gathers x with evict-last (x stays L2-resident) and parks the products in
//    shared memory; phase B walks the merge path per thread, emits row sums and
//    combines the partial rows across threads with a segmented block scan;
//    rows spanning tiles are finished by a tiny deterministic fix-up kernel
//    (carries summed in tile order).  Deterministic for a given matrix.
//  * k_spmv_vector — CSR-vector: L lanes per row (L = 1..32), lane-strided
//    sums + butterfly shuffle.  The order of a row's reduction depends only on
//    L, so any row partition is bitwise equal to the whole-matrix call (the
//    analogue of spmv_csr_parallel's bitwise guarantee, kernels.py:1-6).
#include "common.cuh"

namespace sme {

constexpr int M_NT = 256;
constexpr int M_IPT = 8;
constexpr int M_TILE = M_NT * M_IPT;              // merge items (rows + nnz) per tile
constexpr int M_QG = (M_TILE / 4 + 2 + M_NT - 1) / M_NT;  // 4-element groups per thread

template <typename T> struct V4;
template <> struct V4<double> {
  static __device__ __forceinline__ void load(const double* p, uint64_t pol, double v[4]) {
    double2 a = ld_stream_d2(reinterpret_cast<const double2*>(p), pol);
    double2 b = ld_stream_d2(reinterpret_cast<const double2*>(p) + 1, pol);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
};
template <> struct V4<float> {
  static __device__ __forceinline__ void load(const float* p, uint64_t pol, float v[4]) {
    float4 a = ld_stream_f4(reinterpret_cast<const float4*>(p), pol);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  }
};

template <typename T>
__global__ void __launch_bounds__(M_NT) k_spmv_merge(int32_t n_rows, int32_t nnz, const int32_t* __restrict__ row_ptr,
                                                     const int32_t* __restrict__ col, const T* __restrict__ val,
                                                     const T* __restrict__ x, T* __restrict__ y,
                                                     const int2* __restrict__ plan, T* __restrict__ carry_val,
                                                     int32_t* __restrict__ carry_row, int accumulate) {
  __shared__ T s_prod[M_TILE];
  __shared__ int32_t s_end[M_TILE];
  __shared__ int32_t s_wkey[M_NT / 32], s_wfirst[M_NT / 32];
  __shared__ T s_wval[M_NT / 32];
  __shared__ int32_t s_pkey[M_NT / 32];
  __shared__ T s_pval[M_NT / 32];

  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int t = blockIdx.x;
  const int2 c0 = plan[t], c1 = plan[t + 1];
  const int r0 = c0.x, j0 = c0.y;
  const int nr = c1.x - r0, nj = c1.y - j0;
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();

  // ---- phase A: row ends + products -------------------------------------
  for (int i = tid; i < nr; i += M_NT) s_end[i] = ld_stream_i1(row_ptr + r0 + 1 + i, pol_stream);

  const int j1 = j0 + nj;
  const int gA = j0 >> 2, gB = (j1 + 3) >> 2;
  int cidx[M_QG][4];
  T cv[M_QG][4];
#pragma unroll
  for (int q = 0; q < M_QG; ++q) {
    const int g = gA + tid + q * M_NT;
    const int e = g * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i) { cidx[q][i] = -1; cv[q][i] = T(0); }
    if (g < gB) {
      if (e + 3 < nnz) {
        int4 c = ld_stream_i4(reinterpret_cast<const int4*>(col + e), pol_stream);
        cidx[q][0] = c.x; cidx[q][1] = c.y; cidx[q][2] = c.z; cidx[q][3] = c.w;
        V4<T>::load(val + e, pol_stream, cv[q]);
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i)
          if (e + i < nnz) { cidx[q][i] = col[e + i]; cv[q][i] = val[e + i]; }
      }
#pragma unroll
      for (int i = 0; i < 4; ++i)
        if (e + i < j0 || e + i >= j1) cidx[q][i] = -1;
    }
  }
  T xv[M_QG][4];
#pragma unroll
  for (int q = 0; q < M_QG; ++q)
#pragma unroll
    for (int i = 0; i < 4; ++i) xv[q][i] = cidx[q][i] >= 0 ? ld_keep(x + cidx[q][i], pol_keep) : T(0);
#pragma unroll
  for (int q = 0; q < M_QG; ++q) {
    const int e = (gA + tid + q * M_NT) * 4;
#pragma unroll
    for (int i = 0; i < 4; ++i)
      if (cidx[q][i] >= 0) s_prod[e + i - j0] = cv[q][i] * xv[q][i];
  }
  __syncthreads();

  // ---- phase B: per-thread merge path ----------------------------------
  const int total = nr + nj;
  const int d0 = min(tid * M_IPT, total), d1 = min(d0 + M_IPT, total);
  int lo = max(0, d0 - nj), hi = min(d0, nr);
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (s_end[mid] <= j0 + d0 - 1 - mid) lo = mid + 1; else hi = mid;
  }
  int i = lo, j = d0 - lo;
  T run = T(0);
  int first_row = -1;
  T first_val = T(0);
#pragma unroll
  for (int s = 0; s < M_IPT; ++s) {
    if (d0 + s < d1) {
      if (i < nr && (j >= nj || s_end[i] <= j0 + j)) {
        if (first_row < 0) {
          first_row = i;
          first_val = run;
        } else {
          T* yp = y + r0 + i;
          *yp = accumulate ? *yp + run : run;
        }
        run = T(0);
        ++i;
      } else {
        run += s_prod[j];
        ++j;
      }
    }
  }

  // ---- segmented inclusive scan of (key = open local row, run) ---------
  int key = i;
  T v = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int ok = __shfl_up_sync(0xffffffffu, key, o);
    T ov = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o && ok == key) v += ov;
  }
  const int key_lane0 = __shfl_sync(0xffffffffu, key, 0);
  if (lane == 31) { s_wkey[warp] = key; s_wval[warp] = v; }
  if (lane == 0) s_wfirst[warp] = key;
  __syncthreads();
  if (tid == 0) {
    // exclusive prefix over warps: P_w = combine(warp totals 0..w-1)
    int pk = -1;
    T pv = T(0);
    for (int w = 0; w < M_NT / 32; ++w) {
      s_pkey[w] = pk;
      s_pval[w] = pv;
      const int wk = s_wkey[w];
      const T wv = s_wval[w];
      if (pk == wk && s_wfirst[w] == wk) pv = pv + wv; else pv = wv;
      pk = wk;
    }
  }
  __syncthreads();
  const int pk = s_pkey[warp];
  const T pv = s_pval[warp];
  if (warp > 0 && pk == key && key_lane0 == key) v = pv + v;  // block-inclusive
  // previous thread's block-inclusive value
  int prev_key = __shfl_up_sync(0xffffffffu, key, 1);
  T prev_v = __shfl_up_sync(0xffffffffu, v, 1);
  if (lane == 0) { prev_key = warp > 0 ? pk : -1; prev_v = warp > 0 ? pv : T(0); }
  if (first_row >= 0) {
    T tot = (prev_key == first_row) ? prev_v + first_val : first_val;
    T* yp = y + r0 + first_row;
    *yp = accumulate ? *yp + tot : tot;
  }
  if (tid == M_NT - 1) {
    // carry of the tile's open row (row r0 + nr), if it has elements here
    const bool has = (key == nr) && (nj > 0) && (nr == 0 || j1 > s_end[nr - 1]);
    carry_row[t] = has ? r0 + nr : -1;
    carry_val[t] = has ? v : T(0);
  }
}

template <typename T>
__global__ void k_spmv_fixup(int64_t n_tiles, const int2* __restrict__ plan, const int32_t* __restrict__ carry_row,
                             const T* __restrict__ carry_val, T* __restrict__ y) {
  for (int64_t t = 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t < n_tiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int r0 = plan[t].x;
    if (plan[t + 1].x == r0) continue;  // the tile closes no row
    if (carry_row[t - 1] != r0) continue;
    int64_t f = t - 1;
    while (f > 0 && carry_row[f - 1] == r0) --f;
    T s = carry_val[f];
    for (int64_t u = f + 1; u < t; ++u) s += carry_val[u];
    y[r0] += s;
  }
}

// tile split points on the merge path of A = row ends (row_ptr[1..M]) and B = 0..nnz-1
__global__ void k_spmv_plan(int64_t n_tiles, int32_t n_rows, int32_t nnz, const int32_t* __restrict__ row_ptr,
                            int2* __restrict__ plan) {
  for (int64_t t = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; t <= n_tiles;
       t += (int64_t)gridDim.x * blockDim.x) {
    const int64_t d = min(t * (int64_t)M_TILE, (int64_t)n_rows + nnz);
    int64_t lo = max((int64_t)0, d - nnz), hi = min(d, (int64_t)n_rows);
    while (lo < hi) {
      int64_t mid = (lo + hi) >> 1;
      if ((int64_t)row_ptr[mid + 1] <= d - 1 - mid) lo = mid + 1; else hi = mid;
    }
    plan[t] = make_int2((int)lo, (int)(d - lo));
  }
}

// CSR-vector: L lanes per row; warp-uniform loop over blocks of 32/L rows.
template <typename T, int L>
__global__ void __launch_bounds__(256) k_spmv_vector(int64_t n_rows, const int32_t* __restrict__ row_ptr,
                                                     const int32_t* __restrict__ col, const T* __restrict__ val,
                                                     const T* __restrict__ x, T* __restrict__ y, int accumulate) {
  constexpr int RPW = 32 / L;  // rows per warp step
  const int lane = threadIdx.x & 31;
  const int sub = lane / L, li = lane % L;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  for (int64_t base = warp * RPW; base < n_rows; base += n_warps * RPW) {
    const int64_t r = base + sub;
    T s = T(0);
    if (r < n_rows) {
      const int32_t a = row_ptr[r], b = row_ptr[r + 1];
      for (int32_t k = a + li; k < b; k += L)
        s += ld_stream(val + k, pol_stream) * ld_keep(x + ld_stream_i1(col + k, pol_stream), pol_keep);
    }
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (r < n_rows && li == 0) y[r] = accumulate ? y[r] + s : s;
  }
}

// numpy's pairwise summation (loops_utils.h.src: pairwise_sum) over the
// products of positions [s, s+n), each product separately rounded.
__device__ double pw_sum(const int32_t* __restrict__ col, const double* __restrict__ val,
                         const double* __restrict__ x, int64_t s, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, __dmul_rn(val[s + i], x[col[s + i]]));
    return res;
  } else if (n <= 128) {
    double r[8];
#pragma unroll
    for (int q = 0; q < 8; ++q) r[q] = __dmul_rn(val[s + q], x[col[s + q]]);
    int64_t i;
    for (i = 8; i < n - (n % 8); i += 8) {
#pragma unroll
      for (int q = 0; q < 8; ++q) r[q] = __dadd_rn(r[q], __dmul_rn(val[s + i + q], x[col[s + i + q]]));
    }
    double res = __dadd_rn(__dadd_rn(__dadd_rn(r[0], r[1]), __dadd_rn(r[2], r[3])),
                           __dadd_rn(__dadd_rn(r[4], r[5]), __dadd_rn(r[6], r[7])));
    for (; i < n; ++i) res = __dadd_rn(res, __dmul_rn(val[s + i], x[col[s + i]]));
    return res;
  } else {
    int64_t n2 = n / 2;
    n2 -= n2 % 8;
    return __dadd_rn(pw_sum(col, val, x, s, n2), pw_sum(col, val, x, s + n2, n - n2));
  }
}

__global__ void k_spmv_reduceat_exact(int64_t n_rows, const int32_t* __restrict__ row_ptr,
                                      const int32_t* __restrict__ col, const double* __restrict__ val,
                                      const double* __restrict__ x, double* __restrict__ y) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t a = row_ptr[r], b = row_ptr[r + 1];
    double acc = 0.0;
    if (b > a) acc = __dadd_rn(__dmul_rn(val[a], x[col[a]]), pw_sum(col, val, x, a + 1, b - a - 1));
    y[r] = acc;
  }
}

template <typename T>
__global__ void k_spmv_coo(int64_t nnz, const int32_t* __restrict__ row, const int32_t* __restrict__ col,
                           const T* __restrict__ val, const T* __restrict__ x, T* __restrict__ y) {
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(y + row[k], val[k] * x[col[k]]);
}

template <typename T>
int launch_vector(int lanes, int64_t n_rows, const int32_t* rp, const int32_t* col, const T* val, const T* x, T* y,
                  int acc, cudaStream_t s) {
  const int64_t threads = n_rows * lanes;
  const int blocks = grid_for(threads, 256, 8);
  switch (lanes) {
    case 1: k_spmv_vector<T, 1><<<blocks, 256, 0, s>>>(n_rows, rp, col, val, x, y, acc); break;
    case 2: k_spmv_vector<T, 2><<<blocks, 256, 0, s>>>(n_rows, rp, col, val, x, y, acc); break;
    case 4: k_spmv_vector<T, 4><<<blocks, 256, 0, s>>>(n_rows, rp, col, val, x, y, acc); break;
    case 8: k_spmv_vector<T, 8><<<blocks, 256, 0, s>>>(n_rows, rp, col, val, x, y, acc); break;
    case 16: k_spmv_vector<T, 16><<<blocks, 256, 0, s>>>(n_rows, rp, col, val, x, y, acc); break;
    case 32: k_spmv_vector<T, 32><<<blocks, 256, 0, s>>>(n_rows, rp, col, val, x, y, acc); break;
    default: SME_REQUIRE(false, "lanes must be one of 1,2,4,8,16,32 (got %d)", lanes);
  }
  SME_CHECK_LAUNCH("k_spmv_vector");
  return SME_OK;
}

}  // namespace sme

using namespace sme;

SME_API int sme_spmv_merge_tiles(int64_t n_rows, int64_t nnz, int64_t* n_tiles) {
  SME_REQUIRE(n_tiles && n_rows >= 0 && nnz >= 0, "bad arguments");
  *n_tiles = (n_rows + nnz + M_TILE - 1) / M_TILE;
  return SME_OK;
}

SME_API int sme_spmv_merge_plan(int64_t n_rows, int64_t nnz, const int32_t* row_ptr, int32_t* plan,
                                sme_stream_t stream) {
  SME_REQUIRE(n_rows >= 0 && n_rows < INT32_MAX && nnz >= 0 && nnz < INT32_MAX, "sizes exceed int32");
  const int64_t n_tiles = (n_rows + nnz + M_TILE - 1) / M_TILE;
  cudaStream_t s = as_stream(stream);
  k_spmv_plan<<<grid_for(n_tiles + 1, 256), 256, 0, s>>>(n_tiles, (int32_t)n_rows, (int32_t)nnz, row_ptr,
                                                         reinterpret_cast<int2*>(plan));
  SME_CHECK_LAUNCH("k_spmv_plan");
  return SME_OK;
}

SME_API int sme_spmv_merge_carry_bytes(int dtype, int64_t n_tiles, size_t* bytes) {
  SME_REQUIRE(bytes && n_tiles >= 0, "bad arguments");
  *bytes = align_up((size_t)n_tiles * 8) + align_up((size_t)n_tiles * 4);
  return SME_OK;
}

SME_API int sme_spmv_merge(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* row_ptr,
                           const int32_t* col, const void* val, const void* x, void* y, const int32_t* plan,
                           int64_t n_tiles, void* carry, int accumulate, sme_stream_t stream) {
  SME_REQUIRE(n_rows >= 0 && n_rows < INT32_MAX && nnz >= 0 && nnz < INT32_MAX, "sizes exceed int32");
  SME_REQUIRE(n_tiles == (n_rows + nnz + M_TILE - 1) / M_TILE, "plan was built for another shape");
  SME_REQUIRE(((uintptr_t)col & 15) == 0 && ((uintptr_t)val & 15) == 0,
              "col_idx and values must be 16-byte aligned");
  if (n_tiles == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  const int2* pl = reinterpret_cast<const int2*>(plan);
  char* cb = (char*)carry;
  int32_t* carry_row = (int32_t*)(cb + align_up((size_t)n_tiles * 8));
  if (dtype == SME_F64) {
    double* cval = (double*)cb;
    k_spmv_merge<double><<<(unsigned)n_tiles, M_NT, 0, s>>>((int32_t)n_rows, (int32_t)nnz, row_ptr, col,
                                                            (const double*)val, (const double*)x, (double*)y, pl,
                                                            cval, carry_row, accumulate);
    SME_CHECK_LAUNCH("k_spmv_merge");
    if (n_tiles > 1) {
      k_spmv_fixup<double><<<grid_for(n_tiles, 256), 256, 0, s>>>(n_tiles, pl, carry_row, cval, (double*)y);
      SME_CHECK_LAUNCH("k_spmv_fixup");
    }
  } else if (dtype == SME_F32) {
    float* cval = (float*)cb;
    k_spmv_merge<float><<<(unsigned)n_tiles, M_NT, 0, s>>>((int32_t)n_rows, (int32_t)nnz, row_ptr, col,
                                                          (const float*)val, (const float*)x, (float*)y, pl, cval,
                                                          carry_row, accumulate);
    SME_CHECK_LAUNCH("k_spmv_merge");
    if (n_tiles > 1) {
      k_spmv_fixup<float><<<grid_for(n_tiles, 256), 256, 0, s>>>(n_tiles, pl, carry_row, cval, (float*)y);
      SME_CHECK_LAUNCH("k_spmv_fixup");
    }
  } else {
    SME_REQUIRE(false, "unknown dtype %d", dtype);
  }
  return SME_OK;
}

SME_API int sme_spmv_vector(int dtype, int lanes, int64_t n_rows, int64_t n_cols, const int32_t* row_ptr,
                            const int32_t* col, const void* val, const void* x, void* y, int accumulate,
                            sme_stream_t stream) {
  SME_REQUIRE(n_rows >= 0 && n_rows < INT32_MAX, "n_rows exceeds int32");
  if (n_rows == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == SME_F64)
    return launch_vector<double>(lanes, n_rows, row_ptr, col, (const double*)val, (const double*)x, (double*)y,
                                 accumulate, s);
  if (dtype == SME_F32)
    return launch_vector<float>(lanes, n_rows, row_ptr, col, (const float*)val, (const float*)x, (float*)y,
                                accumulate, s);
  SME_REQUIRE(false, "unknown dtype %d", dtype);
}

SME_API int sme_spmv_reduceat_exact(int64_t n_rows, const int32_t* row_ptr, const int32_t* col, const double* val,
                                    const double* x, double* y, sme_stream_t stream) {
  if (n_rows == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  k_spmv_reduceat_exact<<<grid_for(n_rows, 128, 16), 128, 0, s>>>(n_rows, row_ptr, col, val, x, y);
  SME_CHECK_LAUNCH("k_spmv_reduceat_exact");
  return SME_OK;
}

SME_API int sme_spmv_coo(int dtype, int64_t n_rows, int64_t nnz, const int32_t* row, const int32_t* col,
                         const void* val, const void* x, void* y, sme_stream_t stream) {
  cudaStream_t s = as_stream(stream);
  size_t vs = dtype == SME_F64 ? 8 : 4;
  SME_REQUIRE(dtype == SME_F64 || dtype == SME_F32, "unknown dtype %d", dtype);
  if (n_rows > 0) SME_CUDA(cudaMemsetAsync(y, 0, (size_t)n_rows * vs, s));
  if (nnz == 0) return SME_OK;
  if (dtype == SME_F64)
    k_spmv_coo<double><<<grid_for(nnz, 256), 256, 0, s>>>(nnz, row, col, (const double*)val, (const double*)x,
                                                          (double*)y);
  else
    k_spmv_coo<float><<<grid_for(nnz, 256), 256, 0, s>>>(nnz, row, col, (const float*)val, (const float*)x,
                                                         (float*)y);
  SME_CHECK_LAUNCH("k_spmv_coo");
  return SME_OK;
}
