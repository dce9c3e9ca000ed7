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

#include <algorithm>

namespace sme {

constexpr int M_NT = 256;
constexpr int M_IPT = 8;
constexpr int M_TILE = M_NT * M_IPT;              // merge items (rows + nnz) per tile

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

// Shared scratch of the per-tile segmented scan.
template <typename T, int NT>
struct ScanSmem {
  int32_t wkey[NT / 32], wfirst[NT / 32], pkey[NT / 32];
  T wval[NT / 32], pval[NT / 32];
};

// Phase B of a merge tile: per-thread merge-path walk over IPT items, emitting
// row sums; partial rows across threads combined by a segmented block scan;
// the tile's open row goes to the carry arrays (finished by k_spmv_fixup).
// end_at(i) = row_ptr[r0 + 1 + i] (i < nr), prod_at(j) = product of nnz j0 + j.
template <typename T, int NT, int IPT, class EndFn, class ProdFn>
__device__ __forceinline__ void merge_tile_reduce(const int t, const int r0, const int nr, const int j0, const int nj,
                                                  EndFn end_at, ProdFn prod_at, T* __restrict__ y,
                                                  const int accumulate, T* __restrict__ carry_val,
                                                  int32_t* __restrict__ carry_row, ScanSmem<T, NT>& sm) {
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int total = nr + nj;
  const int d0 = min(tid * IPT, total), d1 = min(d0 + IPT, total);
  int lo = max(0, d0 - nj), hi = min(d0, nr);
  while (lo < hi) {
    int mid = (lo + hi) >> 1;
    if (end_at(mid) <= j0 + d0 - 1 - mid) lo = mid + 1; else hi = mid;
  }
  int i = lo, j = d0 - lo;
  T run = T(0);
  int first_row = -1;
  T first_val = T(0);
  int next_end = (i < nr) ? end_at(i) : INT32_MAX;
#pragma unroll
  for (int s = 0; s < IPT; ++s) {
    if (d0 + s < d1) {
      if (i < nr && (j >= nj || next_end <= j0 + j)) {
        if (first_row < 0) {
          first_row = i;
          first_val = run;
        } else {
          T* yp = y + r0 + i;
          *yp = accumulate ? *yp + run : run;
        }
        run = T(0);
        ++i;
        next_end = (i < nr) ? end_at(i) : INT32_MAX;
      } else {
        run += prod_at(j);
        ++j;
      }
    }
  }
  // segmented inclusive scan of (key = open local row, run)
  const int key = i;
  T v = run;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int ok = __shfl_up_sync(0xffffffffu, key, o);
    T ov = __shfl_up_sync(0xffffffffu, v, o);
    if (lane >= o && ok == key) v += ov;
  }
  const int key_lane0 = __shfl_sync(0xffffffffu, key, 0);
  if (lane == 31) { sm.wkey[warp] = key; sm.wval[warp] = v; }
  if (lane == 0) sm.wfirst[warp] = key;
  __syncthreads();
  if (tid == 0) {
    int pk = -1;
    T pv = T(0);
    for (int w = 0; w < NT / 32; ++w) {
      sm.pkey[w] = pk;
      sm.pval[w] = pv;
      const int wk = sm.wkey[w];
      const T wv = sm.wval[w];
      pv = (pk == wk && sm.wfirst[w] == wk) ? pv + wv : wv;
      pk = wk;
    }
  }
  __syncthreads();
  const int pk = sm.pkey[warp];
  const T pv = sm.pval[warp];
  if (warp > 0 && pk == key && key_lane0 == key) v = pv + v;  // block-inclusive
  int prev_key = __shfl_up_sync(0xffffffffu, key, 1);
  T prev_v = __shfl_up_sync(0xffffffffu, v, 1);
  if (lane == 0) { prev_key = warp > 0 ? pk : -1; prev_v = warp > 0 ? pv : T(0); }
  if (first_row >= 0) {
    const T tot = (prev_key == first_row) ? prev_v + first_val : first_val;
    T* yp = y + r0 + first_row;
    *yp = accumulate ? *yp + tot : tot;
  }
  if (tid == NT - 1) {
    const bool has = (key == nr) && (nj > 0) && (nr == 0 || j0 + nj > end_at(nr - 1));
    carry_row[t] = has ? r0 + nr : -1;
    carry_val[t] = has ? v : T(0);
  }
}

// One CTA per tile, loads straight from global (fallback for unaligned pointers).
template <typename T>
__global__ void __launch_bounds__(M_NT) k_spmv_merge(int32_t n_rows, int32_t nnz, const int32_t* __restrict__ row_ptr,
                                                     const int32_t* __restrict__ col, const T* __restrict__ val,
                                                     const T* __restrict__ x, T* __restrict__ y,
                                                     const int2* __restrict__ plan, T* __restrict__ carry_val,
                                                     int32_t* __restrict__ carry_row, int accumulate) {
  __shared__ T s_prod[M_TILE];
  __shared__ int32_t s_end[M_TILE];
  __shared__ ScanSmem<T, M_NT> sm;
  const int tid = threadIdx.x;
  const int t = blockIdx.x;
  const int2 c0 = plan[t], c1 = plan[t + 1];
  const int r0 = c0.x, j0 = c0.y, nr = c1.x - r0, nj = c1.y - j0;
  const uint64_t pol_keep = policy_evict_last();
  for (int i = tid; i < nr; i += M_NT) s_end[i] = row_ptr[r0 + 1 + i];
  for (int j = tid; j < nj; j += M_NT) s_prod[j] = val[j0 + j] * ld_keep(x + col[j0 + j], pol_keep);
  __syncthreads();
  merge_tile_reduce<T, M_NT, M_IPT>(
      t, r0, nr, j0, nj, [&](int i) { return s_end[i]; }, [&](int j) { return s_prod[j]; }, y, accumulate,
      carry_val, carry_row, sm);
}

// Persistent, TMA-pipelined merge SpMV: one elected thread streams each tile's
// col_idx / values / row_ptr slices into a ring of S shared-memory stages with
// cp.async.bulk (L2 evict-first) completing on per-stage mbarriers, S tiles
// ahead of the consumers; all threads gather x (L2 evict-last), form the
// products in place and run the merge-path reduction.  The last partial group
// of each array (the bulk engine needs 16-byte multiples) is read directly.
constexpr int T_NT = 256;
constexpr int T_IPT = 8;
constexpr int T_TILE = T_NT * T_IPT;
constexpr int T_CAP = T_TILE + 8;  // slack for 4-element alignment at both ends
constexpr int T_STAGES = 3;

template <typename T>
__host__ __device__ constexpr size_t tma_stage_bytes() {
  return (size_t)T_CAP * sizeof(T) + 2 * (size_t)T_CAP * 4;
}
template <typename T>
__host__ __device__ constexpr size_t tma_smem_bytes() {
  return T_STAGES * tma_stage_bytes<T>();
}

template <typename T>
__global__ void __launch_bounds__(T_NT, 2) k_spmv_merge_tma(int32_t n_rows, int32_t nnz,
                                                            const int32_t* __restrict__ row_ptr,
                                                            const int32_t* __restrict__ col, const T* __restrict__ val,
                                                            const T* __restrict__ x, T* __restrict__ y,
                                                            const int2* __restrict__ plan, int32_t n_tiles,
                                                            T* __restrict__ carry_val, int32_t* __restrict__ carry_row,
                                                            int accumulate) {
  extern __shared__ __align__(128) unsigned char smem[];
  __shared__ __align__(8) uint64_t full[T_STAGES];
  __shared__ int4 meta[T_STAGES];   // r0, j0, nr, nj
  __shared__ int2 bounds[T_STAGES]; // a1 (first nnz NOT in smem), b1 (first row_ptr idx NOT in smem)
  __shared__ ScanSmem<T, T_NT> sm;
  const int tid = threadIdx.x;
  const int nnz4 = nnz & ~3;             // bulk-copyable prefix of col/val
  const int ptr4 = (n_rows + 1) & ~3;    // bulk-copyable prefix of row_ptr
  auto s_val = [&](int s) { return reinterpret_cast<T*>(smem + s * tma_stage_bytes<T>()); };
  auto s_col = [&](int s) { return reinterpret_cast<int32_t*>(smem + s * tma_stage_bytes<T>() + T_CAP * sizeof(T)); };
  auto s_end = [&](int s) {
    return reinterpret_cast<int32_t*>(smem + s * tma_stage_bytes<T>() + T_CAP * sizeof(T) + T_CAP * 4);
  };

  if (tid == 0) {
    for (int s = 0; s < T_STAGES; ++s) mbar_init(&full[s], 1);
    fence_mbar_init();
  }
  __syncthreads();

  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();

  auto issue = [&](int s, int t) {  // thread 0 only
    const int2 c0 = plan[t], c1 = plan[t + 1];
    const int r0 = c0.x, j0 = c0.y, nr = c1.x - r0, nj = c1.y - j0;
    const int a0 = j0 & ~3;
    const int a1 = max(a0, min((j0 + nj + 3) & ~3, nnz4));
    const int b0 = (r0 + 1) & ~3;
    const int b1 = max(b0, min((r0 + 1 + nr + 3) & ~3, ptr4));
    meta[s] = make_int4(r0, j0, nr, nj);
    bounds[s] = make_int2(a1, b1);
    const uint32_t na = (uint32_t)(a1 - a0), nb = (uint32_t)(b1 - b0);
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&full[s], na * (4 + (uint32_t)sizeof(T)) + nb * 4);
    if (na) {
      bulk_g2s(s_col(s), col + a0, na * 4, &full[s], pol_stream);
      bulk_g2s(s_val(s), val + a0, na * (uint32_t)sizeof(T), &full[s], pol_stream);
    }
    if (nb) bulk_g2s(s_end(s), row_ptr + b0, nb * 4, &full[s], pol_stream);
  };

  const int first = blockIdx.x;
  const int stride = gridDim.x;
  if (tid == 0) {
    for (int s = 0; s < T_STAGES; ++s) {
      const int t = first + s * stride;
      if (t < n_tiles) issue(s, t);
    }
  }
  int it = 0;
  for (int t = first; t < n_tiles; t += stride, ++it) {
    const int s = it % T_STAGES;
    mbar_wait(&full[s], (uint32_t)((it / T_STAGES) & 1));
    const int4 mt = meta[s];
    const int r0 = mt.x, j0 = mt.y, nr = mt.z, nj = mt.w;
    const int a0 = j0 & ~3, b0 = (r0 + 1) & ~3;
    const int2 bd = bounds[s];
    const int a1 = bd.x, b1 = bd.y;
    T* sv = s_val(s);
    const int32_t* sc = s_col(s);
    const int32_t* se = s_end(s);
    // products in place: sv[k - a0] = val[k] * x[col[k]] for k in [j0, j0 + nj)
    {
      int cidx[T_IPT];
      T vv[T_IPT], xv[T_IPT];
#pragma unroll
      for (int q = 0; q < T_IPT; ++q) {
        const int k = j0 + tid + q * T_NT;
        cidx[q] = -1;
        if (k < j0 + nj) {
          if (k < a1) { cidx[q] = sc[k - a0]; vv[q] = sv[k - a0]; }
          else { cidx[q] = col[k]; vv[q] = val[k]; }
        }
      }
#pragma unroll
      for (int q = 0; q < T_IPT; ++q) xv[q] = cidx[q] >= 0 ? ld_keep(x + cidx[q], pol_keep) : T(0);
#pragma unroll
      for (int q = 0; q < T_IPT; ++q) {
        const int k = j0 + tid + q * T_NT;
        if (cidx[q] >= 0) sv[k - a0] = vv[q] * xv[q];
      }
    }
    __syncthreads();
    merge_tile_reduce<T, T_NT, T_IPT>(
        t, r0, nr, j0, nj,
        [&](int i) {
          const int g = r0 + 1 + i;
          return g < b1 ? se[g - b0] : row_ptr[g];
        },
        [&](int j) { return sv[j0 + j - a0]; }, y, accumulate, carry_val, carry_row, sm);
    __syncthreads();  // every thread is done with stage s
    if (tid == 0) {
      const int tn = t + T_STAGES * stride;
      if (tn < n_tiles) issue(s, tn);
    }
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
// x gathers of the CSR-vector kernels: L1::no_allocate + L2 evict-last.  Measured on
// C2: permuted 0.1066 -> 0.1007 ms, unpermuted (banded) 0.0589 -> 0.0576 ms.
__device__ __forceinline__ double ld_x_na(const double* p, uint64_t pol) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ float ld_x_na(const float* p, uint64_t pol) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol));
  return r;
}

template <typename T, int L, typename IP = int32_t>
__global__ void __launch_bounds__(256) k_spmv_vector(int64_t n_rows, const IP* __restrict__ row_ptr,
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
      const IP a = row_ptr[r], b = row_ptr[r + 1];
      for (IP k = a + li; k < b; k += L)
        if (L >= 8) {
          s += ld_stream(val + k, pol_stream) * ld_x_na(x + ld_stream_i1(col + k, pol_stream), pol_keep);
        } else {
          // narrow groups touch each line several times: let L1 keep it (evict-first in L2)
          s += ld_l1(val + k, pol_stream) * ld_x_na(x + ld_l1(col + k, pol_stream), pol_keep);
        }
    }
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (r < n_rows && li == 0) y[r] = accumulate ? y[r] + s : s;
  }
}

// CSR-vector SpMV with the power-iteration / CG epilogue fused in (the unpermuted,
// banded operators of the iterative drivers; the seg twin is sme_spmv_seg_epi):
// v_r = scale * (A x)_r -> out[r]; sum of v_r * (dotv ? dotv[r] : v_r) accumulated
// per thread in the fixed grid-stride order, per block in a fixed tree, and by the
// last block (ticket) in block order: finish 0 -> result = {1/sqrt(sum), sum},
// finish 1 -> result[1] = result[0] / sum (CG alpha).  Deterministic.
constexpr int VE_NT = 256;

template <typename T, int L>
__global__ void __launch_bounds__(VE_NT) k_spmv_vector_epi(int64_t n_rows, const int32_t* __restrict__ row_ptr,
                                                         const int32_t* __restrict__ col, const T* __restrict__ val,
                                                         const T* __restrict__ x, T* __restrict__ out,
                                                         const double* __restrict__ scale, const T* __restrict__ dotv,
                                                         double* __restrict__ partials, unsigned* ticket,
                                                         double* result, int finish) {
  constexpr int RPW = 32 / L;
  const int lane = threadIdx.x & 31;
  const int sub = lane / L, li = lane % L;
  const int64_t warp = ((int64_t)blockIdx.x * VE_NT + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * VE_NT) >> 5;
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  const T sc = scale ? (T)*scale : T(1);
  double ss = 0.0;
  for (int64_t base = warp * RPW; base < n_rows; base += n_warps * RPW) {
    const int64_t r = base + sub;
    T s = T(0);
    if (r < n_rows) {
      const int32_t a = row_ptr[r], b = row_ptr[r + 1];
      for (int32_t k = a + li; k < b; k += L)
        if (L >= 8)
          s += ld_stream(val + k, pol_stream) * ld_x_na(x + ld_stream_i1(col + k, pol_stream), pol_keep);
        else
          s += ld_l1(val + k, pol_stream) * ld_x_na(x + ld_l1(col + k, pol_stream), pol_keep);
    }
#pragma unroll
    for (int o = L / 2; o > 0; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
    if (r < n_rows && li == 0) {
      const T v = sc * s;
      out[r] = v;
      ss += (double)v * (double)(dotv ? dotv[r] : v);
    }
  }
  // block partial (fixed tree), then the last block folds the partials in block order
  __shared__ double red[VE_NT / 32];
  __shared__ bool last;
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < VE_NT / 32; ++w) t += red[w];
    partials[blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  // every thread folds a fixed stride of the partials, then a fixed tree (deterministic)
  __shared__ double fold[VE_NT];
  double acc = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += VE_NT) acc += __ldcg(partials + b);
  fold[threadIdx.x] = acc;
  __syncthreads();
  for (int o = VE_NT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) fold[threadIdx.x] += fold[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double tot = fold[0];
    if (finish == 1) {
      result[1] = result[0] / tot;
    } else {
      result[1] = tot;
      result[0] = tot > 0.0 ? 1.0 / sqrt(tot) : 0.0;
    }
    *ticket = 0u;
  }
}

// numpy's pairwise summation (loops_utils.h.src: pairwise_sum) over the
// products of positions [s, s+n), each product separately rounded.  Leaves:
__device__ double pw_leaf(const int32_t* __restrict__ col, const double* __restrict__ val,
                          const double* __restrict__ x, int64_t s, int64_t n) {
  if (n < 8) {
    double res = -0.0;
    for (int64_t i = 0; i < n; ++i) res = __dadd_rn(res, __dmul_rn(val[s + i], x[col[s + i]]));
    return res;
  }
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
}

// The recursion pw(s,n) = pw(s,n2) + pw(s+n2,n-n2) (n > 128, n2 = n/2 rounded down
// to a multiple of 8) evaluated with an explicit stack (no device-stack recursion).
__device__ double pw_sum(const int32_t* __restrict__ col, const double* __restrict__ val,
                         const double* __restrict__ x, int64_t s0, int64_t n0) {
  constexpr int DEPTH = 48;
  int64_t S[DEPTH], N[DEPTH];
  double L[DEPTH];
  int state[DEPTH];
  int sp = 1;
  S[0] = s0; N[0] = n0; state[0] = 0;
  double ret = 0.0;
  bool have = false;
  while (true) {
    const int i = sp - 1;
    if (have) {
      if (state[i] == 0) {  // left child done: descend into the right child
        L[i] = ret;
        state[i] = 1;
        int64_t n2 = N[i] / 2;
        n2 -= n2 % 8;
        S[sp] = S[i] + n2; N[sp] = N[i] - n2; state[sp] = 0; ++sp;
        have = false;
      } else {  // both children done
        ret = __dadd_rn(L[i], ret);
        if (--sp == 0) return ret;
      }
      continue;
    }
    if (N[i] <= 128) {
      ret = pw_leaf(col, val, x, S[i], N[i]);
      have = true;
      if (--sp == 0) return ret;
      continue;
    }
    int64_t n2 = N[i] / 2;
    n2 -= n2 % 8;
    S[sp] = S[i]; N[sp] = n2; state[sp] = 0; ++sp;
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

// Deterministic COO SpMV, bitwise equal to the reference's np.add.at (kernels.py:81-86):
// np.add.at applies out[row[k]] += v[k] * x[col[k]] in stored entry order, so each
// row's value is ((0 + p_a) + p_b) + ... over its entries in entry order, with every
// product rounded before the add.  The plan lists each row's entries in entry order
// (order[] = entry ids sorted within rows, vals[] the matching values); a thread per
// row replays that sequence with explicit round-to-nearest mul/add (no FMA
// contraction), so the result is independent of scheduling.
__device__ __forceinline__ double coo_mul(double a, double b) { return __dmul_rn(a, b); }
__device__ __forceinline__ double coo_add(double a, double b) { return __dadd_rn(a, b); }
__device__ __forceinline__ float coo_mul(float a, float b) { return __fmul_rn(a, b); }
__device__ __forceinline__ float coo_add(float a, float b) { return __fadd_rn(a, b); }

template <typename T>
__global__ void k_spmv_coo_ordered(int64_t n_rows, const int32_t* __restrict__ rp, const int32_t* __restrict__ order,
                                   const T* __restrict__ val, const int32_t* __restrict__ col,
                                   const T* __restrict__ x, T* __restrict__ y) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    T acc = T(0);
    for (int32_t p = rp[r], e = rp[r + 1]; p < e; ++p) acc = coo_add(acc, coo_mul(val[p], x[col[order[p]]]));
    y[r] = acc;
  }
}

template <typename T, typename IP>
int launch_vector(int lanes, int64_t n_rows, const IP* rp, const int32_t* col, const T* val, const T* x, T* y,
                  int acc, cudaStream_t s) {
  const int64_t threads = n_rows * lanes;
  const int blocks = grid_for(threads, 256, 8);
  switch (lanes) {
    case 1: k_spmv_vector<T, 1, IP><<<blocks, 256, 0, s>>>(n_rows, rp, col, val, x, y, acc); break;
    case 2: k_spmv_vector<T, 2, IP><<<blocks, 256, 0, s>>>(n_rows, rp, col, val, x, y, acc); break;
    case 4: k_spmv_vector<T, 4, IP><<<blocks, 256, 0, s>>>(n_rows, rp, col, val, x, y, acc); break;
    case 8: k_spmv_vector<T, 8, IP><<<blocks, 256, 0, s>>>(n_rows, rp, col, val, x, y, acc); break;
    case 16: k_spmv_vector<T, 16, IP><<<blocks, 256, 0, s>>>(n_rows, rp, col, val, x, y, acc); break;
    case 32: k_spmv_vector<T, 32, IP><<<blocks, 256, 0, s>>>(n_rows, rp, col, val, x, y, acc); break;
    default: SME_REQUIRE(false, "lanes must be one of 1,2,4,8,16,32 (got %d)", lanes);
  }
  SME_CHECK_LAUNCH("k_spmv_vector");
  return SME_OK;
}


// 0 = one CTA per tile (global loads), 1 = persistent TMA pipeline; -1 = auto.
static int merge_mode_override = -1;

template <typename T>
int launch_merge(int mode, int64_t n_rows, int64_t nnz, const int32_t* row_ptr, const int32_t* col, const T* val,
                 const T* x, T* y, const int32_t* plan, int64_t n_tiles, void* carry, int accumulate, cudaStream_t s) {
  const int2* pl = reinterpret_cast<const int2*>(plan);
  char* cb = (char*)carry;
  T* cval = (T*)cb;
  int32_t* carry_row = (int32_t*)(cb + align_up((size_t)n_tiles * 8));
  if (mode == 1) {
    const size_t smem = tma_smem_bytes<T>();
    SME_CUDA(cudaFuncSetAttribute(k_spmv_merge_tma<T>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    const int grid = (int)std::min<int64_t>(n_tiles, (int64_t)sm_count() * 2);
    k_spmv_merge_tma<T><<<grid, T_NT, smem, s>>>((int32_t)n_rows, (int32_t)nnz, row_ptr, col, val, x, y, pl,
                                                 (int32_t)n_tiles, cval, carry_row, accumulate);
    SME_CHECK_LAUNCH("k_spmv_merge_tma");
  } else {
    k_spmv_merge<T><<<(unsigned)n_tiles, M_NT, 0, s>>>((int32_t)n_rows, (int32_t)nnz, row_ptr, col, val, x, y, pl,
                                                       cval, carry_row, accumulate);
    SME_CHECK_LAUNCH("k_spmv_merge");
  }
  if (n_tiles > 1) {
    k_spmv_fixup<T><<<grid_for(n_tiles, 256), 256, 0, s>>>(n_tiles, pl, carry_row, cval, y);
    SME_CHECK_LAUNCH("k_spmv_fixup");
  }
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
  if (n_tiles == 0) return SME_OK;
  SME_REQUIRE(dtype == SME_F64 || dtype == SME_F32, "unknown dtype %d", dtype);
  cudaStream_t s = as_stream(stream);
  const bool aligned = (((uintptr_t)col | (uintptr_t)val | (uintptr_t)row_ptr) & 15) == 0;
  const int mode = merge_mode_override >= 0 ? merge_mode_override : (aligned ? 1 : 0);
  SME_REQUIRE(mode == 0 || aligned, "the TMA merge kernel needs 16-byte aligned row_ptr/col_idx/values");
  if (dtype == SME_F64)
    return launch_merge<double>(mode, n_rows, nnz, row_ptr, col, (const double*)val, (const double*)x, (double*)y,
                                plan, n_tiles, carry, accumulate, s);
  return launch_merge<float>(mode, n_rows, nnz, row_ptr, col, (const float*)val, (const float*)x, (float*)y, plan,
                             n_tiles, carry, accumulate, s);
}

template <typename IP>
static int spmv_vector_impl(int dtype, int lanes, int64_t n_rows, const IP* row_ptr, const int32_t* col,
                            const void* val, const void* x, void* y, int accumulate, sme_stream_t stream) {
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

SME_API int sme_spmv_vector(int dtype, int lanes, int64_t n_rows, int64_t n_cols, const int32_t* row_ptr,
                            const int32_t* col, const void* val, const void* x, void* y, int accumulate,
                            sme_stream_t stream) {
  return spmv_vector_impl(dtype, lanes, n_rows, row_ptr, col, val, x, y, accumulate, stream);
}

SME_API int sme_spmv_vector_i64(int dtype, int lanes, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                                const int32_t* col, const void* val, const void* x, void* y, int accumulate,
                                sme_stream_t stream) {
  return spmv_vector_impl(dtype, lanes, n_rows, row_ptr, col, val, x, y, accumulate, stream);
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

SME_API int sme_spmv_coo_ordered(int dtype, int64_t n_rows, const int32_t* row_ptr, const int32_t* order,
                                 const void* val, const int32_t* col, const void* x, void* y, sme_stream_t stream) {
  cudaStream_t s = as_stream(stream);
  SME_REQUIRE(dtype == SME_F64 || dtype == SME_F32, "unknown dtype %d", dtype);
  if (n_rows == 0) return SME_OK;
  if (dtype == SME_F64)
    k_spmv_coo_ordered<double><<<grid_for(n_rows, 256), 256, 0, s>>>(n_rows, row_ptr, order, (const double*)val, col,
                                                                     (const double*)x, (double*)y);
  else
    k_spmv_coo_ordered<float><<<grid_for(n_rows, 256), 256, 0, s>>>(n_rows, row_ptr, order, (const float*)val, col,
                                                                    (const float*)x, (float*)y);
  SME_CHECK_LAUNCH("k_spmv_coo_ordered");
  return SME_OK;
}

// Kernel selection for experiments/tests: 0 = per-tile kernel, 1 = TMA pipeline, -1 = auto.
SME_API int sme_spmv_merge_set_mode(int mode) {
  SME_REQUIRE(mode >= -1 && mode <= 1, "mode must be -1, 0 or 1");
  merge_mode_override = mode;
  return SME_OK;
}


// Blocks of sme_spmv_vector_epi's fixed grid (= the length of its partials scratch):
// exactly one resident wave of the kernel (its occupancy at 40 registers is 6 CTAs
// of 256 per SM), never more than the rows need — a partial second wave would idle
// most SMs at the tail (measured: the 8-per-SM grid of k_spmv_vector ran 36 % slower).
static int64_t vector_epi_blocks(int64_t n_rows, int lanes) {
  int occ = 0;
  const void* fn = lanes == 1 ? (const void*)k_spmv_vector_epi<double, 1>
                 : lanes == 2 ? (const void*)k_spmv_vector_epi<double, 2>
                 : lanes == 4 ? (const void*)k_spmv_vector_epi<double, 4>
                 : lanes == 8 ? (const void*)k_spmv_vector_epi<double, 8>
                 : lanes == 16 ? (const void*)k_spmv_vector_epi<double, 16>
                               : (const void*)k_spmv_vector_epi<double, 32>;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, fn, VE_NT, 0) != cudaSuccess || occ < 1) occ = 4;
  return grid_for(std::max<int64_t>(1, n_rows) * lanes, VE_NT, occ);
}

SME_API int sme_spmv_vector_epi_blocks(int64_t n_rows, int lanes, int64_t* blocks) {
  SME_REQUIRE(blocks && n_rows >= 0 && lanes >= 1 && lanes <= 32, "bad arguments");
  *blocks = vector_epi_blocks(n_rows, lanes);
  return SME_OK;
}

// out = scale[0] * (A x) with the iterative drivers' reduction fused (see k_spmv_vector_epi);
// f64; scale may be null (1); dotv null -> sum of squares (power iteration), else
// sum out * dotv (CG's p.Ap, finish = 1 writes alpha = result[0] / sum into result[1]).
SME_API int sme_spmv_vector_epi(int lanes, int64_t n_rows, const int32_t* row_ptr, const int32_t* col,
                                const double* val, const double* x, double* out, const double* scale,
                                const double* dotv, double* partials, uint32_t* ticket, double* result, int finish,
                                sme_stream_t stream) {
  SME_REQUIRE(n_rows >= 1 && n_rows < INT32_MAX && out && partials && ticket && result && (finish == 0 || finish == 1),
              "bad arguments");
  cudaStream_t s = as_stream(stream);
  const int blocks = (int)vector_epi_blocks(n_rows, lanes);
#define VE_CASE(LN)                                                                                             \
  case LN:                                                                                                      \
    k_spmv_vector_epi<double, LN><<<blocks, VE_NT, 0, s>>>(n_rows, row_ptr, col, val, x, out, scale, dotv,     \
                                                           partials, ticket, result, finish);                  \
    break;
  switch (lanes) {
    VE_CASE(1) VE_CASE(2) VE_CASE(4) VE_CASE(8) VE_CASE(16) VE_CASE(32)
    default: SME_REQUIRE(false, "lanes must be one of 1,2,4,8,16,32 (got %d)", lanes);
  }
#undef VE_CASE
  SME_CHECK_LAUNCH("k_spmv_vector_epi");
  return SME_OK;
}

namespace sme {
// The fused epilogue on its own, for layouts whose passes cannot carry it (split-row seg
// plans): v_r = scale * y[r] -> out[qinv ? qinv[r] : r], reduction as k_spmv_vector_epi.
__global__ void __launch_bounds__(VE_NT) k_rows_epi(int64_t n_rows, const double* __restrict__ y,
                                                  double* __restrict__ out, const int32_t* __restrict__ qinv,
                                                  const double* __restrict__ scale, const double* __restrict__ dotv,
                                                  double* __restrict__ partials, unsigned* ticket, double* result,
                                                  int finish) {
  const double sc = scale ? *scale : 1.0;
  double ss = 0.0;
  for (int64_t r = (int64_t)blockIdx.x * VE_NT + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * VE_NT) {
    const double v = sc * y[r];
    const int64_t g = qinv ? qinv[r] : r;
    out[g] = v;
    ss += v * (dotv ? dotv[g] : v);
  }
  __shared__ double red[VE_NT / 32];
  __shared__ bool last;
  const int lane = threadIdx.x & 31;
  for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(0xffffffffu, ss, o);
  if (lane == 0) red[threadIdx.x >> 5] = ss;
  __syncthreads();
  if (threadIdx.x == 0) {
    double t = 0.0;
    for (int w = 0; w < VE_NT / 32; ++w) t += red[w];
    partials[blockIdx.x] = t;
    __threadfence();
    last = atomicAdd(ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  __shared__ double fold[VE_NT];
  double acc = 0.0;
  for (unsigned b = threadIdx.x; b < gridDim.x; b += VE_NT) acc += __ldcg(partials + b);
  fold[threadIdx.x] = acc;
  __syncthreads();
  for (int o = VE_NT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) fold[threadIdx.x] += fold[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double tot = fold[0];
    if (finish == 1) {
      result[1] = result[0] / tot;
    } else {
      result[1] = tot;
      result[0] = tot > 0.0 ? 1.0 / sqrt(tot) : 0.0;
    }
    *ticket = 0u;
  }
}
}  // namespace sme

// Blocks of sme_rows_epi's fixed grid (the length of its partials scratch).
SME_API int sme_rows_epi_blocks(int64_t n_rows, int64_t* blocks) {
  SME_REQUIRE(blocks && n_rows >= 0, "bad arguments");
  *blocks = grid_for(std::max<int64_t>(1, n_rows), VE_NT, 8);
  return SME_OK;
}

// out = scale[0] * y (scale NULL: 1), scattered through qinv (NULL: identity), with the
// iteration's reduction (dotv NULL: sum out^2 -> result {1/sqrt, sum}; else sum out * dotv,
// finish 1 -> result[1] = result[0] / sum).  f64.
SME_API int sme_rows_epi(int64_t n_rows, const double* y, double* out, const int32_t* qinv, const double* scale,
                         const double* dotv, double* partials, uint32_t* ticket, double* result, int finish,
                         sme_stream_t stream) {
  SME_REQUIRE(n_rows >= 1 && y && out && partials && ticket && result && (finish == 0 || finish == 1),
              "bad arguments");
  const int blocks = grid_for(n_rows, VE_NT, 8);
  k_rows_epi<<<blocks, VE_NT, 0, as_stream(stream)>>>(n_rows, y, out, qinv, scale, dotv, partials, ticket, result,
                                                      finish);
  SME_CHECK_LAUNCH("k_rows_epi");
  return SME_OK;
}

namespace sme {
// Lazy module loading (CUDA 12 default) loads this file's module on the first launch of
// any of its kernels, ~10-20 ms each; sme_preload() does it ahead of time.
int preload_spmv() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)k_spmv_plan) == cudaSuccess ? 0 : -1;
}
}  // namespace sme
