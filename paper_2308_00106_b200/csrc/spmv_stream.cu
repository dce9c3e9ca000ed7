// spmv_stream.cu — k_spmv_stream: warp-streaming CSR SpMV with a warp-level
// segmented reduction (the fast path for regular and moderately ragged rows).
//
// Reference: spmv_csr / _accumulate_rows (kernels.py:59-78).
//
// Work split: a per-matrix plan gives every warp a contiguous row range
// holding ~nnz/W nonzeros (W = resident warps of the persistent grid), so a
// row never spans two warps and there is no fix-up pass.  A warp streams its
// nonzeros in 128-element chunks aligned to GLOBAL multiples of 128 (lane l
// holds elements c+4l..c+4l+3: one 128-bit col_idx load and two/one 128-bit
// value loads, L1 no-allocate, L2 evict-first), prefetching the next chunk
// before it gathers x for the current one (L2 evict-last).  Rows are reduced
// with a flag-segmented scan: row starts inside the chunk become head bits
// (__reduce_or_sync), each lane folds its 4 products, a 5-step shuffle scan
// carries partial sums across lanes, the open segment carries into the next
// chunk, and the lane owning row i of a sliding 32-row window picks the row
// total at position end_i - 1.  A row's association depends only on its
// global positions (align_off = global position of local element 0), so row
// shards that keep positions mod 128 reduce bitwise-identically.
#include "common.cuh"

#include <algorithm>

namespace sme {

constexpr int S_NT = 256;

template <typename T> struct Vec4;
template <> struct Vec4<double> {
  static __device__ __forceinline__ void load(const double* p, uint64_t pol, double v[4]) {
    double2 a = ld_stream_d2(reinterpret_cast<const double2*>(p), pol);
    double2 b = ld_stream_d2(reinterpret_cast<const double2*>(p) + 1, pol);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
};
template <> struct Vec4<float> {
  static __device__ __forceinline__ void load(const float* p, uint64_t pol, float v[4]) {
    float4 a = ld_stream_f4(reinterpret_cast<const float4*>(p), pol);
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  }
};

// 4 consecutive elements at local index e (e % 4 == 0 when vec_ok); anything
// outside [0, nnz) reads as col = -1.  Elements of neighbouring rows inside
// the chunk are loaded too and masked later (the aligned chunk is one line).
template <typename T>
__device__ __forceinline__ void chunk_load(const int32_t* __restrict__ col, const T* __restrict__ val, int e,
                                           int nnz, bool vec_ok, uint64_t pol, int c[4], T v[4]) {
  if (vec_ok && e >= 0 && e + 3 < nnz) {
    int4 ci = ld_stream_i4(reinterpret_cast<const int4*>(col + e), pol);
    c[0] = ci.x; c[1] = ci.y; c[2] = ci.z; c[3] = ci.w;
    Vec4<T>::load(val + e, pol, v);
  } else {
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const int k = e + q;
      if (k >= 0 && k < nnz) { c[q] = ld_stream_i1(col + k, pol); v[q] = ld_stream(val + k, pol); }
      else { c[q] = -1; v[q] = T(0); }
    }
  }
}

// warp_rows[w] = first row of warp w: balanced on the cost nnz + 2 * rows (a row
// costs about two nonzeros of window bookkeeping), so matrices with many empty
// rows (R-MAT) do not hand one warp millions of rows: the first row r with
// row_ptr[r] + 2 r >= w * (nnz + 2 n_rows) / W.
static int s_row_cost = 2;  // sme_spmv_stream_set_row_cost

__global__ void k_stream_plan(int32_t n_rows, int32_t nnz, const int32_t* __restrict__ row_ptr, int32_t n_warps,
                              int64_t row_cost, int32_t* __restrict__ warp_rows) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w <= n_warps; w += gridDim.x * blockDim.x) {
    if (w == 0) { warp_rows[0] = 0; continue; }
    if (w == n_warps) { warp_rows[w] = n_rows; continue; }
    const int64_t total = (int64_t)nnz + row_cost * n_rows;
    const int64_t target = (int64_t)w * total / n_warps;
    int lo = 0, hi = n_rows;  // lower_bound of the monotone cost row_ptr[r] + row_cost * r
    while (lo < hi) {
      int mid = (lo + hi) >> 1;
      if ((int64_t)row_ptr[mid] + row_cost * mid < target) lo = mid + 1; else hi = mid;
    }
    warp_rows[w] = lo;
  }
}

// TMA = true: the chunk stream (col_idx, values) arrives through a per-warp ring of
// STAGES shared-memory slots filled by cp.async.bulk (L2 evict-first), STAGES
// chunks ahead, each slot completing on its own mbarrier; TMA = false (unaligned
// arrays): 128-bit register loads prefetched one chunk ahead.
constexpr int S_STAGES = 3;

template <typename T, bool ACC, bool TMA>
__global__ void __launch_bounds__(S_NT) k_spmv_stream(int32_t n_rows, int32_t nnz, const int32_t* __restrict__ row_ptr,
                                                      const int32_t* __restrict__ col, const T* __restrict__ val,
                                                      const T* __restrict__ x, T* __restrict__ y,
                                                      const int32_t* __restrict__ warp_rows, int32_t n_warps,
                                                      int32_t align_off, bool vec_ok) {
  constexpr int CH = 128;       // chunk = 32 lanes x 4 elements
  constexpr int LOOP_MAX = 24;  // per-lane row loops up to this overlap, else segmented scan
  constexpr int SST = TMA ? S_STAGES : 1;
  __shared__ T s_buf[S_NT / 32][CH];
  __shared__ __align__(16) int32_t s_col[S_NT / 32][SST][CH];
  __shared__ __align__(16) T s_val[S_NT / 32][SST][CH];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int wib = threadIdx.x >> 5;
  T* buf = s_buf[wib];
  const int nnz4 = nnz & ~3;  // bulk-copyable prefix of col/val
  const int warp = (blockIdx.x * S_NT + threadIdx.x) >> 5;
  if (warp >= n_warps) return;
  const uint64_t pol_stream = policy_evict_first();
  const uint64_t pol_keep = policy_evict_last();
  const int R0 = warp_rows[warp], R1 = warp_rows[warp + 1];
  if (R0 >= R1) return;
  const int P0 = row_ptr[R0], P1 = row_ptr[R1];

  // window: lane l holds row q + l: its [s, e) and the partial sum acc
  int q = R0;
  int r = q + lane;
  bool live = r < R1;
  int s = live ? row_ptr[r] : P1;
  int e = live ? row_ptr[r + 1] : P1;
  T acc = T(0);
  // accumulate mode: y of a window row is fetched when the row enters the window,
  // long before it retires, so the read-modify-write never waits on DRAM
  T yv = (ACC && live) ? y[r] : T(0);
  // prefetched next window W1: rows q + 32 + lane
  int s1, e1;
  T yv1 = T(0);
  {
    const int r1 = r + 32;
    s1 = r1 < R1 ? row_ptr[r1] : P1;
    e1 = r1 < R1 ? row_ptr[r1 + 1] : P1;
    if (ACC && r1 < R1) yv1 = y[r1];
  }

  int c = ((P0 + align_off) & ~(CH - 1)) - align_off;
  // async copy of this lane's 4-element group of chunk cc into ring slot st
  // (LDGSTS; the group is copied only when it lies inside [0, nnz4), the rest is
  // read directly at consume time).  Every call commits one group, possibly empty.
  auto issue = [&](int st, int cc) {
    const int e0 = cc + 4 * lane;
    if (cc < P1 && e0 >= 0 && e0 + 3 < nnz4) {
      cp_async16(&s_col[wib][st][4 * lane], col + e0, 16, pol_stream);
      for (int h = 0; h < (int)sizeof(T) / 4; ++h)
        cp_async16(&s_val[wib][st][4 * lane + 4 / ((int)sizeof(T) / 4) * h], val + e0 + 4 / ((int)sizeof(T) / 4) * h,
                   16, pol_stream);
    }
    cp_async_commit();
  };
  int ci[4];
  T vv[4];
  int it = 0;  // chunk counter (ring slot = it % SST)
  if (TMA) {
    if (P0 >= P1) c = P1;
#pragma unroll
    for (int st = 0; st < SST; ++st) issue(st, c + st * CH);
  } else {
    if (P0 < P1) chunk_load<T>(col, val, c + 4 * lane, nnz, vec_ok, pol_stream, ci, vv);
    else c = P1;  // only empty rows
  }
  while (q < R1) {
    const bool have = c < P1;
    const int cend = have ? c + CH : INT32_MAX;
    int nci[4];
    T nvv[4];
    if (!TMA && c + CH < P1) chunk_load<T>(col, val, c + CH + 4 * lane, nnz, vec_ok, pol_stream, nci, nvv);
    if (TMA && have) {
      const int st = it % SST;
      cp_async_wait<SST - 1>();  // this lane's copies of chunk `it` have landed
      const int a = max(c, 0), b = nnz4;
      const int e0 = c + 4 * lane;
      if (e0 >= a && e0 + 3 < b) {
        const int4 cc4 = *reinterpret_cast<const int4*>(&s_col[wib][st][4 * lane]);
        ci[0] = cc4.x; ci[1] = cc4.y; ci[2] = cc4.z; ci[3] = cc4.w;
#pragma unroll
        for (int k = 0; k < 4; ++k) vv[k] = s_val[wib][st][4 * lane + k];
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          const int pos = e0 + k;
          // partial groups (array ends) were not copied: read them directly
          if (pos >= 0 && pos < nnz) { ci[k] = col[pos]; vv[k] = val[pos]; }
          else { ci[k] = -1; vv[k] = T(0); }
        }
      }
    }
    if (have) {
      T xv[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        const int pos = c + 4 * lane + k;
        if (pos < P0 || pos >= P1) ci[k] = -1;
        xv[k] = ci[k] >= 0 ? ld_keep(x + ci[k], pol_keep) : T(0);
      }
      T p[4];
#pragma unroll
      for (int k = 0; k < 4; ++k) p[k] = ci[k] >= 0 ? vv[k] * xv[k] : T(0);
      // overlap of every window row with this chunk decides the reduction
      const int lo0 = max(s, c), hi0 = min(e, cend);
      const unsigned ov0 = live && hi0 > lo0 ? (unsigned)(hi0 - lo0) : 0u;
      const unsigned maxov = __reduce_max_sync(FULL, ov0);
      if (maxov > LOOP_MAX) {
        // long rows: flag-segmented scan restarting at the chunk start; afterwards
        // buf[j] = sum of the row segment ending at position c + j inside the chunk
        unsigned f0 = 0, f1 = 0, f2 = 0, f3 = 0;
        {
          int wq = q, ws = s, we = e;
          while (true) {
            const int rel = ws - c;
            const bool head = wq + lane < R1 && ws < we && rel >= 0 && rel < CH;
            const unsigned bit = head ? (1u << (rel & 31)) : 0u;
            const int word = rel >> 5;
            f0 |= __reduce_or_sync(FULL, (head && word == 0) ? bit : 0u);
            f1 |= __reduce_or_sync(FULL, (head && word == 1) ? bit : 0u);
            f2 |= __reduce_or_sync(FULL, (head && word == 2) ? bit : 0u);
            f3 |= __reduce_or_sync(FULL, (head && word == 3) ? bit : 0u);
            const int last_s = __shfl_sync(FULL, ws, 31);
            if (wq + 32 >= R1 || last_s >= cend) break;
            wq += 32;
            const int rr = wq + lane;
            ws = rr < R1 ? row_ptr[rr] : P1;
            we = rr < R1 ? row_ptr[rr + 1] : P1;
          }
        }
        const int wsel = lane >> 3;
        const unsigned fw = wsel == 0 ? f0 : (wsel == 1 ? f1 : (wsel == 2 ? f2 : f3));
        const unsigned my = (fw >> ((4 * lane) & 31)) & 0xFu;
        T a[4];
        a[0] = p[0];
#pragma unroll
        for (int k = 1; k < 4; ++k) a[k] = ((my >> k) & 1u) ? p[k] : a[k - 1] + p[k];
        T v = a[3];
        bool f = my != 0u;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const T ov = __shfl_up_sync(FULL, v, o);
          const bool of = __shfl_up_sync(FULL, (int)f, o) != 0;
          if (lane >= o) {
            if (!f) v = ov + v;
            f = f || of;
          }
        }
        T ex = __shfl_up_sync(FULL, v, 1);
        if (lane == 0) ex = T(0);
        bool open = true;
#pragma unroll
        for (int k = 0; k < 4; ++k) {
          if ((my >> k) & 1u) open = false;
          buf[4 * lane + k] = open ? ex + a[k] : a[k];
        }
      } else {
#pragma unroll
        for (int k = 0; k < 4; ++k) buf[4 * lane + k] = p[k];
      }
      __syncwarp();
      const bool scanned = maxov > LOOP_MAX;
      // every window row adds its overlap with the chunk; finished rows retire and
      // the window refills (several passes when rows are shorter than ~4 nnz)
      bool counted = false;
      while (true) {
        if (!counted && live) {
          const int lo = max(s, c), hi = min(e, cend);
          if (hi > lo) {
            if (scanned) {
              acc += buf[hi - 1 - c];
            } else {
              T t = T(0);
              for (int k = lo; k < hi; ++k) t += buf[k - c];
              acc += t;
            }
          }
          counted = true;
        }
        const unsigned done = __ballot_sync(FULL, live && e <= cend);
        const int n_done = __popc(done);  // finished rows form a prefix of the window
        if (lane < n_done) y[r] = ACC ? yv + acc : acc;
        if (n_done == 0) break;
        q += n_done;
        const T acc_n = __shfl_down_sync(FULL, acc, n_done);
        const T yv_n = ACC ? __shfl_down_sync(FULL, yv, n_done) : T(0);
        const int s_n = __shfl_down_sync(FULL, s, n_done), e_n = __shfl_down_sync(FULL, e, n_done);
        const bool cnt_n = __shfl_down_sync(FULL, (int)counted, n_done) != 0;
        // rotate the prefetched window: lane l reads W1[(l + n) % 32]; W0's new tail
        // lanes take W1's head, W1 shifts down and loads its new tail (needed ~32 rows
        // later, so that latency is hidden)
        const int rot = (lane + n_done) & 31;
        const int s_w = __shfl_sync(FULL, s1, rot), e_w = __shfl_sync(FULL, e1, rot);
        const T y_w = ACC ? __shfl_sync(FULL, yv1, rot) : T(0);
        r = q + lane;
        live = r < R1;
        if (lane < 32 - n_done) {
          acc = acc_n; s = s_n; e = e_n; counted = cnt_n;
          if (ACC) yv = yv_n;
          s1 = s_w; e1 = e_w;
          if (ACC) yv1 = y_w;
        } else {
          acc = T(0);
          s = s_w; e = e_w;
          if (ACC) yv = y_w;
          counted = false;
          const int r1 = r + 32;
          s1 = r1 < R1 ? row_ptr[r1] : P1;
          e1 = r1 < R1 ? row_ptr[r1 + 1] : P1;
          if (ACC) yv1 = r1 < R1 ? y[r1] : T(0);
        }
        // stop when no uncounted live row reaches into this chunk
        if (!__any_sync(FULL, live && !counted && s < cend) && !__any_sync(FULL, live && e <= cend)) break;
        if (q >= R1) break;
      }
      __syncwarp();
    } else {
      // no nonzeros left: the remaining rows of the range are empty
      const unsigned done = __ballot_sync(FULL, live);
      const int n_done = __popc(done);
      if (live && !ACC) y[r] = T(0);
      q += n_done;
      r = q + lane;
      live = r < R1;
      s = e = P1;
      continue;
    }
    if (TMA) {
      // this lane is done with its slot: refill it STAGES chunks ahead
      if (have) {
        issue(it % SST, c + SST * CH);
        ++it;
      }
    } else {
#pragma unroll
      for (int k = 0; k < 4; ++k) { ci[k] = nci[k]; vv[k] = nvv[k]; }
    }
    c += CH;
  }
}

static int stream_ring_mode = 0;  // 0 = register prefetch, 1 = per-lane cp.async ring

template <typename T>
int launch_stream(int64_t n_rows, int64_t nnz, const int32_t* row_ptr, const int32_t* col, const T* val, const T* x,
                  T* y, const int32_t* plan, int32_t n_warps, int accumulate, int32_t align_off, bool vec,
                  cudaStream_t s) {
  const int grid = (n_warps * 32 + S_NT - 1) / S_NT;
#define SME_LAUNCH_STREAM(ACC, TMA)                                                                          \
  k_spmv_stream<T, ACC, TMA><<<grid, S_NT, 0, s>>>((int32_t)n_rows, (int32_t)nnz, row_ptr, col, val, x, y, plan, \
                                                   n_warps, align_off, vec)
  // the cp.async ring measured slower than the one-chunk register prefetch on B200
  // (C4 panel SpMV 7.99 vs 6.36 ms): it is opt-in (sme_spmv_stream_set_mode(1))
  if (vec && stream_ring_mode == 1) {
    if (accumulate) SME_LAUNCH_STREAM(true, true); else SME_LAUNCH_STREAM(false, true);
  } else {
    if (accumulate) SME_LAUNCH_STREAM(true, false); else SME_LAUNCH_STREAM(false, false);
  }
#undef SME_LAUNCH_STREAM
  SME_CHECK_LAUNCH("k_spmv_stream");
  return SME_OK;
}

}  // namespace sme

using namespace sme;

// Plan weight of one row in nonzero units (warp ranges balance nnz + row_cost * rows).
SME_API int sme_spmv_stream_set_row_cost(int cost) {
  SME_REQUIRE(cost >= 0 && cost <= 64, "row cost must lie in [0, 64]");
  s_row_cost = cost;
  return SME_OK;
}

SME_API int sme_spmv_stream_set_mode(int mode) {
  SME_REQUIRE(mode == 0 || mode == 1, "mode must be 0 (register prefetch) or 1 (cp.async ring)");
  stream_ring_mode = mode;
  return SME_OK;
}

SME_API int sme_spmv_stream_warps(int64_t n_rows, int64_t nnz, int32_t* n_warps) {
  SME_REQUIRE(n_warps && n_rows >= 0 && nnz >= 0, "bad arguments");
  // exactly the resident warps of the persistent grid (static ranges need them all
  // running at once), never more than ~1 warp per 32 rows
  int per_sm = 0;
  per_sm = 1 << 20;
  auto occ = [&](const void* fn) {
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, fn, S_NT, 0) == cudaSuccess) per_sm = std::min(per_sm, v);
  };
  occ((const void*)k_spmv_stream<double, false, true>);
  occ((const void*)k_spmv_stream<double, true, true>);
  occ((const void*)k_spmv_stream<double, false, false>);
  occ((const void*)k_spmv_stream<double, true, false>);
  per_sm = std::max(1, per_sm);
  int64_t w = (int64_t)sm_count() * per_sm * (S_NT / 32);
  w = std::min<int64_t>(w, std::max<int64_t>(1, (n_rows + 31) / 32));
  *n_warps = (int32_t)w;
  return SME_OK;
}

SME_API int sme_spmv_stream_plan(int64_t n_rows, int64_t nnz, const int32_t* row_ptr, int32_t n_warps,
                                 int32_t* plan, sme_stream_t stream) {
  SME_REQUIRE(n_rows >= 0 && n_rows < INT32_MAX - 256 && nnz >= 0 && nnz < INT32_MAX - 256, "sizes exceed int32");
  SME_REQUIRE(n_warps >= 1, "n_warps must be >= 1");
  cudaStream_t s = as_stream(stream);
  k_stream_plan<<<grid_for((int64_t)n_warps + 1, 256), 256, 0, s>>>((int32_t)n_rows, (int32_t)nnz, row_ptr, n_warps,
                                                                     (int64_t)s_row_cost, plan);
  SME_CHECK_LAUNCH("k_stream_plan");
  return SME_OK;
}

SME_API int sme_spmv_stream(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* row_ptr,
                            const int32_t* col, const void* val, const void* x, void* y, const int32_t* plan,
                            int32_t n_warps, int accumulate, int32_t align_off, sme_stream_t stream) {
  SME_REQUIRE(n_rows >= 0 && n_rows < INT32_MAX - 256 && nnz >= 0 && nnz < INT32_MAX - 256, "sizes exceed int32");
  SME_REQUIRE(plan && n_warps >= 1, "missing stream plan");
  SME_REQUIRE(align_off >= 0 && align_off < 128, "align_off must lie in [0, 128)");
  if (n_rows == 0) return SME_OK;
  SME_REQUIRE(dtype == SME_F64 || dtype == SME_F32, "unknown dtype %d", dtype);
  // 128-bit loads need 16-byte aligned arrays and local index = global index (mod 4)
  const bool vec = (((uintptr_t)col | (uintptr_t)val) & 15) == 0 && (align_off & 3) == 0;
  cudaStream_t s = as_stream(stream);
  if (dtype == SME_F64)
    return launch_stream<double>(n_rows, nnz, row_ptr, col, (const double*)val, (const double*)x, (double*)y, plan,
                                 n_warps, accumulate, align_off, vec, s);
  return launch_stream<float>(n_rows, nnz, row_ptr, col, (const float*)val, (const float*)x, (float*)y, plan, n_warps,
                              accumulate, align_off, vec, s);
}

namespace sme {
// Lazy module loading (CUDA 12 default) loads this file's module on the first launch of
// any of its kernels, ~10-20 ms each; sme_preload() does it ahead of time.
int preload_spmv_stream() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)k_stream_plan) == cudaSuccess ? 0 : -1;
}
}  // namespace sme
