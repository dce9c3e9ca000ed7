// spmv_seg.cu — the "segmented chunk" SpMV layout and kernel: the fast path for
// randomly permuted matrices (short, uniform rows; x gathers that only an
// L2-resident x slice can serve).
//
// Reference: spmv_csr / _accumulate_rows (kernels.py:59-78): y_i = sum_k v_k x[c_k]
// over row i, empty rows give 0.  Same products; the row sums are associated
// in chunk order instead of numpy's pairwise order (tolerance 1e-12, the
// reference's CORRECTNESS_RTOL, bench.py:34).
//
// Why a new layout.  After a random permutation the x gathers of a CSR SpMV are
// uniformly random.  On B200 every such gather is one L1tex wavefront (one
// 128-B line per lane; 1 wavefront / clk / SM = 291 G gathers/s at 1965 MHz,
// measured 285 G/s, tools/gather_bench.cu — TMA gather4 measured 120 G/s and
// per-lane bulk copies 63 G/s, so LDG is the gather path).  The kernel is
// therefore bounded by wavefronts per nonzero, and everything else it does
// must cost a small fraction of one wavefront per nonzero:
//   * no row_ptr: each 32-bit entry packs the panel-local column (23 bits) and
//     the row offset from its 128-entry chunk's header row (9 bits), so the
//     per-pass row_ptr stream of a column-panel CSR (4 B/row/panel) disappears;
//   * a warp reads a 128-entry chunk with three coalesced 128-bit loads per
//     lane (pk, and val as 2 x 16 B), gathers 4 x values per lane, and sums
//     rows with a key-segmented warp scan (keys = absolute rows, which are
//     non-decreasing inside the chunk);
//   * the row total is written (or accumulated, for panel passes p > 0) by the
//     lane holding the row's last entry; a row continuing into the next chunk
//     is carried in registers.
//
// Layout of one panel (columns [b_p, b_{p+1})), n_pad = round_up(entries, 128):
//   pk[n_pad]  uint32  (col - b_p) << 9 | (row - hdr[chunk])   (col field 0x7FFFFF = explicit zero)
//   val[n_pad] f64/f32 (0 for explicit zeros and tail padding)
//   hdr[n_pad / 128] int32 row of the chunk's first entry
// Rows keep their CSR (row-major, column-ascending) order.  Explicit zeros are
// added (a) in panel 0 for every row without entries there, so the
// non-accumulating pass writes every y row, and (b) in later panels for empty
// rows r with r % 4 == 0, so consecutive entries are at most 4 rows apart and
// a 128-entry chunk spans at most 508 rows (fits the 9-bit offset).
//
// Work split: warp w of the persistent grid owns entry positions
// [plan[w], plan[w+1]), which always start and end on row boundaries (rows are
// whole within one warp, so every y row has exactly one writer: deterministic).
#include "common.cuh"
#include "scan.cuh"

#include <algorithm>

namespace sme {

constexpr int SEG_NT = 256;
constexpr int SEG_CH = 128;
constexpr int SEG_DBITS = 9;
constexpr uint32_t SEG_DMASK = (1u << SEG_DBITS) - 1;
constexpr uint32_t SEG_MARK = (1u << (32 - SEG_DBITS)) - 1;  // col field of an explicit zero
constexpr int SEG_GAP = 4;                                   // padding stride of empty rows (p > 0)

// ---------------------------------------------------------------------------
// layout build
// ---------------------------------------------------------------------------

// counts[p * n + r] = entries of row r in panel p (rows are column-sorted)
__global__ void k_seg_count(int64_t n_rows, const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                            int32_t n_panels, const int32_t* __restrict__ bounds, int32_t* __restrict__ counts) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = row_ptr[r], b = row_ptr[r + 1];
    int32_t k = a;
    for (int p = 0; p < n_panels; ++p) {
      const int32_t hi = bounds[p + 1];
      // binary search for the first column >= hi in [k, b)
      int32_t lo = k, up = b;
      while (lo < up) {
        const int32_t mid = (lo + up) >> 1;
        if (col[mid] < hi) lo = mid + 1; else up = mid;
      }
      counts[(int64_t)p * n_rows + r] = lo - k;
      k = lo;
    }
  }
}

// entries of row r in the panel layout: its count, or one explicit zero
struct SegLen {
  const int32_t* counts;  // this panel's counts
  int32_t panel;
  __device__ __forceinline__ int64_t operator()(int64_t r) const {
    const int32_t c = counts[r];
    return c > 0 ? c : ((panel == 0 || (r % SEG_GAP) == 0) ? 1 : 0);
  }
};

// hdr[c] = row of the entry at position 128 c (one panel)
__global__ void k_seg_hdr(int64_t n_rows, const int32_t* __restrict__ pos, int32_t* __restrict__ hdr) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = pos[r], b = pos[r + 1];
    for (int32_t c = (a + SEG_CH - 1) / SEG_CH; c * SEG_CH < b; ++c) hdr[c] = (int32_t)r;
  }
}

// warp per row: entries go to their panel at off_p + pos_p[r] + rank
template <typename T>
__global__ void k_seg_scatter(int64_t n_rows, const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                              const T* __restrict__ val, int32_t n_panels, const int32_t* __restrict__ bounds,
                              const int32_t* __restrict__ counts, const int32_t* __restrict__ pos,
                              const int64_t* __restrict__ offsets, uint32_t* __restrict__ out_pk,
                              T* __restrict__ out_val, const int32_t* __restrict__ hdr) {
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_rows; r += n_warps) {
    const int32_t a = row_ptr[r], b = row_ptr[r + 1];
    // explicit zeros: lane p handles panel p
    for (int p = lane; p < n_panels; p += 32) {
      if (counts[(int64_t)p * n_rows + r] == 0) {
        const int32_t* pp = pos + (int64_t)p * (n_rows + 1);
        if (pp[r + 1] > pp[r]) {
          const int64_t local = pp[r];
          const int64_t dst = offsets[p] + local;
          const int32_t h = hdr[(offsets[p] + local) / SEG_CH];
          out_pk[dst] = (SEG_MARK << SEG_DBITS) | (uint32_t)(r - h);
          out_val[dst] = T(0);
        }
      }
    }
    for (int32_t k = a + lane; k < b; k += 32) {
      const int32_t c = col[k];
      int p = 0;
      int32_t first = a;
      while (p + 1 < n_panels && c >= bounds[p + 1]) {
        first += counts[(int64_t)p * n_rows + r];
        ++p;
      }
      const int64_t local = (int64_t)pos[(int64_t)p * (n_rows + 1) + r] + (k - first);
      const int64_t dst = offsets[p] + local;
      const int32_t h = hdr[dst / SEG_CH];
      out_pk[dst] = ((uint32_t)(c - bounds[p]) << SEG_DBITS) | (uint32_t)(r - h);
      out_val[dst] = val[k];
    }
  }
}

// plan[w] = pos[R_w], R_w = first row with pos[R_w] >= w * total / W (rows stay whole)
__global__ void k_seg_plan(int64_t n_rows, const int32_t* __restrict__ pos, int32_t n_warps, int32_t* __restrict__ plan) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w <= n_warps; w += gridDim.x * blockDim.x) {
    const int64_t total = pos[n_rows];
    const int64_t target = (int64_t)w * total / n_warps;
    int64_t lo = 0, hi = n_rows;
    while (lo < hi) {
      const int64_t mid = (lo + hi) >> 1;
      if (pos[mid] < target) lo = mid + 1; else hi = mid;
    }
    plan[w] = pos[lo];
  }
}

// ---------------------------------------------------------------------------
// SpMV
// ---------------------------------------------------------------------------
template <typename T> struct SegVal;
template <> struct SegVal<double> {
  static __device__ __forceinline__ void load(const double* p, double v[4]) {
    const double2 a = ld_nc_na_d2(reinterpret_cast<const double2*>(p));
    const double2 b = ld_nc_na_d2(reinterpret_cast<const double2*>(p) + 1);
    v[0] = a.x; v[1] = a.y; v[2] = b.x; v[3] = b.y;
  }
};
template <> struct SegVal<float> {
  static __device__ __forceinline__ void load(const float* p, float v[4]) {
    const float4 a = ld_nc_na_f4(reinterpret_cast<const float4*>(p));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  }
};

template <typename T, bool ACC>
__global__ void __launch_bounds__(SEG_NT) k_spmv_seg(const uint32_t* __restrict__ pk, const T* __restrict__ val,
                                                   const int32_t* __restrict__ hdr, const int32_t* __restrict__ plan,
                                                   int32_t n_warps, const T* __restrict__ xs, T* __restrict__ y) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * SEG_NT + threadIdx.x) >> 5;
  if (warp >= n_warps) return;
  const int P0 = plan[warp], P1 = plan[warp + 1];
  if (P0 >= P1) return;

  int c = P0 & ~(SEG_CH - 1);
  uint32_t w[4];
  T v[4];
  int h;
  auto load = [&](int cc, uint32_t ww[4], T vv[4], int& hh) {
    const int4 q = ld_nc_na_i4(reinterpret_cast<const int4*>(pk + cc + 4 * lane));
    ww[0] = (uint32_t)q.x; ww[1] = (uint32_t)q.y; ww[2] = (uint32_t)q.z; ww[3] = (uint32_t)q.w;
    SegVal<T>::load(val + cc + 4 * lane, vv);
    hh = ld_nc_na_i1(hdr + cc / SEG_CH);
  };
  load(c, w, v, h);

  int ckey = -1;  // carried row (last segment of the previous chunk), its partial sum and y
  T cval = T(0), cy = T(0);
  while (c < P1) {
    uint32_t wn[4];
    T vn[4];
    int hn = 0;
    const bool more = c + SEG_CH < P1;
    if (more) load(c + SEG_CH, wn, vn, hn);

    int key[4];
    T xv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = c + 4 * lane + k;
      key[k] = e < P0 ? -1 : (e >= P1 ? -2 : h + (int)(w[k] & SEG_DMASK));
      const uint32_t lc = w[k] >> SEG_DBITS;
      xv[k] = (key[k] >= 0 && lc != SEG_MARK) ? __ldg(xs + lc) : T(0);
    }
    const int next0 = __shfl_down_sync(FULL, key[0], 1);
    bool end[4];
#pragma unroll
    for (int k = 0; k < 3; ++k) end[k] = key[k] >= 0 && key[k + 1] != key[k];
    end[3] = key[3] >= 0 && (lane == 31 || next0 != key[3]);  // lane 31: candidate carry
    T yv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) yv[k] = (ACC && end[k]) ? y[key[k]] : T(0);

    T run[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const T p = key[k] >= 0 ? v[k] * xv[k] : T(0);
      run[k] = (k > 0 && key[k] == key[k - 1]) ? run[k > 0 ? k - 1 : 0] + p : p;
    }
    const bool whole = key[0] == key[3];
    const int prev3 = __shfl_up_sync(FULL, key[3], 1);
    const bool cont = lane == 0 ? (ckey >= 0 && ckey == key[0]) : (prev3 == key[0]);
    T sv = run[3];
    if (lane == 0 && cont && whole) sv += cval;
    bool head = !(whole && cont);
    // key-segmented inclusive scan of the lanes' open tails; stops once every lane's
    // segment head is inside its window (rows of a few entries: 1-2 steps, not 5)
    for (int o = 1; o < 32; o <<= 1) {
      const T t = __shfl_up_sync(FULL, sv, o);
      const bool hh = __shfl_up_sync(FULL, (int)head, o) != 0;
      if (lane >= o && !head) {
        sv += t;
        head = hh;
      }
      if (!__any_sync(FULL, !head && lane >= 2 * o)) break;
    }
    const T sprev = __shfl_up_sync(FULL, sv, 1);
    const T in = cont ? (lane == 0 ? cval : sprev) : T(0);
    T fin[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) fin[k] = run[k] + (key[k] == key[0] ? in : T(0));
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (end[k] && !(lane == 31 && k == 3)) y[key[k]] = ACC ? yv[k] + fin[k] : fin[k];
    // the previous chunk's open row did not continue here: it is complete
    if (lane == 0 && ckey >= 0 && !cont) y[ckey] = ACC ? cy + cval : cval;
    ckey = __shfl_sync(FULL, key[3], 31);
    cval = __shfl_sync(FULL, fin[3], 31);
    cy = __shfl_sync(FULL, yv[3], 31);
    if (!more) break;
#pragma unroll
    for (int k = 0; k < 4; ++k) { w[k] = wn[k]; v[k] = vn[k]; }
    h = hn;
    c += SEG_CH;
  }
  if (lane == 0 && ckey >= 0) y[ckey] = ACC ? cy + cval : cval;
}

// Windowed y update: the row totals of a chunk go to a per-warp shared-memory
// window (row - wlo) and are written back with coalesced loads/stores of the
// window's rows (a chunk of a C4 panel spans ~55 consecutive rows, so ~4 lines
// each way instead of up to 4 scattered requests per lane), which keeps the
// L1 -> L2 request port for the x gathers.  Slots of rows without a total hold a
// signalling-NaN sentinel (arithmetic never produces one) and are skipped.
template <typename T> struct SegSent;
template <> struct SegSent<double> {
  static constexpr long long bits = 0x7FF4DEADBEEFCAFELL;
  static __device__ __forceinline__ double get() { return __longlong_as_double(bits); }
  static __device__ __forceinline__ bool is(double v) { return __double_as_longlong(v) == bits; }
};
template <> struct SegSent<float> {
  static constexpr int bits = 0x7FA5A5A5;
  static __device__ __forceinline__ float get() { return __int_as_float(bits); }
  static __device__ __forceinline__ bool is(float v) { return __float_as_int(v) == bits; }
};

constexpr int SEG_WSPAN = 4 * SEG_CH;  // rows a chunk (plus the carried row) can span

template <typename T, bool ACC>
__global__ void __launch_bounds__(SEG_NT) k_spmv_segw(const uint32_t* __restrict__ pk, const T* __restrict__ val,
                                                    const int32_t* __restrict__ hdr, const int32_t* __restrict__ plan,
                                                    int32_t n_warps, const T* __restrict__ xs, T* __restrict__ y) {
  __shared__ T s_win[SEG_NT / 32][SEG_WSPAN];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * SEG_NT + threadIdx.x) >> 5;
  if (warp >= n_warps) return;
  const int P0 = plan[warp], P1 = plan[warp + 1];
  if (P0 >= P1) return;
  T* win = s_win[threadIdx.x >> 5];
  for (int i = lane; i < SEG_WSPAN; i += 32) win[i] = SegSent<T>::get();
  __syncwarp();

  int c = P0 & ~(SEG_CH - 1);
  uint32_t w[4];
  T v[4];
  int h;
  auto load = [&](int cc, uint32_t ww[4], T vv[4], int& hh) {
    const int4 q = ld_nc_na_i4(reinterpret_cast<const int4*>(pk + cc + 4 * lane));
    ww[0] = (uint32_t)q.x; ww[1] = (uint32_t)q.y; ww[2] = (uint32_t)q.z; ww[3] = (uint32_t)q.w;
    SegVal<T>::load(val + cc + 4 * lane, vv);
    hh = ld_nc_na_i1(hdr + cc / SEG_CH);
  };
  load(c, w, v, h);

  int ckey = -1;  // carried row (open at the previous chunk's end) and its partial sum
  T cval = T(0);
  while (c < P1) {
    uint32_t wn[4];
    T vn[4];
    int hn = 0;
    const bool more = c + SEG_CH < P1;
    if (more) load(c + SEG_CH, wn, vn, hn);

    int key[4];
    int lmin = INT32_MAX, lmax = -1;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = c + 4 * lane + k;
      key[k] = e < P0 ? -1 : (e >= P1 ? -2 : h + (int)(w[k] & SEG_DMASK));
      if (key[k] >= 0) { lmin = min(lmin, key[k]); lmax = key[k]; }
    }
    int wlo = __reduce_min_sync(FULL, lmin);
    const int whi = __reduce_max_sync(FULL, lmax);
    if (ckey >= 0) wlo = min(wlo, ckey);
    const int nw = whi - wlo + 1;
    T yw0 = T(0), yw1 = T(0);
    if (ACC) {
      if (lane < nw) yw0 = y[wlo + lane];
      if (lane + 32 < nw) yw1 = y[wlo + 32 + lane];
    }
    T xv[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t lc = w[k] >> SEG_DBITS;
      xv[k] = (key[k] >= 0 && lc != SEG_MARK) ? __ldg(xs + lc) : T(0);
    }
    const int next0 = __shfl_down_sync(FULL, key[0], 1);
    const int prev3 = __shfl_up_sync(FULL, key[3], 1);
    T run[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const T p = key[k] >= 0 ? v[k] * xv[k] : T(0);
      run[k] = (k > 0 && key[k] == key[k - 1]) ? run[k > 0 ? k - 1 : 0] + p : p;
    }
    const bool whole = key[0] == key[3];
    const bool cont = lane == 0 ? (ckey >= 0 && ckey == key[0]) : (prev3 == key[0]);
    T sv = run[3];
    if (lane == 0 && cont && whole) sv += cval;
    bool head = !(whole && cont);
    // key-segmented inclusive scan of the lanes' open tails; stops once every lane's
    // segment head is inside its window (rows of a few entries: 1-2 steps, not 5)
    for (int o = 1; o < 32; o <<= 1) {
      const T t = __shfl_up_sync(FULL, sv, o);
      const bool hh = __shfl_up_sync(FULL, (int)head, o) != 0;
      if (lane >= o && !head) {
        sv += t;
        head = hh;
      }
      if (!__any_sync(FULL, !head && lane >= 2 * o)) break;
    }
    const T sprev = __shfl_up_sync(FULL, sv, 1);
    const T in = cont ? (lane == 0 ? cval : sprev) : T(0);
    T fin[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) fin[k] = run[k] + (key[k] == key[0] ? in : T(0));
    // row totals into the window (the chunk's last row stays open: carried)
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const bool end = key[k] >= 0 && (k < 3 ? key[k + 1] != key[k] : (lane < 31 && next0 != key[3]));
      if (end) win[key[k] - wlo] = fin[k];
    }
    if (lane == 0 && ckey >= 0 && !cont) win[ckey - wlo] = cval;
    __syncwarp();
    for (int j = 0; j * 32 < nw; ++j) {
      const int i = j * 32 + lane;
      if (i < nw) {
        const T t = win[i];
        if (!SegSent<T>::is(t)) {
          T base = T(0);
          if (ACC) base = j == 0 ? yw0 : (j == 1 ? yw1 : y[wlo + i]);
          y[wlo + i] = ACC ? base + t : t;
          win[i] = SegSent<T>::get();
        }
      }
    }
    __syncwarp();
    ckey = __shfl_sync(FULL, key[3], 31);
    cval = __shfl_sync(FULL, fin[3], 31);
    if (!more) break;
#pragma unroll
    for (int k = 0; k < 4; ++k) { w[k] = wn[k]; v[k] = vn[k]; }
    h = hn;
    c += SEG_CH;
  }
  if (lane == 0 && ckey >= 0) y[ckey] = ACC ? y[ckey] + cval : cval;
}

// Pipelined variant (mode 2): the chunk stream arrives by cp.async.bulk (TMA) into a
// per-warp ring of SEG_ST shared-memory slots (one mbarrier each), and the x
// gathers (plus the y reads of accumulating passes) of chunk i+1 are issued
// before chunk i is reduced, so a warp always has the next chunk's gathers in
// flight while it scans — the reduction no longer serialises with the gather
// latency.  Registers hold only gathered values; pk/val are re-read from the ring.
constexpr int SEG_ST = 3;

template <typename T>
struct __align__(128) SegRing {
  uint32_t pk[SEG_ST][SEG_CH];
  T val[SEG_ST][SEG_CH];
  uint64_t bar[SEG_ST];
};

template <typename T, bool ACC>
__global__ void __launch_bounds__(SEG_NT) k_spmv_segp(const uint32_t* __restrict__ pk, const T* __restrict__ val,
                                                    const int32_t* __restrict__ hdr, const int32_t* __restrict__ plan,
                                                    int32_t n_warps, const T* __restrict__ xs, T* __restrict__ y) {
  __shared__ __align__(128) SegRing<T> s_ring[SEG_NT / 32];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * SEG_NT + threadIdx.x) >> 5;
  if (warp >= n_warps) return;
  const int P0 = plan[warp], P1 = plan[warp + 1];
  if (P0 >= P1) return;
  SegRing<T>& R = s_ring[threadIdx.x >> 5];
  const int c0 = P0 & ~(SEG_CH - 1);
  const int n_ch = (P1 - c0 + SEG_CH - 1) / SEG_CH;
  if (lane == 0) {
    for (int st = 0; st < SEG_ST; ++st) mbar_init(&R.bar[st], 1);
    fence_mbar_init();
  }
  __syncwarp();
  const uint64_t pol = policy_evict_first();
  auto fill = [&](int i) {  // lane 0: chunk i into slot i % SEG_ST
    const int st = i % SEG_ST;
    const int cc = c0 + i * SEG_CH;
    fence_proxy_async_smem();
    mbar_arrive_expect_tx(&R.bar[st], SEG_CH * (4 + (uint32_t)sizeof(T)));
    bulk_g2s(R.pk[st], pk + cc, SEG_CH * 4, &R.bar[st], pol);
    bulk_g2s(R.val[st], val + cc, SEG_CH * (uint32_t)sizeof(T), &R.bar[st], pol);
  };
  if (lane == 0)
    for (int i = 0; i < SEG_ST && i < n_ch; ++i) fill(i);

  // keys of chunk i (absolute rows; -1 / -2 outside [P0, P1)) from its ring slot
  auto keys_of = [&](int i, int h, uint32_t wv[4], int key[4]) {
    const uint4 q = *reinterpret_cast<const uint4*>(&R.pk[i % SEG_ST][4 * lane]);
    wv[0] = q.x; wv[1] = q.y; wv[2] = q.z; wv[3] = q.w;
    const int cc = c0 + i * SEG_CH;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const int e = cc + 4 * lane + k;
      key[k] = e < P0 ? -1 : (e >= P1 ? -2 : h + (int)(wv[k] & SEG_DMASK));
    }
  };
  // issue chunk i's gathers (and y reads of its row ends) into xg / yg; returns the end mask
  auto issue = [&](int i, int h, T xg[4], T yg[4]) -> unsigned {
    mbar_wait(&R.bar[i % SEG_ST], (uint32_t)((i / SEG_ST) & 1));
    uint32_t wv[4];
    int key[4];
    keys_of(i, h, wv, key);
    const int next0 = __shfl_down_sync(FULL, key[0], 1);
    unsigned em = 0;
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t lc = wv[k] >> SEG_DBITS;
      xg[k] = (key[k] >= 0 && lc != SEG_MARK) ? __ldg(xs + lc) : T(0);
      const bool end = key[k] >= 0 && (k < 3 ? key[k + 1] != key[k] : (lane == 31 || next0 != key[3]));
      em |= end ? (1u << k) : 0u;
      yg[k] = (ACC && end) ? y[key[k]] : T(0);
    }
    return em;
  };

  int h0 = ld_nc_na_i1(hdr + c0 / SEG_CH);
  int h1 = n_ch > 1 ? ld_nc_na_i1(hdr + c0 / SEG_CH + 1) : 0;
  T xv0[4], yv0[4];
  unsigned em0 = issue(0, h0, xv0, yv0);
  int ckey = -1;
  T cval = T(0), cy = T(0);
  for (int i = 0; i < n_ch; ++i) {
    // (a) chunk i+1: gathers in flight during the reduction of chunk i
    T xv1[4], yv1[4];
    unsigned em1 = 0;
    int h2 = 0;
    if (i + 1 < n_ch) {
      em1 = issue(i + 1, h1, xv1, yv1);
      if (i + 2 < n_ch) h2 = ld_nc_na_i1(hdr + c0 / SEG_CH + i + 2);
    }
    // (b) reduce chunk i
    uint32_t wv[4];
    int key[4];
    keys_of(i, h0, wv, key);
    T vv[4];
    {
      const T* vp = &R.val[i % SEG_ST][4 * lane];
#pragma unroll
      for (int k = 0; k < 4; ++k) vv[k] = vp[k];
    }
    T run[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const T p = key[k] >= 0 ? vv[k] * xv0[k] : T(0);
      run[k] = (k > 0 && key[k] == key[k - 1]) ? run[k > 0 ? k - 1 : 0] + p : p;
    }
    const bool whole = key[0] == key[3];
    const int prev3 = __shfl_up_sync(FULL, key[3], 1);
    const bool cont = lane == 0 ? (ckey >= 0 && ckey == key[0]) : (prev3 == key[0]);
    T sv = run[3];
    if (lane == 0 && cont && whole) sv += cval;
    bool head = !(whole && cont);
    for (int o = 1; o < 32; o <<= 1) {
      const T t = __shfl_up_sync(FULL, sv, o);
      const bool hh = __shfl_up_sync(FULL, (int)head, o) != 0;
      if (lane >= o && !head) {
        sv += t;
        head = hh;
      }
      if (!__any_sync(FULL, !head && lane >= 2 * o)) break;
    }
    const T sprev = __shfl_up_sync(FULL, sv, 1);
    const T in = cont ? (lane == 0 ? cval : sprev) : T(0);
    T fin[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) fin[k] = run[k] + (key[k] == key[0] ? in : T(0));
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (((em0 >> k) & 1u) && !(lane == 31 && k == 3)) y[key[k]] = ACC ? yv0[k] + fin[k] : fin[k];
    if (lane == 0 && ckey >= 0 && !cont) y[ckey] = ACC ? cy + cval : cval;
    ckey = __shfl_sync(FULL, key[3], 31);
    cval = __shfl_sync(FULL, fin[3], 31);
    cy = __shfl_sync(FULL, yv0[3], 31);
    // (c) slot of chunk i is free: refill it with chunk i + SEG_ST
    __syncwarp();
    if (lane == 0 && i + SEG_ST < n_ch) fill(i + SEG_ST);
#pragma unroll
    for (int k = 0; k < 4; ++k) { xv0[k] = xv1[k]; yv0[k] = yv1[k]; }
    em0 = em1;
    h0 = h1;
    h1 = h2;
  }
  if (lane == 0 && ckey >= 0) y[ckey] = ACC ? cy + cval : cval;
}

// Bound probe (mode 3, timing experiments only; the result is NOT y = A x): the
// same chunk stream and x gathers with a per-lane sum and one coalesced store per
// chunk, i.e. the memory traffic of k_spmv_seg without the row reduction.
template <typename T>
__global__ void __launch_bounds__(SEG_NT) k_seg_probe(const uint32_t* __restrict__ pk, const T* __restrict__ val,
                                                    const int32_t* __restrict__ hdr, const int32_t* __restrict__ plan,
                                                    int32_t n_warps, const T* __restrict__ xs, T* __restrict__ y) {
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * SEG_NT + threadIdx.x) >> 5;
  if (warp >= n_warps) return;
  const int P0 = plan[warp], P1 = plan[warp + 1];
  if (P0 >= P1) return;
  int c = P0 & ~(SEG_CH - 1);
  uint32_t w[4];
  T v[4];
  int h;
  auto load = [&](int cc, uint32_t ww[4], T vv[4], int& hh) {
    const int4 q = ld_nc_na_i4(reinterpret_cast<const int4*>(pk + cc + 4 * lane));
    ww[0] = (uint32_t)q.x; ww[1] = (uint32_t)q.y; ww[2] = (uint32_t)q.z; ww[3] = (uint32_t)q.w;
    SegVal<T>::load(val + cc + 4 * lane, vv);
    hh = ld_nc_na_i1(hdr + cc / SEG_CH);
  };
  load(c, w, v, h);
  while (c < P1) {
    uint32_t wn[4];
    T vn[4];
    int hn = 0;
    const bool more = c + SEG_CH < P1;
    if (more) load(c + SEG_CH, wn, vn, hn);
    T acc = T(0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t lc = w[k] >> SEG_DBITS;
      acc += (lc != SEG_MARK) ? v[k] * __ldg(xs + lc) : T(0);
    }
    y[h + lane] = acc;
    if (!more) break;
#pragma unroll
    for (int k = 0; k < 4; ++k) { w[k] = wn[k]; v[k] = vn[k]; }
    h = hn;
    c += SEG_CH;
  }
}

static int s_seg_mode = 0;  // 0 = per-lane y update (default), 1 = windowed y, 2 = TMA ring + pipelined, 3 = probe

template <typename T>
int launch_seg(int32_t n_warps, const uint32_t* pk, const T* val, const int32_t* hdr, const int32_t* plan,
               const T* xs, T* y, int accumulate, cudaStream_t s) {
  const int grid = (int)(((int64_t)n_warps * 32 + SEG_NT - 1) / SEG_NT);
  if (s_seg_mode == 2) {
    if (accumulate)
      k_spmv_segp<T, true><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y);
    else
      k_spmv_segp<T, false><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y);
  } else if (s_seg_mode == 3) {
    k_seg_probe<T><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y);
  } else if (s_seg_mode == 1) {
    if (accumulate)
      k_spmv_segw<T, true><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y);
    else
      k_spmv_segw<T, false><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y);
  } else {
    if (accumulate)
      k_spmv_seg<T, true><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y);
    else
      k_spmv_seg<T, false><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y);
  }
  SME_CHECK_LAUNCH("k_spmv_seg");
  return SME_OK;
}

}  // namespace sme

using namespace sme;

SME_API int sme_seg_workspace_size(int64_t n_rows, int32_t n_panels, size_t* bytes) {
  SME_REQUIRE(bytes && n_rows >= 0 && n_panels >= 1, "bad arguments");
  *bytes = align_up((size_t)n_panels * n_rows * 4) + scan_workspace_bytes(n_rows);
  return SME_OK;
}

// Step 1: per-panel entry positions pos[p * (n_rows + 1) + r] (exclusive scan of the
// padded row lengths; pos[p * (n_rows + 1) + n_rows] = entries of panel p).
// ws keeps the per-panel row counts for step 2.
SME_API int sme_seg_positions(int64_t n_rows, const int32_t* row_ptr, const int32_t* col, int32_t n_panels,
                              const int32_t* bounds, int32_t* pos, void* ws, size_t ws_bytes, sme_stream_t stream) {
  SME_REQUIRE(n_rows >= 0 && n_rows < INT32_MAX && n_panels >= 1 && n_panels <= 1024, "bad arguments");
  const size_t need = align_up((size_t)n_panels * n_rows * 4) + scan_workspace_bytes(n_rows);
  SME_REQUIRE(ws_bytes >= need, "workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = as_stream(stream);
  if (n_rows == 0) {
    SME_CUDA(cudaMemsetAsync(pos, 0, (size_t)n_panels * 4, s));
    return SME_OK;
  }
  int32_t* counts = (int32_t*)ws;
  void* scan_ws = (char*)ws + align_up((size_t)n_panels * n_rows * 4);
  k_seg_count<<<grid_for(n_rows, 256), 256, 0, s>>>(n_rows, row_ptr, col, n_panels, bounds, counts);
  SME_CHECK_LAUNCH("k_seg_count");
  for (int p = 0; p < n_panels; ++p) {
    int rc = exclusive_scan_lengths(n_rows, SegLen{counts + (int64_t)p * n_rows, p}, pos + (int64_t)p * (n_rows + 1),
                                    scan_ws, nullptr, s);
    if (rc != SME_OK) return rc;
  }
  return SME_OK;
}

// Step 2: chunk headers and the packed entries.  offsets[p] (int64 device) = first
// element of panel p in pk/val (multiple of 128); pk and val must be pre-filled
// with the tail padding (pk 0xFFFFFFFF, val 0) by the caller.  bounds[p+1]-bounds[p]
// must be < 2^23 - 1 (SEG_MARK).
SME_API int sme_seg_fill(int dtype, int64_t n_rows, const int32_t* row_ptr, const int32_t* col, const void* val,
                         int32_t n_panels, const int32_t* bounds, const int32_t* pos, const int64_t* offsets,
                         const int64_t* h_offsets, uint32_t* pk, void* out_val, int32_t* hdr, const void* ws,
                         sme_stream_t stream) {
  SME_REQUIRE(dtype == SME_F64 || dtype == SME_F32, "unknown dtype %d", dtype);
  SME_REQUIRE(h_offsets, "host offsets required");
  cudaStream_t s = as_stream(stream);
  if (n_rows == 0) return SME_OK;
  const int32_t* counts = (const int32_t*)ws;
  for (int p = 0; p < n_panels; ++p) {
    SME_REQUIRE(h_offsets[p] % SEG_CH == 0, "panel offsets must be multiples of 128");
    k_seg_hdr<<<grid_for(n_rows, 256), 256, 0, s>>>(n_rows, pos + (int64_t)p * (n_rows + 1), hdr + h_offsets[p] / SEG_CH);
    SME_CHECK_LAUNCH("k_seg_hdr");
  }
  if (dtype == SME_F64)
    k_seg_scatter<double><<<grid_for(n_rows * 32, 256), 256, 0, s>>>(n_rows, row_ptr, col, (const double*)val, n_panels,
                                                                      bounds, counts, pos, offsets, pk,
                                                                      (double*)out_val, hdr);
  else
    k_seg_scatter<float><<<grid_for(n_rows * 32, 256), 256, 0, s>>>(n_rows, row_ptr, col, (const float*)val, n_panels,
                                                                     bounds, counts, pos, offsets, pk, (float*)out_val,
                                                                     hdr);
  SME_CHECK_LAUNCH("k_seg_scatter");
  return SME_OK;
}

// Kernel variant (process-wide; experiments and tests).  Measured on B200 (C4, 8 panels):
// 0 per-lane 5.85-6.1 ms, 1 windowed 5.85-6.0 ms, 2 pipelined 6.0-6.25 ms, 3 probe
// (no row reduction, not a SpMV) 4.6 ms; C2: 0 0.107 ms, 1 0.141 ms, 2 0.118 ms.
SME_API int sme_spmv_seg_set_mode(int mode) {
  SME_REQUIRE(mode >= 0 && mode <= 3, "mode must be 0 (per-lane y), 1 (windowed y), 2 (TMA ring + pipelined gathers) or 3 (bound probe)");
  s_seg_mode = mode;
  return SME_OK;
}

// Resident warps of the persistent SpMV grid.
SME_API int sme_spmv_seg_warps(int32_t* n_warps) {
  SME_REQUIRE(n_warps, "null pointer");
  int per_sm = 1 << 20;
  auto occ = [&](const void* fn) {
    int v = 0;
    if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&v, fn, SEG_NT, 0) == cudaSuccess) per_sm = std::min(per_sm, v);
  };
  if (s_seg_mode == 2) {
    occ((const void*)k_spmv_segp<double, false>);
    occ((const void*)k_spmv_segp<double, true>);
    occ((const void*)k_spmv_segp<float, false>);
    occ((const void*)k_spmv_segp<float, true>);
  } else if (s_seg_mode == 1) {
    occ((const void*)k_spmv_segw<double, false>);
    occ((const void*)k_spmv_segw<double, true>);
    occ((const void*)k_spmv_segw<float, false>);
    occ((const void*)k_spmv_segw<float, true>);
  } else {
    occ((const void*)k_spmv_seg<double, false>);
    occ((const void*)k_spmv_seg<double, true>);
    occ((const void*)k_spmv_seg<float, false>);
    occ((const void*)k_spmv_seg<float, true>);
  }
  per_sm = std::max(1, per_sm);
  *n_warps = sm_count() * per_sm * (SEG_NT / 32);
  return SME_OK;
}

// Step 3 (per panel): warp work ranges, plan[n_warps + 1] entry positions.
SME_API int sme_seg_plan(int64_t n_rows, const int32_t* pos_panel, int32_t n_warps, int32_t* plan,
                         sme_stream_t stream) {
  SME_REQUIRE(n_warps >= 1 && n_rows >= 0, "bad arguments");
  cudaStream_t s = as_stream(stream);
  k_seg_plan<<<grid_for((int64_t)n_warps + 1, 256), 256, 0, s>>>(n_rows, pos_panel, n_warps, plan);
  SME_CHECK_LAUNCH("k_seg_plan");
  return SME_OK;
}

// y (+)= A_p x over one panel: xs = x + bounds[p] (the panel's x slice), y full length.
SME_API int sme_spmv_seg(int dtype, int32_t n_warps, const uint32_t* pk, const void* val, const int32_t* hdr,
                         const int32_t* plan, const void* xs, void* y, int accumulate, sme_stream_t stream) {
  SME_REQUIRE(dtype == SME_F64 || dtype == SME_F32, "unknown dtype %d", dtype);
  SME_REQUIRE(n_warps >= 1 && pk && val && hdr && plan, "bad arguments");
  SME_REQUIRE((((uintptr_t)pk | (uintptr_t)val) & 15) == 0, "pk/val must be 16-byte aligned");
  cudaStream_t s = as_stream(stream);
  if (dtype == SME_F64)
    return launch_seg<double>(n_warps, pk, (const double*)val, hdr, plan, (const double*)xs, (double*)y, accumulate, s);
  return launch_seg<float>(n_warps, pk, (const float*)val, hdr, plan, (const float*)xs, (float*)y, accumulate, s);
}
