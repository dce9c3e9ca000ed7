// hist.cu — 2-D tile histogram and its Shannon entropy (K5/K6).
//
// Reference: histogram_2d / _counts_2d (entropy.py:91-101) = bincount of
// rbin * bc + cbin with _bin_index (entropy.py:65-67): width = n // bins and
// the last bin absorbs the remainder; shannon_entropy (entropy.py:104-119).
//
// CSR path (two kernels, same result): k_hist2d_csr_lanes (default for bins_c <=
// 128: lane-private u16 counters, C4 128x128 in 1.0 ms = 4.0 TB/s of col_idx) and
// the shared-window kernel below (any bins_c; C4 5.1 ms).
// The row bin of a nonzero only depends on which [row_ptr[e_b],
// row_ptr[e_{b+1}]) span holds its position, so the kernel never reads row ids:
// it streams col_idx once (4 B/nnz, the whole algorithmic traffic), keeps a
// window of the count grid in shared memory (u32), aggregates equal bins of a
// warp with __match_any_sync + ballot-popc before the shared atomics, and
// flushes the touched part of the window with one u64 global atomic per
// non-zero counter.  Counts are integers, so the result is bit-exact.
#include "common.cuh"

#include <algorithm>

namespace sme {

constexpr int H_NT = 512;
constexpr int H_WIN = 16384;       // u32 counters in shared memory (64 KB)
constexpr int H_EDGE_SMEM = 4096;  // row-bin edges cached in shared memory

// add `cnt` (1..4) to flat bin `bin` (-1 = nothing) with warp aggregation
__device__ __forceinline__ void warp_agg_add(int64_t bin, int cnt, uint32_t* s_cnt, int64_t win_base,
                                             int64_t win_len, unsigned long long* g_counts) {
  const int lane = threadIdx.x & 31;
  const bool valid = bin >= 0;
  // invalid lanes get a unique key so they never match anyone
  long long key = valid ? (long long)bin : -1ll - lane;
  unsigned mask = __match_any_sync(0xffffffffu, key);
  unsigned b1 = __ballot_sync(0xffffffffu, cnt >= 1), b2 = __ballot_sync(0xffffffffu, cnt >= 2);
  unsigned b3 = __ballot_sync(0xffffffffu, cnt >= 3), b4 = __ballot_sync(0xffffffffu, cnt >= 4);
  if (valid && lane == __ffs(mask) - 1) {
    unsigned tot = __popc(mask & b1) + __popc(mask & b2) + __popc(mask & b3) + __popc(mask & b4);
    int64_t off = bin - win_base;
    if (off >= 0 && off < win_len)
      atomicAdd(&s_cnt[off], tot);
    else
      atomicAdd(&g_counts[bin], (unsigned long long)tot);
  }
}

// Fold 4 flat bins (-1 = absent) into up to 4 (bin, count) slots, equal
// adjacent bins merged; returns the slot count.
__device__ __forceinline__ int fold4(const int64_t fb[4], int64_t ob[4], int oc[4]) {
  int n = 0;
#pragma unroll
  for (int i = 0; i < 4; ++i) {
    if (fb[i] < 0) continue;
    if (n > 0 && ob[n - 1] == fb[i]) {
      oc[n - 1]++;
    } else {
      ob[n] = fb[i];
      oc[n] = 1;
      ++n;
    }
  }
  return n;
}

// IP: row_ptr element type (int32_t; int64_t for nnz >= 2^31); the row-bin edges are
// kept in that type
template <bool SMEM_EDGES, typename IP = int32_t>
__global__ void __launch_bounds__(H_NT) k_hist2d_csr(int64_t n_rows, int64_t nnz, const IP* __restrict__ row_ptr,
                                                     const int32_t* __restrict__ col, int32_t br, int32_t bc,
                                                     int64_t width_r, Binner cb, unsigned long long* counts,
                                                     int64_t chunk, bool vec_ok) {
  extern __shared__ uint32_t smem[];
  uint32_t* s_cnt = smem;
  IP* s_edge = (IP*)(smem + H_WIN);
  auto edge = [&](int32_t b) -> IP {
    if (SMEM_EDGES) return s_edge[b];
    return row_ptr[b < br ? (int64_t)b * width_r : n_rows];
  };
  if (SMEM_EDGES) {
    for (int b = threadIdx.x; b <= br; b += H_NT) s_edge[b] = row_ptr[b < br ? (int64_t)b * width_r : n_rows];
    __syncthreads();
  }
  // largest b in [0, br) with edge(b) <= k
  auto rowbin = [&](int64_t k) -> int32_t {
    int32_t lo = 0, hi = br - 1;
    while (lo < hi) {
      int32_t mid = (lo + hi + 1) >> 1;
      if (edge(mid) <= k) lo = mid; else hi = mid - 1;
    }
    return lo;
  };
  const int64_t total_grid = (int64_t)br * bc;
  const uint64_t pol = policy_evict_first();
  for (int64_t k0 = (int64_t)blockIdx.x * chunk; k0 < nnz; k0 += (int64_t)gridDim.x * chunk) {
    const int64_t k1 = min(nnz, k0 + chunk);
    const int32_t b_lo = rowbin(k0), b_hi = rowbin(k1 - 1);
    const int64_t win_base = (int64_t)b_lo * bc;
    const int64_t win_len = min((int64_t)H_WIN, min(total_grid, (int64_t)(b_hi + 1) * bc) - win_base);
    for (int64_t i = threadIdx.x; i < win_len; i += H_NT) s_cnt[i] = 0;
    __syncthreads();
    // groups of 4 consecutive positions, k0 is a multiple of 4; a thread's groups
    // are increasing positions, so its row bin only ever advances (no search)
    const int64_t n_groups = (k1 - k0 + 3) >> 2;
    int32_t rb = b_lo;
    constexpr int HU = 4;  // groups in flight per thread
    for (int64_t gb = 0; gb < n_groups; gb += (int64_t)H_NT * HU) {
      int cu[HU][4];
#pragma unroll
      for (int u = 0; u < HU; ++u) {
        const int64_t g = gb + (int64_t)u * H_NT + threadIdx.x;
        const int64_t e = k0 + g * 4;
        if (g < n_groups && vec_ok && e + 3 < k1) {
          int4 v = ld_stream_i4(reinterpret_cast<const int4*>(col + e), pol);
          cu[u][0] = v.x; cu[u][1] = v.y; cu[u][2] = v.z; cu[u][3] = v.w;
        } else {
#pragma unroll
          for (int i = 0; i < 4; ++i) cu[u][i] = (g < n_groups && e + i < k1) ? col[e + i] : -1;
        }
      }
#pragma unroll 1
      for (int u = 0; u < HU; ++u) {
      const int64_t g = gb + (int64_t)u * H_NT + threadIdx.x;
      int64_t fb[4] = {-1, -1, -1, -1};
      if (g < n_groups) {
        const int64_t e = k0 + g * 4;
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          if (cu[u][i] < 0) continue;
          while (rb + 1 < br && edge(rb + 1) <= e + i) ++rb;
          fb[i] = (int64_t)rb * bc + bin_of(cu[u][i], cb);
        }
      }
      int64_t ob[4];
      int oc[4] = {0, 0, 0, 0};
      const int ns = fold4(fb, ob, oc);
      // banded inputs: the whole warp's group often lands in one bin -> one atomic;
      // otherwise (random/permuted inputs) plain shared atomics per folded slot
      const int64_t b0 = __shfl_sync(0xffffffffu, ns > 0 ? ob[0] : -1, 0);
      const bool uniform = __all_sync(0xffffffffu, ns == 0 || (ns == 1 && ob[0] == b0)) && b0 >= 0;
      if (uniform) {
        const unsigned tot = __reduce_add_sync(0xffffffffu, (unsigned)(ns ? oc[0] : 0));
        if ((threadIdx.x & 31) == 0) {
          const int64_t off = b0 - win_base;
          if (off >= 0 && off < win_len) atomicAdd(&s_cnt[off], tot);
          else atomicAdd(&counts[b0], (unsigned long long)tot);
        }
      } else {
#pragma unroll
        for (int sl = 0; sl < 4; ++sl) {
          if (sl < ns) {
            const int64_t off = ob[sl] - win_base;
            if (off >= 0 && off < win_len) atomicAdd(&s_cnt[off], (unsigned)oc[sl]);
            else atomicAdd(&counts[ob[sl]], (unsigned long long)oc[sl]);
          }
        }
      }
      }
    }
    __syncthreads();
    for (int64_t i = threadIdx.x; i < win_len; i += H_NT)
      if (s_cnt[i]) atomicAdd(&counts[win_base + i], (unsigned long long)s_cnt[i]);
    __syncthreads();
  }
}

// Lane-private counters (the default for bins_c <= 128): each warp streams a
// contiguous range of col_idx; its 32 lanes count the current row bin's column
// bins in u16 counters cnt[bin][lane] of their own (bank = lane / 2: no
// conflicts, no atomics, ~9 instructions per nonzero), so the kernel runs near the
// col_idx stream rate.  A row bin spans ~nnz/br consecutive positions, so a warp
// changes row bin at most a few times: then (and every HL_FLUSH iterations, so a
// u16 never overflows) the warp sums its counters across lanes and adds them to
// the global grid with one u64 atomic per non-zero bin.  The rare iteration that
// straddles a row-bin edge sends its entries beyond the edge straight to global
// atomics.  Integer counts: bit-exact, order-free.
constexpr int HL_MAXC = 128;
constexpr int HL_FLUSH_ENTRIES = 65000;  // per-lane entries between flushes (< 65536: a u16 never overflows)

// Counter layouts of k_hist2d_csr_lanes (CL): 0 = u16 cnt[bin][lane] (lanes 2k, 2k+1
// share a bank, so two lanes with different bins of equal parity conflict); 1 = u32
// words cnt[bin / 2][lane] holding bins 2j and 2j+1 in their halves (bank = lane: no
// conflicts), u16 load / store; 2 = the same words, one shared atomic add of
// 1 << 16 (bin & 1) per entry (no load-modify-store chain in the thread).
template <int NT, int U, bool PF, int CL = 0, typename IP = int32_t>
__global__ void __launch_bounds__(NT) k_hist2d_csr_lanes(int64_t n_rows, int64_t nnz,
                                                         const IP* __restrict__ row_ptr,
                                                         const int32_t* __restrict__ col, int32_t br, int32_t bc,
                                                         int64_t width_r, Binner cb, unsigned long long* counts,
                                                         bool vec_ok) {
  constexpr int WARPS = NT / 32;
  extern __shared__ uint32_t smem[];
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  uint16_t* cnt = reinterpret_cast<uint16_t*>(smem) + (size_t)wib * HL_MAXC * 32;  // [bin][lane]
  uint32_t* cnt32 = reinterpret_cast<uint32_t*>(cnt);                                // CL 1, 2: [bin / 2][lane]
  auto inc = [&](int32_t bin) {
    if (CL == 0) {
      uint16_t* p = cnt + bin * 32 + lane;
      *p = (uint16_t)(*p + 1);
    } else if (CL == 1) {
      uint16_t* p = cnt + ((((bin >> 1) << 5) + lane) << 1) + (bin & 1);
      *p = (uint16_t)(*p + 1);
    } else {
      atomicAdd(cnt32 + ((bin >> 1) << 5) + lane, 1u << ((bin & 1) << 4));
    }
  };
  IP* s_edge = reinterpret_cast<IP*>(smem + WARPS * HL_MAXC * 16);
  for (int b = threadIdx.x; b <= br; b += NT) s_edge[b] = row_ptr[b < br ? (int64_t)b * width_r : n_rows];
  for (int i = lane; i < HL_MAXC * 32; i += 32) cnt[i] = 0;
  __syncthreads();
  auto rowbin = [&](int64_t k) -> int32_t {  // largest b in [0, br) with edge(b) <= k
    int32_t lo = 0, hi = br - 1;
    while (lo < hi) {
      const int32_t mid = (lo + hi + 1) >> 1;
      if (s_edge[mid] <= k) lo = mid; else hi = mid - 1;
    }
    return lo;
  };
  // this warp's range, 4-aligned
  const int64_t n_warps = (int64_t)gridDim.x * WARPS;
  const int64_t w = (int64_t)blockIdx.x * WARPS + wib;
  const int64_t q = (nnz + 3) / 4;
  const int64_t w0 = (q * w / n_warps) * 4, w1 = min(nnz, (q * (w + 1) / n_warps) * 4);
  if (w0 >= w1) return;
  const uint64_t pol = policy_evict_first();
  int32_t rbw = rowbin(w0);
  int64_t E = rbw + 1 < br ? (int64_t)s_edge[rbw + 1] : INT64_MAX;  // end of row bin rbw
  auto flush = [&]() {
    __syncwarp();
    if (CL == 0) {
      for (int c = lane; c < bc; c += 32) {
        uint32_t t = 0;
        for (int j = 0; j < 32; ++j) {
          const int jj = (j + lane) & 31;
          t += cnt[c * 32 + jj];
          cnt[c * 32 + jj] = 0;
        }
        if (t) atomicAdd(&counts[(int64_t)rbw * bc + c], (unsigned long long)t);
      }
    } else {
      for (int c2 = lane; 2 * c2 < bc; c2 += 32) {
        uint32_t t0 = 0, t1 = 0;
        for (int j = 0; j < 32; ++j) {
          const int idx = c2 * 32 + ((j + lane) & 31);
          const uint32_t wv = cnt32[idx];
          t0 += wv & 0xffffu;
          t1 += wv >> 16;
          cnt32[idx] = 0;
        }
        if (t0) atomicAdd(&counts[(int64_t)rbw * bc + 2 * c2], (unsigned long long)t0);
        if (t1 && 2 * c2 + 1 < bc) atomicAdd(&counts[(int64_t)rbw * bc + 2 * c2 + 1], (unsigned long long)t1);
      }
    }
    __syncwarp();
  };
  constexpr int64_t SPAN = (int64_t)32 * 4 * U;  // positions per warp iteration
  constexpr int FLUSH_ITERS = HL_FLUSH_ENTRIES / (4 * U);
  int since_flush = 0;
  auto load = [&](int64_t base, int (&c4)[U][4]) {
#pragma unroll
    for (int u = 0; u < U; ++u) {
      const int64_t e = base + ((int64_t)u * 32 + lane) * 4;
      if (vec_ok && e + 3 < w1) {
        const int4 v = ld_stream_i4(reinterpret_cast<const int4*>(col + e), pol);
        c4[u][0] = v.x; c4[u][1] = v.y; c4[u][2] = v.z; c4[u][3] = v.w;
      } else {
#pragma unroll
        for (int i = 0; i < 4; ++i) c4[u][i] = (e + i < w1) ? col[e + i] : -1;
      }
    }
  };
  int cur[U][4];
  load(w0, cur);
  for (int64_t base = w0; base < w1; base += SPAN) {
    int nxt[U][4];
    if (PF && base + SPAN < w1) load(base + SPAN, nxt);  // next iteration's loads in flight during this one
    if (base + SPAN <= E) {  // the whole iteration lies in row bin rbw (warp-uniform)
      if (CL != 0 && base + SPAN <= w1) {  // interior: every position valid (warp-uniform)
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int i = 0; i < 4; ++i) inc(bin_of(cur[u][i], cb));
      } else {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int i = 0; i < 4; ++i)
            if (cur[u][i] >= 0) inc(bin_of(cur[u][i], cb));
      }
      if (++since_flush == FLUSH_ITERS) {
        flush();
        since_flush = 0;
      }
    } else {  // straddles one or more row-bin edges: entries past E go to global atomics
#pragma unroll
      for (int u = 0; u < U; ++u)
#pragma unroll
        for (int i = 0; i < 4; ++i) {
          const int64_t e = base + ((int64_t)u * 32 + lane) * 4 + i;
          if (cur[u][i] < 0) continue;
          const int32_t cbin = bin_of(cur[u][i], cb);
          if (e < E) {
            inc(cbin);
          } else {
            atomicAdd(&counts[(int64_t)rowbin(e) * bc + cbin], 1ull);
          }
        }
      // the warp's row bin moves to the next iteration's first position
      flush();
      since_flush = 0;
      if (base + SPAN < w1) {
        rbw = rowbin(base + SPAN);
        E = rbw + 1 < br ? (int64_t)s_edge[rbw + 1] : INT64_MAX;
      }
    }
    if (base + SPAN < w1) {
      if (PF) {
#pragma unroll
        for (int u = 0; u < U; ++u)
#pragma unroll
          for (int i = 0; i < 4; ++i) cur[u][i] = nxt[u][i];
      } else {
        load(base + SPAN, cur);
      }
    }
  }
  flush();
}

template <int NT, int U, bool PF, int CL = 0, typename IP = int32_t>
static int launch_hist_lanes(int64_t n_rows, int64_t nnz, const IP* row_ptr, const int32_t* col, int32_t br,
                             int32_t bc, int64_t width_r, Binner cb, unsigned long long* counts, bool vec_ok,
                             bool one_cta, cudaStream_t s) {
  auto kern = k_hist2d_csr_lanes<NT, U, PF, CL, IP>;
  const size_t sm = (size_t)(NT / 32) * HL_MAXC * 32 * 2 + ((size_t)br + 1) * sizeof(IP);
  SME_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)sm));
  const int64_t need = (nnz + 4095) / 4096;  // >= 4096 positions per CTA
  const int grid = one_cta ? 1 : (int)std::max<int64_t>(1, std::min<int64_t>(sm_count(), need));
  kern<<<grid, NT, sm, s>>>(n_rows, nnz, row_ptr, col, br, bc, width_r, cb, counts, vec_ok);
  SME_CHECK_LAUNCH("k_hist2d_csr_lanes");
  return SME_OK;
}

// COO triplets in any order: full grid in shared memory when it fits (window at 0),
// otherwise the out-of-window bins go to global atomics.
__global__ void __launch_bounds__(H_NT) k_hist2d_coo(int64_t nnz, const int32_t* __restrict__ row,
                                                     const int32_t* __restrict__ col, int32_t bc, Binner rb,
                                                     Binner cb, int64_t total_grid, unsigned long long* counts) {
  extern __shared__ uint32_t s_cnt[];
  const int64_t win_len = min((int64_t)H_WIN, total_grid);
  for (int64_t i = threadIdx.x; i < win_len; i += H_NT) s_cnt[i] = 0;
  __syncthreads();
  const int64_t stride = (int64_t)gridDim.x * H_NT;
  const int64_t n_iter = (nnz + stride - 1) / stride;
  for (int64_t it = 0; it < n_iter; ++it) {
    int64_t k = it * stride + (int64_t)blockIdx.x * H_NT + threadIdx.x;
    int64_t b = -1;
    if (k < nnz) b = (int64_t)bin_of(row[k], rb) * bc + bin_of(col[k], cb);
    warp_agg_add(b, b >= 0 ? 1 : 0, s_cnt, 0, win_len, counts);
  }
  __syncthreads();
  for (int64_t i = threadIdx.x; i < win_len; i += H_NT)
    if (s_cnt[i]) atomicAdd(&counts[i], (unsigned long long)s_cnt[i]);
}

template <typename IP>
__global__ void k_row_hist_csr(int64_t n_rows, const IP* __restrict__ row_ptr, int32_t bins, int64_t width,
                               int64_t* counts) {
  for (int b = blockIdx.x * blockDim.x + threadIdx.x; b < bins; b += gridDim.x * blockDim.x) {
    int64_t lo = (int64_t)b * width, hi = (b + 1 < bins) ? (int64_t)(b + 1) * width : n_rows;
    counts[b] += (int64_t)row_ptr[hi] - row_ptr[lo];
  }
}

// -sum p log p over the bins in a fixed order (thread-strided sums, then a fixed
// tree): deterministic.  total by exact int64 reduction first.
__global__ void __launch_bounds__(1024) k_entropy(int64_t n, const int64_t* __restrict__ counts, double base,
                                                  double* out, int64_t* total_out) {
  __shared__ long long s_tot[32];
  __shared__ double s_h[32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  long long t = 0;
  for (int64_t i = threadIdx.x; i < n; i += 1024) t += counts[i];
  for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
  if (lane == 0) s_tot[warp] = t;
  __syncthreads();
  if (warp == 0) {
    long long v = s_tot[lane];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) s_tot[0] = v;
  }
  __syncthreads();
  const long long total = s_tot[0];
  const bool base2 = (base == 2.0);
  double h = 0.0;
  if (total > 0) {
    const double dt = (double)total;
    for (int64_t i = threadIdx.x; i < n; i += 1024) {
      long long c = counts[i];
      if (c > 0) {
        double p = (double)c / dt;
        h += p * (base2 ? log2(p) : log(p));
      }
    }
  }
  for (int o = 16; o; o >>= 1) h += __shfl_xor_sync(0xffffffffu, h, o);
  if (lane == 0) s_h[warp] = h;
  __syncthreads();
  if (warp == 0) {
    double v = s_h[lane];
    for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
    if (lane == 0) {
      double r = -v;
      if (!base2) r = r / log(base);
      *out = r;
      if (total_out) *total_out = total;
    }
  }
}

}  // namespace sme

using namespace sme;

// 0 = lane-private counters when bins_c <= 128 (default), 1 = shared-atomic window
// kernel, 2 = lane counters on a single CTA (tests: long warp ranges)
static int s_hist_mode = 0;
// lane-kernel tiling (experiments): 0 = 864 x 4 loads (768 x 4 when br > ~1500),
// others see the dispatch; measured C4: 864x4 1.00 ms, 768x4 1.06, 512x8 1.25
static int s_hist_variant = 0;

SME_API int sme_hist2d_set_variant(int v) {
  SME_REQUIRE(v >= 0 && v <= 12, "variant must be in [0, 12]");
  s_hist_variant = v;
  return SME_OK;
}

SME_API int sme_hist2d_set_mode(int mode) {
  SME_REQUIRE(mode >= 0 && mode <= 2, "mode must be 0 (lane counters), 1 (shared atomics) or 2 (one CTA)");
  s_hist_mode = mode;
  return SME_OK;
}

static int check_bins(int64_t n, int32_t bins, const char* what) {
  SME_REQUIRE(bins >= 1, "%s bin count must be >= 1", what);
  SME_REQUIRE(bins <= n, "%s bin count %d exceeds dimension %lld", what, bins, (long long)n);
  return SME_OK;
}

SME_API int sme_hist2d_csr(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* row_ptr, const int32_t* col,
                           int32_t bins_r, int32_t bins_c, int64_t* counts, sme_stream_t stream) {
  int rc;
  if ((rc = check_bins(n_rows, bins_r, "row")) != SME_OK) return rc;
  if ((rc = check_bins(n_cols, bins_c, "column")) != SME_OK) return rc;
  SME_REQUIRE(nnz >= 0 && nnz < INT32_MAX && n_cols < INT32_MAX, "sizes exceed int32");
  if (nnz == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  Binner cb = make_binner(n_cols, bins_c);
  int64_t width_r = n_rows / bins_r;
  int blocks_cap = sm_count() * 2;
  int64_t chunk = (nnz + blocks_cap - 1) / blocks_cap;
  chunk = ((chunk + 4095) / 4096) * 4096;  // multiple of 4 (aligned int4) and of the tile
  int blocks = (int)((nnz + chunk - 1) / chunk);
  size_t smem = H_WIN * 4 + (H_EDGE_SMEM + 1) * 4;
  const bool vec_ok = ((uintptr_t)col & 15) == 0;
  if (bins_c <= HL_MAXC && bins_r <= H_EDGE_SMEM && s_hist_mode != 1) {
    auto ull = (unsigned long long*)counts;
    const bool one = s_hist_mode == 2;
    const bool fits864 = (size_t)27 * HL_MAXC * 64 + ((size_t)bins_r + 1) * 4 <= 227 * 1024;
    int variant = s_hist_variant;
    if (!fits864 && (variant == 5 || variant == 6)) variant = 1;  // 27 warps of counters + edges > 227 KB
    switch (variant) {
      case 1: return launch_hist_lanes<768, 4, false>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
      case 2: return launch_hist_lanes<512, 4, true>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
      case 3: return launch_hist_lanes<768, 2, true>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
      case 4: return launch_hist_lanes<640, 4, true>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
      case 5: return launch_hist_lanes<864, 4, false>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
      case 6: return launch_hist_lanes<864, 2, false>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
      case 7: return launch_hist_lanes<512, 8, false>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
      case 8:
        if (fits864) return launch_hist_lanes<864, 4, false, 1>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
        return launch_hist_lanes<768, 4, false, 1>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
      case 9:
        if (fits864) return launch_hist_lanes<864, 4, false, 2>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
        return launch_hist_lanes<768, 4, false, 2>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
      case 10: return launch_hist_lanes<864, 2, false, 2>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
      case 11: return launch_hist_lanes<640, 4, true, 2>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
      case 12: return launch_hist_lanes<512, 8, false, 2>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
      default:  // 27 warps of counters (221 KB) when the row-bin edges fit beside them, else 24;
                // conflict-free counter words with shared atomic adds (CL 2: C4 0.996 -> 0.745 ms)
        if (fits864)
          return launch_hist_lanes<864, 4, false, 2>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
        return launch_hist_lanes<768, 4, false, 2>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull, vec_ok, one, s);
    }
  } else if (bins_r <= H_EDGE_SMEM) {
    SME_CUDA(cudaFuncSetAttribute(k_hist2d_csr<true>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_hist2d_csr<true><<<blocks, H_NT, smem, s>>>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb,
                                                  (unsigned long long*)counts, chunk, vec_ok);
  } else {
    SME_CUDA(cudaFuncSetAttribute(k_hist2d_csr<false>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_hist2d_csr<false><<<blocks, H_NT, smem, s>>>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb,
                                                   (unsigned long long*)counts, chunk, vec_ok);
  }
  SME_CHECK_LAUNCH("k_hist2d_csr");
  return SME_OK;
}

// int64 row_ptr (nnz >= 2^31): the default lane-counter tiling (bins_c <= 128) or the
// row-bin window kernel, edges kept as int64
SME_API int sme_hist2d_csr_i64(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                               const int32_t* col, int32_t bins_r, int32_t bins_c, int64_t* counts,
                               sme_stream_t stream) {
  int rc;
  if ((rc = check_bins(n_rows, bins_r, "row")) != SME_OK) return rc;
  if ((rc = check_bins(n_cols, bins_c, "column")) != SME_OK) return rc;
  SME_REQUIRE(nnz >= 0 && n_cols < INT32_MAX, "bad sizes");
  if (nnz == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  Binner cb = make_binner(n_cols, bins_c);
  const int64_t width_r = n_rows / bins_r;
  const bool vec_ok = ((uintptr_t)col & 15) == 0;
  auto ull = (unsigned long long*)counts;
  if (bins_c <= HL_MAXC && bins_r <= H_EDGE_SMEM) {
    const bool fits864 = (size_t)27 * HL_MAXC * 64 + ((size_t)bins_r + 1) * 8 <= 227 * 1024;
    if (fits864)
      return launch_hist_lanes<864, 4, false, 2, int64_t>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull,
                                                           vec_ok, false, s);
    return launch_hist_lanes<768, 4, false, 2, int64_t>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull,
                                                         vec_ok, false, s);
  }
  const int blocks_cap = sm_count() * 2;
  int64_t chunk = (nnz + blocks_cap - 1) / blocks_cap;
  chunk = ((chunk + 4095) / 4096) * 4096;
  const int blocks = (int)((nnz + chunk - 1) / chunk);
  const size_t smem = H_WIN * 4 + (H_EDGE_SMEM + 1) * 8;
  if (bins_r <= H_EDGE_SMEM) {
    SME_CUDA(cudaFuncSetAttribute(k_hist2d_csr<true, int64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_hist2d_csr<true, int64_t><<<blocks, H_NT, smem, s>>>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull,
                                                           chunk, vec_ok);
  } else {
    SME_CUDA(cudaFuncSetAttribute(k_hist2d_csr<false, int64_t>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
    k_hist2d_csr<false, int64_t><<<blocks, H_NT, smem, s>>>(n_rows, nnz, row_ptr, col, bins_r, bins_c, width_r, cb, ull,
                                                            chunk, vec_ok);
  }
  SME_CHECK_LAUNCH("k_hist2d_csr");
  return SME_OK;
}

SME_API int sme_hist2d_coo(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* row, const int32_t* col,
                           int32_t bins_r, int32_t bins_c, int64_t* counts, sme_stream_t stream) {
  int rc;
  if ((rc = check_bins(n_rows, bins_r, "row")) != SME_OK) return rc;
  if ((rc = check_bins(n_cols, bins_c, "column")) != SME_OK) return rc;
  // entry positions are int64 (COO triplets of any count); row / column ids int32
  SME_REQUIRE(nnz >= 0 && n_rows < INT32_MAX && n_cols < INT32_MAX, "sizes exceed int32");
  if (nnz == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  Binner rb = make_binner(n_rows, bins_r), cb = make_binner(n_cols, bins_c);
  size_t smem = H_WIN * 4;
  SME_CUDA(cudaFuncSetAttribute(k_hist2d_coo, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
  int blocks = grid_for(nnz, H_NT, 2);
  k_hist2d_coo<<<blocks, H_NT, smem, s>>>(nnz, row, col, bins_c, rb, cb, (int64_t)bins_r * bins_c,
                                          (unsigned long long*)counts);
  SME_CHECK_LAUNCH("k_hist2d_coo");
  return SME_OK;
}

template <typename IP>
static int row_hist_impl(int64_t n_rows, const IP* row_ptr, int32_t bins, int64_t* counts, sme_stream_t stream) {
  int rc;
  if ((rc = check_bins(n_rows, bins, "row")) != SME_OK) return rc;
  cudaStream_t s = as_stream(stream);
  k_row_hist_csr<IP><<<(bins + 255) / 256, 256, 0, s>>>(n_rows, row_ptr, bins, n_rows / bins, counts);
  SME_CHECK_LAUNCH("k_row_hist_csr");
  return SME_OK;
}

SME_API int sme_row_hist_csr(int64_t n_rows, const int32_t* row_ptr, int32_t bins, int64_t* counts,
                             sme_stream_t stream) {
  return row_hist_impl(n_rows, row_ptr, bins, counts, stream);
}

SME_API int sme_row_hist_csr_i64(int64_t n_rows, const int64_t* row_ptr, int32_t bins, int64_t* counts,
                                 sme_stream_t stream) {
  return row_hist_impl(n_rows, row_ptr, bins, counts, stream);
}

SME_API int sme_entropy(int64_t n_bins, const int64_t* counts, double base, double* out, int64_t* total,
                        sme_stream_t stream) {
  SME_REQUIRE(n_bins >= 1, "histogram has no bins");
  SME_REQUIRE(base > 0.0 && base != 1.0, "entropy base must be > 0 and != 1");
  cudaStream_t s = as_stream(stream);
  k_entropy<<<1, 1024, 0, s>>>(n_bins, counts, base, out, total);
  SME_CHECK_LAUNCH("k_entropy");
  return SME_OK;
}

namespace sme {
// Lazy module loading (CUDA 12 default) loads this file's module on the first launch of
// any of its kernels, ~10-20 ms each; sme_preload() does it ahead of time.
int preload_hist() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)k_hist2d_coo) == cudaSuccess ? 0 : -1;
}
}  // namespace sme
