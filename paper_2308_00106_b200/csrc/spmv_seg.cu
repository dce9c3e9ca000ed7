// spmv_seg.cu — the "segmented chunk" SpMV layout and kernel: the fast path for
// randomly permuted matrices (short, uniform rows; x gathers that only an
// L2-resident x slice can serve).
//
// Reference: spmv_csr / _accumulate_rows (kernels.py:59-78): y_i = sum_k v_k x[c_k]
// over row i, empty rows give 0.  Same products; the row sums are associated
// in chunk order instead of numpy's pairwise order (tolerance 1e-12, the
// reference's CORRECTNESS_RTOL, bench.py:34).
//
// What bounds it.  After a random permutation the x gathers of a CSR SpMV are
// uniformly random: every gather is its own 128-B line, i.e. one L1 -> L2
// request.  The SM's L1 -> crossbar request port takes about one request per
// clock (ncu l1tex__m_l1tex2xbar_req_cycles_active: 80-87 % busy in every
// variant measured), so a 1e9-nonzero SpMV needs >= 1e9 / (148 SMs x clock)
// no matter how it is written — 3.4 ms at 1965 MHz, 3.8 ms at the ~1760 MHz
// the part settles at under its 1 kW cap.  LDG is the best gather path (TMA
// gather4 120 G rows/s, per-lane bulk copies 63 G/s, LDG 285 G/s:
// tools/gather_bench.cu).  Everything else the kernel does must cost a small
// fraction of one request per nonzero:
//   * no row_ptr: each 32-bit entry packs the panel-local column (23 bits), an
//     end-of-row flag (1 bit) and the row offset from its 128-entry chunk's
//     header row (8 bits), so a pass streams 4 + sizeof(value) bytes per entry;
//   * a warp reads a 128-entry chunk with three coalesced 128-bit loads per
//     lane (pk, and val as 2 x 16 B), gathers 4 x values per lane, and sums
//     rows from the end flags: in-lane runs, then one shuffle of each lane's
//     open tail to the next lane (a longer chain of whole-lane rows takes a
//     segmented scan, ballot-detected and rare);
//   * the lane holding a row's last entry writes (panel 0) or accumulates
//     (panels p > 0) y — with a fire-and-forget RED.ADD.F64 at L2, so no y read
//     crosses back to the SM (each row has one adder per pass and the passes are
//     ordered launches: deterministic, same bits as load + add + store).
//
// Layout of one panel (columns [b_p, b_{p+1})), n_pad = round_up(entries, 128):
//   pk[n_pad]  uint32  (col - b_p) << 9 | end << 8 | (row - hdr[chunk])
//                      (col field 0x7FFFFF = explicit zero: no gather, product 0)
//   val[n_pad] f64/f32 (0 for explicit zeros and tail padding)
//   hdr[n_pad / 128] int32 row of the chunk's first entry
// Rows keep their CSR (row-major, column-ascending) order.  Explicit zeros are
// added (a) in panel 0 for every row without entries there, so the
// non-accumulating pass writes every y row, and (b) in later panels for empty
// rows r with r % 2 == 0, so consecutive entries are at most 2 rows apart and a
// 128-entry chunk spans at most 254 rows (fits the 8-bit offset).
//
// Work split: warp w of the persistent grid owns entry positions
// [plan[w], plan[w+1]), which always start and end on row boundaries: rows are
// whole within one warp (every y row has exactly one writer: deterministic) and
// nothing is carried across a warp boundary.
#include "common.cuh"
#include "scan.cuh"

#include <algorithm>

namespace sme {

constexpr int SEG_NT = 256;
static bool s_seg_scatter_groups = true;  // sme_seg_set_scatter_groups
static bool s_seg_fill_ballot = true;     // sme_seg_set_fill_ballot
static bool s_seg_fill_direct = true;    // sme_seg_set_fill_direct
constexpr int SEG_CH = 128;
constexpr int SEG_DBITS = 8;
constexpr uint32_t SEG_DMASK = (1u << SEG_DBITS) - 1;
constexpr uint32_t SEG_END = 1u << SEG_DBITS;
constexpr int SEG_CSHIFT = SEG_DBITS + 1;
constexpr uint32_t SEG_MARK = (1u << (32 - SEG_CSHIFT)) - 1;  // col field of an explicit zero
constexpr int SEG_GAP = 2;                                    // padding stride of empty rows (p > 0)
// row-total staging (CMP, see seg_warp_body) pays for f64 (C4 -3.8 %, C5 -3 %) but not for
// f32 (C3 +7 %: 4-byte y words already share lines, and the scan's instructions dominate)
template <typename T>
constexpr bool kStageRows = sizeof(T) == 8;

// ---------------------------------------------------------------------------
// layout build
// ---------------------------------------------------------------------------

// counts[p * n + r] = entries of row r in panel p (rows are column-sorted)
// IP: row_ptr element type (int32_t; int64_t for nnz >= 2^31 — the per-panel positions
// stay int32: every panel holds < 2^31 slots)
template <typename IP>
__global__ void k_seg_count(int64_t n_rows, const IP* __restrict__ row_ptr, const int32_t* __restrict__ col,
                            int32_t n_panels, const int32_t* __restrict__ bounds, int32_t* __restrict__ counts) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    const IP a = row_ptr[r], b = row_ptr[r + 1];
    IP k = a;
    for (int p = 0; p < n_panels; ++p) {
      const int32_t hi = bounds[p + 1];
      // binary search for the first column >= hi in [k, b)
      IP lo = k, up = b;
      while (lo < up) {
        const IP mid = (lo + up) >> 1;
        if (col[mid] < hi) lo = mid + 1; else up = mid;
      }
      counts[(int64_t)p * n_rows + r] = (int32_t)(lo - k);
      k = lo;
    }
  }
}

// entries of row r in the panel layout: its count, or one explicit zero (every
// row of panel 0, of the last panel when `full` (the epilogue pass of
// sme_spmv_seg_epi must visit every row), and even rows of the others)
struct SegLen {
  const int32_t* counts;  // this panel's counts
  int32_t panel;
  bool full;
  __device__ __forceinline__ int64_t operator()(int64_t r) const {
    const int32_t c = counts[r];
    return c > 0 ? c : ((panel == 0 || full || (r % SEG_GAP) == 0) ? 1 : 0);
  }
};

// hdr[c] = row of the entry at position 128 c (one panel)
__global__ void k_seg_hdr(int64_t n_rows, const int32_t* __restrict__ pos, int32_t* __restrict__ hdr) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = pos[r], b = pos[r + 1];
    for (int32_t c = (a + SEG_CH - 1) / SEG_CH; c * SEG_CH < b; ++c) hdr[c] = (int32_t)r;
  }
}

// warp per row: entries go to their panel at off_p + pos_p[r] + rank.  Lane p < P
// holds panel p's per-row data (count, position, panel offset, first entry of the
// row in that panel); an entry finds its panel among the bounds and takes the
// panel's data by shuffle — no per-entry walk over the panels' count arrays.
template <typename T, typename IP>
__global__ void k_seg_scatter(int64_t n_rows, const IP* __restrict__ row_ptr, const int32_t* __restrict__ col,
                              const T* __restrict__ val, int32_t n_panels, const int32_t* __restrict__ bounds,
                              const int32_t* __restrict__ counts, const int32_t* __restrict__ pos,
                              const int64_t* __restrict__ offsets, uint32_t* __restrict__ out_pk,
                              T* __restrict__ out_val, const int32_t* __restrict__ hdr) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  const bool direct = n_panels <= 32;
  const int32_t my_hi = (direct && lane < n_panels) ? bounds[lane + 1] : INT32_MAX;
  const int32_t my_lo = (direct && lane < n_panels) ? bounds[lane] : 0;
  const int64_t my_off = (direct && lane < n_panels) ? offsets[lane] : 0;
  for (int64_t r = warp; r < n_rows; r += n_warps) {
    const IP a = row_ptr[r], b = row_ptr[r + 1];
    if (!direct) {  // > 32 panels: walk the count arrays (rare, small matrices)
      for (int p = lane; p < n_panels; p += 32) {
        if (counts[(int64_t)p * n_rows + r] == 0) {
          const int32_t* pp = pos + (int64_t)p * (n_rows + 1);
          if (pp[r + 1] > pp[r]) {
            const int64_t dst = offsets[p] + pp[r];
            out_pk[dst] = (SEG_MARK << SEG_CSHIFT) | SEG_END | (uint32_t)(r - hdr[dst / SEG_CH]);
            out_val[dst] = T(0);
          }
        }
      }
      for (IP k = a + lane; k < b; k += 32) {
        const int32_t c = col[k];
        int p = 0;
        IP first = a;
        while (p + 1 < n_panels && c >= bounds[p + 1]) {
          first += counts[(int64_t)p * n_rows + r];
          ++p;
        }
        const int64_t dst = offsets[p] + (int64_t)pos[(int64_t)p * (n_rows + 1) + r] + (k - first);
        const bool last = k - first == counts[(int64_t)p * n_rows + r] - 1;
        out_pk[dst] = ((uint32_t)(c - bounds[p]) << SEG_CSHIFT) | (last ? SEG_END : 0u) |
                      (uint32_t)(r - hdr[dst / SEG_CH]);
        out_val[dst] = val[k];
      }
      continue;
    }
    int32_t cnt = 0, ppos = 0, pnext = 0;
    if (lane < n_panels) {
      cnt = counts[(int64_t)lane * n_rows + r];
      const int32_t* pp = pos + (int64_t)lane * (n_rows + 1);
      ppos = pp[r];
      pnext = pp[r + 1];
    }
    // first entry of the row in panel `lane`: exclusive prefix of the counts
    int32_t incl = cnt;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    const IP first = a + incl - cnt;
    // explicit zero of this row in panel `lane`
    if (lane < n_panels && cnt == 0 && pnext > ppos) {
      const int64_t dst = my_off + ppos;
      out_pk[dst] = (SEG_MARK << SEG_CSHIFT) | SEG_END | (uint32_t)(r - hdr[dst / SEG_CH]);
      out_val[dst] = T(0);
    }
    for (IP k0 = a; k0 < b; k0 += 32) {
      const IP k = k0 + lane;
      const int32_t c = k < b ? col[k] : INT32_MAX;
      // panel of c: number of panel upper bounds <= c (bounds held by lanes)
      int p = 0;
      for (int q = 0; q < n_panels; ++q) p += (c >= __shfl_sync(FULL, my_hi, q)) ? 1 : 0;
      if (p >= n_panels) p = n_panels - 1;
      const IP f = __shfl_sync(FULL, first, p);
      const int32_t pc = __shfl_sync(FULL, cnt, p);
      const int32_t pp = __shfl_sync(FULL, ppos, p);
      const int64_t po = __shfl_sync(FULL, my_off, p);
      const int32_t lo = __shfl_sync(FULL, my_lo, p);
      if (k < b) {
        const int64_t dst = po + pp + (int64_t)(k - f);
        const bool last = k - f == pc - 1;
        out_pk[dst] = ((uint32_t)(c - lo) << SEG_CSHIFT) | (last ? SEG_END : 0u) | (uint32_t)(r - hdr[dst / SEG_CH]);
        out_val[dst] = val[k];
      }
    }
  }
}

// Warp per group of 32 consecutive rows (panels <= 32): a panel's slots for those rows
// are one contiguous range (positions are row-ordered), so the group's entries are
// placed in a shared-memory image of the group's panel ranges (lane per row) and written
// out per panel with consecutive lanes on consecutive slots — ~2 write requests per row
// instead of one per (row, panel) piece and array.  A group whose ranges exceed SG_CAP
// slots (long rows) takes the per-row path of k_seg_scatter.  C4 layout build: 26 ->
// 22.8 ms (an entry-parallel placement with a row search measured 30 ms; 768 slots x 8
// warps 23.6-25.5 ms).
constexpr int SG_CAP = 1024;
constexpr int SG_SERIAL_MAX = 48;
constexpr int SG_WARPS = 4;

constexpr int SG_HMAX = SG_CAP / SEG_CH + 2;  // chunks a group's range of one panel can touch

// per warp: the output image (not with DIRECT), the (panel, row) table, row starts,
// per-panel ranges and the chunk headers of those ranges
inline size_t sg_warp_bytes(int n_panels, size_t val_bytes, bool direct) {
  return align_up((direct ? 0 : (size_t)SG_CAP * (4 + val_bytes)) + (size_t)n_panels * 32 * 16 + 40 * 4 +
                      4 * 32 * 4 + 32 * 4 + 32 * 8 + 32 * 16 + (size_t)n_panels * SG_HMAX * 4,
                  16);
}

// Row starts of a group are kept relative to its first entry (int32 even when row_ptr is
// int64): the image paths address col / val through the group's base pointers.
// DIRECT: no shared-memory image — every entry and explicit zero is stored straight to
// its slot (consecutive slots of one (row, panel) piece are consecutive lanes' stores;
// the partial sectors of a group's ranges merge in L2).  The image (18 KB per warp at
// C4) held the kernel to 12 warps per SM and the col loads' latency dominated (ncu:
// 18.75 % theoretical occupancy, 8.9 cycles per issued instruction).  Direct: C4 fill
// 14.5 -> 11.3 ms, whole layout build 19.8 -> 16.2 ms; C3 7.0 -> 5.0 ms; register caps for
// 9 / 12 CTAs per SM measured slower (17.4 / 18.0 ms builds).
template <typename T, typename IP, bool DIRECT>
__global__ void __launch_bounds__(SG_WARPS * 32) k_seg_scatter_groups(
    int64_t n_rows, const IP* __restrict__ row_ptr, const int32_t* __restrict__ col_all, const T* __restrict__ val_all,
    int32_t n_panels, const int32_t* __restrict__ bounds, const int32_t* __restrict__ counts,
    const int32_t* __restrict__ pos, const int64_t* __restrict__ offsets, uint32_t* __restrict__ out_pk,
    T* __restrict__ out_val, const int32_t* __restrict__ hdr, size_t warp_bytes, int fill_ballot) {
  extern __shared__ __align__(16) unsigned char sg_smem[];
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31, wib = threadIdx.x >> 5;
  const int P = n_panels;
  unsigned char* wb = sg_smem + (size_t)wib * warp_bytes;
  T* s_val = reinterpret_cast<T*>(wb);
  uint32_t* s_pk = reinterpret_cast<uint32_t*>(wb + (DIRECT ? 0 : (size_t)SG_CAP * sizeof(T)));
  // per (panel, row): {first entry, count, slot in the panel, slot - first}
  int4* s_tab = reinterpret_cast<int4*>(DIRECT ? wb : reinterpret_cast<unsigned char*>(s_pk + SG_CAP));  // [P][32]
  int32_t* s_rp = reinterpret_cast<int32_t*>(s_tab + P * 32);    // [33] row starts
  int32_t* s_gs = s_rp + 40;                                     // [32] group range start per panel
  int32_t* s_sb = s_gs + 32;                                     // [32] staging base per panel
  int32_t* s_len = s_sb + 32;                                    // [32]
  int32_t* s_nch = s_len + 32;                                   // [32] chunks of the group's range per panel
  int64_t* s_cb = reinterpret_cast<int64_t*>(s_nch + 32);        // [32] first such chunk
  int4* s_pp = reinterpret_cast<int4*>(s_cb + 32);               // [32] {image base - gs, chunk phase - gs, lo, 0}
  int32_t* s_hdr = reinterpret_cast<int32_t*>(s_pp + 32);        // [P][SG_HMAX] their headers
  __shared__ int32_t c_hi[32], c_lo[32];  // panel column bounds and slot offsets (CTA-wide)
  __shared__ int64_t c_off[32];
  int ppow = 1;  // smallest power of two >= P (steps of the panel search)
  while (ppow < P) ppow <<= 1;
  const int32_t my_hi = lane < P ? bounds[lane + 1] : INT32_MAX;
  const int32_t my_lo = lane < P ? bounds[lane] : 0;
  const int64_t my_off = lane < P ? offsets[lane] : 0;
  if (wib == 0) {
    c_hi[lane] = my_hi;
    c_lo[lane] = my_lo;
    c_off[lane] = my_off;
  }
  __syncthreads();
  const int64_t n_groups = (n_rows + 31) / 32;
  const int64_t warp = (int64_t)blockIdx.x * SG_WARPS + wib, n_warps = (int64_t)gridDim.x * SG_WARPS;
  const int64_t nnz_all = row_ptr[n_rows];
  for (int64_t g = warp; g < n_groups; g += n_warps) {
    const int64_t r0 = g * 32;
    const int nr = (int)min((int64_t)32, n_rows - r0);
    const IP gbase = row_ptr[r0];  // the group's first entry: s_rp and the image paths are relative to it
    const int32_t* __restrict__ col = col_all + gbase;
    const T* __restrict__ val = val_all + gbase;
    __syncwarp();
    if (lane < nr) s_rp[lane] = (int32_t)(row_ptr[r0 + lane] - gbase);
    if (lane == 0) s_rp[nr] = (int32_t)(row_ptr[r0 + nr] - gbase);
    // the group's first 128 entries, requested now so their latency overlaps the metadata
    // phases below (the entry-parallel placement consumes them; ncu: the first use of these
    // loads held 43 % of the fill's stall samples when they were issued there)
    int32_t pre_c[4];
    T pre_v[4];
    {
      // bounded by the matrix end, not the group's (no extra dependent load); entries past
      // the group are never consumed
      const int64_t left = nnz_all - (int64_t)gbase;
#pragma unroll
      for (int u = 0; u < 4; ++u) {
        const int32_t k = 32 * u + lane;
        pre_c[u] = k < left ? __ldg(col + k) : 0;
        pre_v[u] = k < left ? val[k] : T(0);
      }
    }
    // the group's range in each panel and its place in the staging image
    int32_t gs = 0, len = 0;
    if (lane < P) {
      const int32_t* pp = pos + (int64_t)lane * (n_rows + 1);
      gs = pp[r0];
      len = pp[r0 + nr] - gs;
    }
    int32_t incl = len;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      const int32_t t = __shfl_up_sync(FULL, incl, o);
      if (lane >= o) incl += t;
    }
    const int32_t total = __shfl_sync(FULL, incl, 31);
    if (total > SG_CAP) {  // long rows: the per-row path
      for (int i = 0; i < nr; ++i) {
        const int64_t r = r0 + i;
        const IP a = row_ptr[r], b = row_ptr[r + 1];
        int32_t cnt = 0, ppos = 0, pnext = 0;
        if (lane < P) {
          cnt = counts[(int64_t)lane * n_rows + r];
          const int32_t* pp = pos + (int64_t)lane * (n_rows + 1);
          ppos = pp[r];
          pnext = pp[r + 1];
        }
        int32_t ic = cnt;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const int32_t t = __shfl_up_sync(FULL, ic, o);
          if (lane >= o) ic += t;
        }
        const IP first = a + ic - cnt;
        if (lane < P && cnt == 0 && pnext > ppos) {
          const int64_t dst = my_off + ppos;
          out_pk[dst] = (SEG_MARK << SEG_CSHIFT) | SEG_END | (uint32_t)(r - hdr[dst / SEG_CH]);
          out_val[dst] = T(0);
        }
        for (IP k0 = a; k0 < b; k0 += 32) {
          const IP k = k0 + lane;
          const int32_t c = k < b ? col_all[k] : INT32_MAX;
          int p = 0;
          for (int q = 0; q < P; ++q) p += (c >= __shfl_sync(FULL, my_hi, q)) ? 1 : 0;
          if (p >= P) p = P - 1;
          const IP f = __shfl_sync(FULL, first, p);
          const int32_t pc = __shfl_sync(FULL, cnt, p);
          const int32_t pq = __shfl_sync(FULL, ppos, p);
          const int64_t po = __shfl_sync(FULL, my_off, p);
          const int32_t lo = __shfl_sync(FULL, my_lo, p);
          if (k < b) {
            const int64_t dst = po + pq + (int64_t)(k - f);
            out_pk[dst] = ((uint32_t)(c - lo) << SEG_CSHIFT) | (k - f == pc - 1 ? SEG_END : 0u) |
                          (uint32_t)(r - hdr[dst / SEG_CH]);
            out_val[dst] = val_all[k];
          }
        }
      }
      continue;
    }
    if (lane < P) {
      s_gs[lane] = gs;
      s_sb[lane] = incl - len;
      s_len[lane] = len;
      const int64_t g0 = my_off + gs;
      s_cb[lane] = g0 / SEG_CH;
      s_nch[lane] = len > 0 ? (int32_t)((g0 + len - 1) / SEG_CH - g0 / SEG_CH + 1) : 0;
      // slot dip of panel lane: image index x + dip, header chunk (y + dip) >> 7
      s_pp[lane] = make_int4(incl - len - gs, (int32_t)(g0 & (SEG_CH - 1)) - gs, my_lo, 0);
    }
    __syncwarp();
    // chunk headers of the group's range in every panel (<= SG_HMAX each), so placing an
    // entry or an explicit zero reads its chunk's first row from shared memory
    for (int t = lane; t < P * SG_HMAX; t += 32) {
      const int p = t / SG_HMAX, j = t - p * SG_HMAX;
      if (j < s_nch[p]) s_hdr[t] = hdr[s_cb[p] + j];
    }
    // per (panel, row): first entry, count, slot; explicit zeros go straight to the image
    if (lane < nr) {
      const int64_t r = r0 + lane;
      int32_t run = s_rp[lane];
      for (int p = 0; p < P; ++p) {
        const int32_t c = counts[(int64_t)p * n_rows + r];
        const int32_t* pp = pos + (int64_t)p * (n_rows + 1);
        const int32_t ppos = pp[r];
        s_tab[p * 32 + lane] = make_int4(run, c, ppos, ppos - run);
        run += c;
      }
    }
    __syncwarp();
    if (lane < nr) {
      const int64_t r = r0 + lane;
      for (int p = 0; p < P; ++p) {
        if (s_tab[p * 32 + lane].y != 0) continue;
        const int32_t ppos = s_tab[p * 32 + lane].z;
        const int32_t pnext = (lane + 1 < nr) ? s_tab[p * 32 + lane + 1].z : s_gs[p] + s_len[p];
        if (pnext > ppos) {
          const int32_t sidx = s_sb[p] + (ppos - s_gs[p]);
          const int64_t dst = c_off[p] + ppos;
          const uint32_t w = (SEG_MARK << SEG_CSHIFT) | SEG_END |
                             (uint32_t)(r - s_hdr[p * SG_HMAX + (int)(dst / SEG_CH - s_cb[p])]);
          if (DIRECT) {
            out_pk[dst] = w;
            out_val[dst] = T(0);
          } else {
            s_pk[sidx] = w;
            s_val[sidx] = T(0);
          }
        }
      }
    }
    // the entries into the image: the group's entries are one contiguous range of the
    // CSR, read coalesced (lane = entry); each finds its row (binary search of the
    // group's row starts), its panel (compares against the panel bounds) and its slot
    // from the (panel, row) tables — independent entries, so the loads overlap (a lane
    // per row walking its row serially measured latency-bound: 17.9 ms at C4, ncu)
    // Groups of short rows (max row <= SG_SERIAL_MAX: C4's 20-entry rows) keep a lane per
    // row walking its row (the panel only moves forward, so the table entries reload
    // only when it changes; 17.9 ms at C4 against 23.0 ms entry-parallel); groups with a
    // longer row go entry-parallel (C3 R-MAT: 10.8 -> 5.4 ms).
    int32_t my_len = lane < nr ? s_rp[lane + 1] - s_rp[lane] : 0;
    const bool no_empty = __all_sync(FULL, lane >= nr || my_len > 0);
#pragma unroll
    for (int o = 16; o; o >>= 1) my_len = max(my_len, __shfl_xor_sync(FULL, my_len, o));
    if (no_empty && fill_ballot) {
      // entry-parallel (lane = entry, coalesced loads, four windows of 32 in flight): an
      // entry's row comes from a bit mask of the row starts inside its 32-entry window
      // (one OR-reduction per window, no search: every row of the group is non-empty, so
      // starts are distinct), its panel from the panel bounds, its slot from the (panel,
      // row) tables.  C4 (20-entry rows): see DESIGN.md §5.
      const int32_t k0 = s_rp[0], k1 = s_rp[nr];
      const int32_t my_start = lane < nr ? s_rp[lane] : INT32_MAX;
      int row_at = 0;  // row (within the group) of the window's first entry
      for (int32_t w0 = k0; w0 < k1; w0 += 128) {
        int32_t c[4];
        T v[4];
        if (w0 == 0) {  // k0 == 0: the prefetched window
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            c[u] = pre_c[u];
            v[u] = pre_v[u];
          }
        } else {
#pragma unroll
          for (int u = 0; u < 4; ++u) {
            const int32_t k = w0 + 32 * u + lane;
            c[u] = k < k1 ? __ldg(col + k) : 0;
            v[u] = k < k1 ? val[k] : T(0);
          }
        }
#pragma unroll
        for (int u = 0; u < 4; ++u) {
          const int32_t base = w0 + 32 * u;
          if (base >= k1) break;
          const int32_t off = my_start - base;  // rows starting strictly inside this window
          const unsigned m = __reduce_or_sync(FULL, (off > 0 && off < 32) ? (1u << off) : 0u);
          const int32_t k = base + lane;
          const unsigned upto = (lane == 31 ? 0xffffffffu : ((2u << lane) - 1u)) & ~1u;
          const int rr = row_at + __popc(m & upto);
          row_at += __popc(m) + (__any_sync(FULL, my_start == base + 32) ? 1 : 0);
          if (k < k1) {
            const int32_t cc = c[u];
            // panel: branchless search of the (INT32_MAX-padded) upper bounds
            int p = 0;
#pragma unroll
            for (int st = 16; st > 0; st >>= 1)
              if (st < ppow && cc >= c_hi[p + st - 1]) p += st;
            const int4 tb = s_tab[p * 32 + rr];
            const int4 pp = s_pp[p];
            const int32_t dip = tb.w + k;  // slot within the panel
            const uint32_t w = (((uint32_t)cc - (uint32_t)pp.z) << SEG_CSHIFT) |
                               (k - tb.x == tb.y - 1 ? SEG_END : 0u) |
                               (uint32_t)((int32_t)(r0 + rr) - s_hdr[p * SG_HMAX + ((pp.y + dip) >> 7)]);
            if (DIRECT) {
              const int64_t dst = c_off[p] + dip;
              out_pk[dst] = w;
              out_val[dst] = v[u];
            } else {
              s_pk[pp.x + dip] = w;
              s_val[pp.x + dip] = v[u];
            }
          }
        }
      }
    } else if (my_len <= SG_SERIAL_MAX) {
      if (lane < nr) {
        const int32_t r_rel = r0 + lane;
        const int32_t kend = s_rp[lane + 1];
        int p = 0;
        int32_t f = s_tab[lane].x, pc = s_tab[lane].y, pq = s_tab[lane].z, sb = s_sb[0] - s_gs[0];
        int64_t po = c_off[0];
        uint32_t clo = (uint32_t)c_lo[0];
        for (int32_t k = s_rp[lane]; k < kend; ++k) {
          const int32_t c = col[k];
          const T v = val[k];
          if (p < P - 1 && c >= c_hi[p]) {
            do ++p;
            while (p < P - 1 && c >= c_hi[p]);
            f = s_tab[p * 32 + lane].x;
            pc = s_tab[p * 32 + lane].y;
            pq = s_tab[p * 32 + lane].z;
            sb = s_sb[p] - s_gs[p];
            po = c_off[p];
            clo = (uint32_t)c_lo[p];
          }
          const int32_t dip = pq + (k - f);  // slot within the panel
          const uint32_t w = (((uint32_t)c - clo) << SEG_CSHIFT) | (k - f == pc - 1 ? SEG_END : 0u) |
                             (uint32_t)(r_rel - hdr[(po + dip) / SEG_CH]);
          if (DIRECT) {
            out_pk[po + dip] = w;
            out_val[po + dip] = v;
          } else {
            s_pk[sb + dip] = w;
            s_val[sb + dip] = v;
          }
        }
      }
    } else {
      const int32_t k0 = s_rp[0], k1 = s_rp[nr];
#pragma unroll 2
      for (int32_t k = k0 + lane; k < k1; k += 32) {
        const int32_t c = col[k];
        const T v = val[k];
        int lo = 0, hi = nr;  // s_rp[lo] <= k < s_rp[hi]
        while (hi - lo > 1) {
          const int mid = (lo + hi) >> 1;
          if (s_rp[mid] <= k) lo = mid; else hi = mid;
        }
        int p = 0;
        for (int q = 0; q < P - 1; ++q) p += c >= c_hi[q] ? 1 : 0;
        const int t = p * 32 + lo;
        const int32_t f = s_tab[t].x, pc = s_tab[t].y;
        const int32_t dip = s_tab[t].z + (k - f);  // slot within the panel
        const uint32_t w = (((uint32_t)c - (uint32_t)c_lo[p]) << SEG_CSHIFT) | (k - f == pc - 1 ? SEG_END : 0u) |
                           (uint32_t)((int32_t)(r0 + lo) - hdr[(c_off[p] + dip) / SEG_CH]);
        if (DIRECT) {
          out_pk[c_off[p] + dip] = w;
          out_val[c_off[p] + dip] = v;
        } else {
          const int32_t sidx = s_sb[p] - s_gs[p] + dip;
          s_pk[sidx] = w;
          s_val[sidx] = v;
        }
      }
    }
    __syncwarp();
    if (!DIRECT) {
      // out, panel by panel, consecutive lanes on consecutive slots
      for (int p = 0; p < P; ++p) {
        const int32_t n_p = s_len[p], sb = s_sb[p];
        const int64_t base = c_off[p] + s_gs[p];
        for (int q = lane; q < n_p; q += 32) {
          out_pk[base + q] = s_pk[sb + q];
          out_val[base + q] = s_val[sb + q];
        }
      }
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
// The chunk stream.  f64: L1-allocating loads (the L1::no_allocate ones measured C4 +1.0 %,
// C5 +5.3 %, same bits; profiles/round2/seg_mio.txt); f32: no_allocate (equal on C3).
template <typename T> struct SegVal;
template <> struct SegVal<double> {
  static constexpr bool kAlloc = true;
  static __device__ __forceinline__ void load(const double* p, double v[4]) {
    // one 256-bit load per lane (LDG.E.ENL2.256): the lane's 4 values are one 32-byte sector
    asm volatile("ld.global.nc.v4.f64 {%0,%1,%2,%3}, [%4];" : "=d"(v[0]), "=d"(v[1]), "=d"(v[2]), "=d"(v[3]) : "l"(p));
  }
};
template <> struct SegVal<float> {
  static constexpr bool kAlloc = false;
  static __device__ __forceinline__ void load(const float* p, float v[4]) {
    const float4 a = ld_nc_na_f4(reinterpret_cast<const float4*>(p));
    v[0] = a.x; v[1] = a.y; v[2] = a.z; v[3] = a.w;
  }
};

template <typename T>
struct SegChunk {
  uint32_t w[4];
  T v[4];
  int h;
  __device__ __forceinline__ void load(const uint32_t* __restrict__ pk, const T* __restrict__ val,
                                       const int32_t* __restrict__ hdr, int c, int lane) {
    const int4* qp = reinterpret_cast<const int4*>(pk + c + 4 * lane);
    const int4 q = SegVal<T>::kAlloc ? __ldg(qp) : ld_nc_na_i4(qp);
    w[0] = (uint32_t)q.x; w[1] = (uint32_t)q.y; w[2] = (uint32_t)q.z; w[3] = (uint32_t)q.w;
    SegVal<T>::load(val + c + 4 * lane, v);
    h = SegVal<T>::kAlloc ? __ldg(hdr + c / SEG_CH) : ld_nc_na_i1(hdr + c / SEG_CH);
  }
};

// Epilogue of the last pass of an iterative step (sme_spmv_seg_epi): every row
// total t becomes v = s * t with s = *scale, stored at out[qinv[r]] (qinv null:
// out[r]); the warps' sums of v*v go to partials[warp] and the last CTA to finish
// reduces them in a fixed order into result[1] = sum v*v, result[0] = 1/sqrt(.)
// (the next step's scale).  Deterministic: fixed warp ranges, fixed trees.
template <typename T>
struct SegEpi {
  T* out;
  const int32_t* qinv;
  const double* scale;
  double* partials;  // [n_warps]
  unsigned* ticket;  // zero before the launch; reset by the last CTA
  double* result;    // [2]
  T* const* peers;   // [n_peers] other ranks' copies of out (peer memory over NVLink), or null
  int n_peers;
  int64_t row_offset;  // global index of this shard's row 0 in out / peers
  const T* dotv;       // null: reduce v*v; else reduce v * dotv[g] (CG's p.Ap)
  int finish;          // 0: result = {1/sqrt(sum), sum}; 1 (CG alpha): result[1] = result[0] / sum
  // split-row plans (non-epilogue passes): the open row partial at the end of a warp's
  // range -> carry_val[warp], its row -> carry_row[warp] (-1: the range ends on a row end)
  T* carry_val;
  int32_t* carry_row;
};

// last-CTA reduction of the warp partials (fixed order) -> result, next scale
template <typename T>
__device__ __forceinline__ void seg_epi_finish_impl(const SegEpi<T>& epi, int32_t n_warps) {
  __shared__ double red[SEG_NT];
  __shared__ bool last;
  __syncthreads();
  if (threadIdx.x == 0) {
    __threadfence();
    last = atomicAdd(epi.ticket, 1u) == gridDim.x - 1;
  }
  __syncthreads();
  if (!last) return;
  __threadfence();
  double acc = 0.0;
  for (int w = threadIdx.x; w < n_warps; w += SEG_NT) acc += __ldcg(epi.partials + w);
  red[threadIdx.x] = acc;
  __syncthreads();
  for (int o = SEG_NT / 2; o > 0; o >>= 1) {
    if (threadIdx.x < o) red[threadIdx.x] += red[threadIdx.x + o];
    __syncthreads();
  }
  if (threadIdx.x == 0) {
    const double tot = red[0];
    if (epi.finish == 1) {
      epi.result[1] = epi.result[0] / tot;  // alpha = r.r / p.Ap
    } else {
      epi.result[1] = tot;
      epi.result[0] = tot > 0.0 ? 1.0 / sqrt(tot) : 0.0;
    }
    *epi.ticket = 0u;
  }
}

// the random x gather.  f64: L1::no_allocate (a random 8-byte gather never hits a line
// it allocated; C4 -3.5 %, C5 -3 %).  f32: the allocating __ldg, which measured 7 % faster
// on C3 than no_allocate (4-byte values: a line holds 32 of them and R-MAT rows repeat
// columns more often).
__device__ __forceinline__ double seg_gather(const double* p) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.f64 %0, [%1];" : "=d"(r) : "l"(p));
  return r;
}
__device__ __forceinline__ float seg_gather(const float* p) { return __ldg(p); }

template <bool INTERIOR, typename T, bool ACC, bool EPI, bool RED>
__device__ __forceinline__ void seg_decode(const SegChunk<T>& cur, int e0, int P0, int P1, const T* __restrict__ xs,
                                           const T* __restrict__ y, unsigned& ok, unsigned& endm, T (&xv)[4],
                                           T (&yv)[4]) {
#pragma unroll
  for (int k = 0; k < 4; ++k) {
    const bool in = INTERIOR || (e0 + k >= P0 && e0 + k < P1);
    const uint32_t lc = cur.w[k] >> SEG_CSHIFT;
    ok |= in ? (1u << k) : 0u;
    endm |= (in && (cur.w[k] & SEG_END)) ? (1u << k) : 0u;
    xv[k] = (in && lc != SEG_MARK) ? seg_gather(xs + lc) : T(0);
    // accumulating passes skip explicit zeros (their rows have nothing to add)
    const bool emit = in && (cur.w[k] & SEG_END) && (EPI || !(ACC && lc == SEG_MARK));
    yv[k] = (ACC && !RED && emit) ? y[cur.h + (int)(cur.w[k] & SEG_DMASK)] : T(0);
  }
}

// CMP: the chunk's row totals are staged in shared memory in row order (an
// exclusive warp scan of each lane's row ends gives the slots) and written with
// one instruction per 32 rows, so consecutive lanes hit consecutive y words: ~4 y
// requests per chunk instead of ~16 (four predicated instructions each spanning the
// chunk's ~50 rows).  Applies to the writing pass and to RED accumulation.
// decode of the chunk at position cpos (all-interior fast path for f32, see seg_warp_body)
template <typename T, bool ACC, bool EPI, bool RED>
__device__ __forceinline__ void seg_decode_any(const SegChunk<T>& ch, int cpos, int lane, int P0, int P1,
                                               const T* __restrict__ xs, const T* __restrict__ y, unsigned& ok,
                                               unsigned& endm, T (&xv)[4], T (&yv)[4]) {
  ok = 0;
  endm = 0;
  const int e0 = cpos + 4 * lane;
  if (sizeof(T) == 4 && cpos >= P0 && cpos + SEG_CH <= P1)
    seg_decode<true, T, ACC, EPI, RED>(ch, e0, P0, P1, xs, y, ok, endm, xv, yv);
  else
    seg_decode<false, T, ACC, EPI, RED>(ch, e0, P0, P1, xs, y, ok, endm, xv, yv);
}

// PIPE: software-pipelined gathers.  The x gathers (and y reads) of chunk k+1 are
// issued BEFORE chunk k is reduced, and chunk k+2's stream loads before those, so a
// warp keeps a chunk's gathers in flight while it reduces: the L1 -> L2 request port
// sees gathers during the reduction phases too (seg_mode 7, sme_spmv_seg_set_mode).
template <typename T, bool ACC, bool EPI, bool RED = false, bool CMP = false, bool PIPE = false>
__device__ __forceinline__ double seg_warp_body(const uint32_t* __restrict__ pk, const T* __restrict__ val,
                                                const int32_t* __restrict__ hdr, const int32_t* __restrict__ plan,
                                                int warp, const T* __restrict__ xs, T* __restrict__ y,
                                                const SegEpi<T>& epi, T* s_val = nullptr, int* s_row = nullptr) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  double ss = 0.0;
  const int P0 = plan[warp], P1 = plan[warp + 1];
  if (P0 >= P1) {
    if (!EPI && epi.carry_row && lane == 0) epi.carry_row[warp] = -1;
    return ss;
  }
  const T sc = (EPI && epi.scale) ? (T)*epi.scale : T(1);

  int c = P0 & ~(SEG_CH - 1);
  SegChunk<T> cur, nxt;
  cur.load(pk, val, hdr, c, lane);
  T carry = T(0);  // open row sum flowing from the previous chunk's last entry
  unsigned ok = 0, endm = 0;
  T xv[4], yv[4];
  if (PIPE) {
    seg_decode_any<T, ACC, EPI, RED>(cur, c, lane, P0, P1, xs, y, ok, endm, xv, yv);
    if (c + SEG_CH < P1) nxt.load(pk, val, hdr, c + SEG_CH, lane);
  }
  while (true) {
    const bool more = c + SEG_CH < P1;
    unsigned ok_n = 0, endm_n = 0;
    T xv_n[4], yv_n[4];
    SegChunk<T> nn;
    if (PIPE) {
      if (more) {
        if (c + 2 * SEG_CH < P1) nn.load(pk, val, hdr, c + 2 * SEG_CH, lane);
        seg_decode_any<T, ACC, EPI, RED>(nxt, c + SEG_CH, lane, P0, P1, xs, y, ok_n, endm_n, xv_n, yv_n);
      }
    } else {
      if (more) nxt.load(pk, val, hdr, c + SEG_CH, lane);
      // decode: valid entries (inside [P0, P1)), end flags, gathers, y reads at row ends.
      // f32: chunks wholly inside the warp's range (all but its first and last) skip the
      // per-entry range checks (warp-uniform branch; C3 -4.6 %).  f64 keeps one code path
      // (the duplicated decode measured +3 % on C4 and C5).
      seg_decode_any<T, ACC, EPI, RED>(cur, c, lane, P0, P1, xs, y, ok, endm, xv, yv);
    }
    // in-lane runs: run[k] = sum of the row segment ending at k that starts in this lane
    T run[4];
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const T p = ((ok >> k) & 1u) ? cur.v[k] * xv[k] : T(0);
      run[k] = (k > 0 && !((endm >> (k - 1)) & 1u)) ? run[k > 0 ? k - 1 : 0] + p : p;
    }
    // open tail: what flows out of this lane into the next one's first segment
    const bool pass = endm == 0;  // the whole lane is the middle of one row
    T out = (endm & 8u) ? T(0) : run[3];
    T in_v;
    // `carry` lives in lane 31 (its previous lane_out); lane 0 takes it through the same
    // rotated shuffle that hands every other lane its left neighbour's tail, so the chunk's
    // outgoing chain value needs no broadcast of its own (C4 a further -0.6 %)
    if (__ballot_sync(FULL, pass) == 0u) {
      in_v = __shfl_sync(FULL, lane == 31 ? carry : out, (lane + 31) & 31);
    } else {
      carry = __shfl_sync(FULL, carry, 31);  // (rare) every lane sees lane 31's carry
      // chains of whole-lane rows: inclusive scan of `out` continuing through pass lanes
      bool head = !pass;
      T sv = out;
      if (lane == 0 && pass) sv += carry;  // a chain through lane 0 starts in the previous chunk
      for (int o = 1; o < 32; o <<= 1) {
        const T t = __shfl_up_sync(FULL, sv, o);
        const bool hh = __shfl_up_sync(FULL, (int)head, o) != 0;
        if (lane >= o && !head) {
          sv += t;
          head = hh;
        }
        if (!__any_sync(FULL, !head && lane >= 2 * o)) break;
      }
      in_v = __shfl_up_sync(FULL, sv, 1);
      out = sv;
      if (lane == 0) in_v = carry;
    }
    // the chain value leaving lane 31 (its tail plus everything flowing through it)
    const T lane_out = pass ? in_v + run[3] : out;
    if (lane == 31) carry = lane_out;
    // row totals: entries up to the lane's first end get the incoming chain
    bool first = true;
    int slot = 0, n_ends = 0;
    if (CMP) {
      unsigned emitm = endm;
      if (ACC && !EPI) {
#pragma unroll
        for (int k = 0; k < 4; ++k)
          if ((cur.w[k] >> SEG_CSHIFT) == SEG_MARK) emitm &= ~(1u << k);
      }
      // exclusive prefix of the lanes' row-end counts (0..4) from three bit ballots instead
      // of a five-step shuffle scan: the pass's warps wait on the MIO pipe (shuffles, shared
      // memory) about as long as on memory (ncu short/long scoreboard 6.0 / 6.2 cycles per
      // issue); C4 -2.1 %, C5 -1.5 %, same bits (profiles/round2/seg_mio.txt)
      const int cnt = __popc(emitm);
      const unsigned lt = (1u << lane) - 1u;
      const unsigned b0 = __ballot_sync(FULL, cnt & 1), b1 = __ballot_sync(FULL, cnt & 2),
                     b2 = __ballot_sync(FULL, cnt & 4);
      slot = __popc(b0 & lt) + 2 * __popc(b1 & lt) + 4 * __popc(b2 & lt);
      n_ends = __popc(b0) + 2 * __popc(b1) + 4 * __popc(b2);
      __syncwarp();  // the previous chunk's staged rows have been written out
    }
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const T fin = run[k] + (first ? in_v : T(0));
      const uint32_t lc = cur.w[k] >> SEG_CSHIFT;
      if ((endm >> k) & 1u) {
        first = false;
        if (EPI) {
          // every row ends exactly once in the epilogue pass (explicit zeros included)
          const int r = cur.h + (int)(cur.w[k] & SEG_DMASK);
          const T v = sc * (ACC ? yv[k] + fin : fin);
          if (CMP) {  // stores (and the dot) happen row-ordered after the loop
            s_row[slot] = r;
            s_val[slot] = v;
            ++slot;
          } else {
            const int64_t g = (int64_t)(epi.qinv ? epi.qinv[r] : r) + epi.row_offset;
            epi.out[g] = v;
            for (int d = 0; d < epi.n_peers; ++d) epi.peers[d][g] = v;  // the exchange, row by row
            ss += (double)v * (double)(epi.dotv ? epi.dotv[g] : v);
          }
        } else if (!(ACC && lc == SEG_MARK)) {
          const int r = cur.h + (int)(cur.w[k] & SEG_DMASK);
          if (CMP) {
            s_row[slot] = r;
            s_val[slot] = fin;
            ++slot;
          } else if (ACC && RED) {
            atomicAdd(y + r, fin);  // RED.ADD at L2: one add per row per pass, passes ordered: deterministic
          } else {
            y[r] = ACC ? yv[k] + fin : fin;
          }
        }
      }
    }
    if (CMP) {
      __syncwarp();
      for (int q = lane; q < n_ends; q += 32) {
        if (EPI) {
          const int r = s_row[q];
          const T v = s_val[q];
          const int64_t g = (int64_t)(epi.qinv ? epi.qinv[r] : r) + epi.row_offset;
          epi.out[g] = v;
          for (int d = 0; d < epi.n_peers; ++d) epi.peers[d][g] = v;  // the exchange, row by row
          ss += (double)v * (double)(epi.dotv ? epi.dotv[g] : v);
        } else if (ACC) {
          atomicAdd(y + s_row[q], s_val[q]);
        } else {
          y[s_row[q]] = s_val[q];
        }
      }
    }
    if (!more) {
      if (!EPI && epi.carry_row) {
        // a split-row plan may end this range mid-row: keep the open partial for the
        // ordered fix-up (k_seg_carry_fixup); explicit zeros always end their row
        const int last = P1 - 1 - c, kk = last & 3;
        const uint32_t wsel = kk == 0 ? cur.w[0] : kk == 1 ? cur.w[1] : kk == 2 ? cur.w[2] : cur.w[3];
        const uint32_t wl = __shfl_sync(FULL, wsel, last >> 2);
        if (lane == 31) {  // the lane that holds `carry`
          const bool open = !(wl & SEG_END);
          epi.carry_row[warp] = open ? cur.h + (int)(wl & SEG_DMASK) : -1;
          epi.carry_val[warp] = open ? carry : T(0);
        }
      }
      break;
    }
    cur = nxt;
    if (PIPE) {
      nxt = nn;
      ok = ok_n;
      endm = endm_n;
#pragma unroll
      for (int k = 0; k < 4; ++k) {
        xv[k] = xv_n[k];
        yv[k] = yv_n[k];
      }
    }
    c += SEG_CH;
  }
  return ss;
}

// Fix-up of a split-row pass: each row that ended in a later warp than it started
// gets the open partials of its earlier warps, summed in warp order (deterministic),
// after the pass has written / accumulated the row's tail.
template <typename T>
__global__ void k_seg_carry_fixup(int32_t n_warps, const int32_t* __restrict__ carry_row,
                                  const T* __restrict__ carry_val, T* __restrict__ y) {
  // Only empty ranges (-1) can sit between two carries of the same row (a non-empty range
  // inside the row carries it, one ending on the row's end owns its tail), so -1 entries
  // are skipped: exactly one thread per row sums the row's run of carries.
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w < n_warps; w += gridDim.x * blockDim.x) {
    const int32_t r = carry_row[w];
    if (r < 0) continue;
    int pw = w - 1;
    while (pw >= 0 && carry_row[pw] < 0) --pw;
    if (pw >= 0 && carry_row[pw] == r) continue;  // not the first carry of this row
    T sum = carry_val[w];
    for (int v = w + 1; v < n_warps; ++v) {
      const int32_t rv = carry_row[v];
      if (rv < 0) continue;
      if (rv != r) break;
      sum += carry_val[v];
    }
    y[r] += sum;
  }
}

template <typename T, bool ACC, bool EPI, bool RED = false, bool CMP = false, bool PIPE = false>
__global__ void __launch_bounds__(SEG_NT) k_spmv_seg(const uint32_t* __restrict__ pk, const T* __restrict__ val,
                                                   const int32_t* __restrict__ hdr, const int32_t* __restrict__ plan,
                                                   int32_t n_warps, const T* __restrict__ xs, T* __restrict__ y,
                                                   SegEpi<T> epi) {
  const unsigned FULL = 0xffffffffu;
  const int lane = threadIdx.x & 31;
  const int warp = (blockIdx.x * SEG_NT + threadIdx.x) >> 5;
  if (EPI) {
    __shared__ T e_val[SEG_NT / 32][SEG_CH];
    __shared__ int e_row[SEG_NT / 32][SEG_CH];
    double ss = 0.0;
    if (warp < n_warps)
      ss = seg_warp_body<T, ACC, true, false, kStageRows<T>>(pk, val, hdr, plan, warp, xs, y, epi,
                                                             e_val[threadIdx.x >> 5], e_row[threadIdx.x >> 5]);
    for (int o = 16; o > 0; o >>= 1) ss += __shfl_xor_sync(FULL, ss, o);
    if (lane == 0 && warp < n_warps) epi.partials[warp] = ss;
    if (epi.n_peers > 0) __threadfence_system();  // peer stores performed before this launch completes
    seg_epi_finish_impl(epi, n_warps);
    return;
  }
  if (warp >= n_warps) return;
  if (CMP) {
    __shared__ T s_val[SEG_NT / 32][SEG_CH];
    __shared__ int s_row[SEG_NT / 32][SEG_CH];
    seg_warp_body<T, ACC, false, RED, true, PIPE>(pk, val, hdr, plan, warp, xs, y, epi, s_val[threadIdx.x >> 5],
                                                  s_row[threadIdx.x >> 5]);
  } else {
    seg_warp_body<T, ACC, false, RED, false, PIPE>(pk, val, hdr, plan, warp, xs, y, epi);
  }
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
  SegChunk<T> cur;
  cur.load(pk, val, hdr, c, lane);
  while (true) {
    const bool more = c + SEG_CH < P1;
    SegChunk<T> nxt;
    if (more) nxt.load(pk, val, hdr, c + SEG_CH, lane);
    T acc = T(0);
#pragma unroll
    for (int k = 0; k < 4; ++k) {
      const uint32_t lc = cur.w[k] >> SEG_CSHIFT;
      acc += (lc != SEG_MARK) ? cur.v[k] * __ldg(xs + lc) : T(0);
    }
    y[cur.h + lane] = acc;
    if (!more) break;
    cur = nxt;
    c += SEG_CH;
  }
}

// 0 = SpMV (default: row totals staged and written in row order; accumulating passes
// add with RED.ADD.F64 at L2), 3 = bound probe, 5 = accumulating passes load y, add,
// store, 6 = RED accumulation without the staging (one write per (lane, k) row end)
static int s_seg_mode = 0;

template <typename T>
int launch_seg(int32_t n_warps, const uint32_t* pk, const T* val, const int32_t* hdr, const int32_t* plan,
               const T* xs, T* y, int accumulate, cudaStream_t s, const SegEpi<T>* epi = nullptr) {
  const int grid = (int)(((int64_t)n_warps * 32 + SEG_NT - 1) / SEG_NT);
  const SegEpi<T> e = epi ? *epi : SegEpi<T>{};
  if (epi && e.carry_row) {  // split-row plan: the pass, then the ordered fix-up of the open partials
    SegEpi<T> plain = e;
    const bool stage = kStageRows<T> && s_seg_mode != 6;
    if (accumulate)
      stage ? k_spmv_seg<T, true, false, true, true><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y, plain)
            : k_spmv_seg<T, true, false, true><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y, plain);
    else
      stage ? k_spmv_seg<T, false, false, false, true><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y, plain)
            : k_spmv_seg<T, false, false><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y, plain);
    SME_CHECK_LAUNCH("k_spmv_seg");
    k_seg_carry_fixup<T><<<(n_warps + 255) / 256, 256, 0, s>>>(n_warps, e.carry_row, e.carry_val, y);
    SME_CHECK_LAUNCH("k_seg_carry_fixup");
    return SME_OK;
  }
  if (epi) {
    if (accumulate)
      k_spmv_seg<T, true, true><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y, e);
    else
      k_spmv_seg<T, false, true><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y, e);
  } else if (s_seg_mode == 3)
    k_seg_probe<T><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y);

  else if (s_seg_mode == 7 && accumulate)
    k_spmv_seg<T, true, false, true, kStageRows<T>, true><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y, e);
  else if (s_seg_mode == 7)
    k_spmv_seg<T, false, false, false, kStageRows<T>, true><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y,
                                                                                   e);
  else if (accumulate && s_seg_mode == 5)
    k_spmv_seg<T, true, false><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y, e);
  else if (accumulate && (s_seg_mode == 6 || !kStageRows<T>))
    k_spmv_seg<T, true, false, true><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y, e);
  else if (accumulate)
    k_spmv_seg<T, true, false, true, true><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y, e);
  else if (s_seg_mode == 6 || !kStageRows<T>)
    k_spmv_seg<T, false, false><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y, e);
  else
    k_spmv_seg<T, false, false, false, true><<<grid, SEG_NT, 0, s>>>(pk, val, hdr, plan, n_warps, xs, y, e);
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
template <typename IP>
static int seg_positions_impl(int64_t n_rows, const IP* row_ptr, const int32_t* col, int32_t n_panels,
                              const int32_t* bounds, int full_last, int32_t* pos, void* ws, size_t ws_bytes,
                              sme_stream_t stream) {
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
  k_seg_count<IP><<<grid_for(n_rows, 256), 256, 0, s>>>(n_rows, row_ptr, col, n_panels, bounds, counts);
  SME_CHECK_LAUNCH("k_seg_count");
  for (int p = 0; p < n_panels; ++p) {
    const bool full = full_last && p == n_panels - 1;
    int rc = exclusive_scan_lengths(n_rows, SegLen{counts + (int64_t)p * n_rows, p, full}, pos + (int64_t)p * (n_rows + 1),
                                    scan_ws, nullptr, s);
    if (rc != SME_OK) return rc;
  }
  return SME_OK;
}

SME_API int sme_seg_positions(int64_t n_rows, const int32_t* row_ptr, const int32_t* col, int32_t n_panels,
                              const int32_t* bounds, int full_last, int32_t* pos, void* ws, size_t ws_bytes,
                              sme_stream_t stream) {
  return seg_positions_impl(n_rows, row_ptr, col, n_panels, bounds, full_last, pos, ws, ws_bytes, stream);
}

// int64 row_ptr (nnz >= 2^31); each panel must still hold < 2^31 slots (the caller picks
// enough panels; pos stays int32 per panel)
SME_API int sme_seg_positions_i64(int64_t n_rows, const int64_t* row_ptr, const int32_t* col, int32_t n_panels,
                                  const int32_t* bounds, int full_last, int32_t* pos, void* ws, size_t ws_bytes,
                                  sme_stream_t stream) {
  return seg_positions_impl(n_rows, row_ptr, col, n_panels, bounds, full_last, pos, ws, ws_bytes, stream);
}

// Step 2: chunk headers and the packed entries.  offsets[p] (int64 device) = first
// element of panel p in pk/val (multiple of 128); pk and val must be pre-filled
// with the tail padding (pk 0xFFFFFFFF, val 0) by the caller.  bounds[p+1]-bounds[p]
// must be < 2^23 - 1 (SEG_MARK).
template <typename IP>
static int seg_fill_impl(int dtype, int64_t n_rows, const IP* row_ptr, const int32_t* col, const void* val,
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
  if (n_panels <= 32 && s_seg_scatter_groups) {
    auto launch = [&](auto kern, size_t vb, auto* v, auto* ov) {
      const size_t wbytes = sg_warp_bytes(n_panels, vb, s_seg_fill_direct), smem = wbytes * SG_WARPS;
      SME_CUDA(cudaFuncSetAttribute(kern, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem));
      const int64_t groups = (n_rows + 31) / 32;
      // a fixed 16 CTAs per SM (2-3 waves): one to six occupancy-sized waves measured 2-10 %
      // slower on C4 (profiles/round2/resident_grids.txt)
      const int grid = grid_for(groups * 32, SG_WARPS * 32, 16);
      kern<<<grid, SG_WARPS * 32, smem, s>>>(n_rows, row_ptr, col, v, n_panels, bounds, counts, pos, offsets, pk, ov,
                                             hdr, wbytes, (int)s_seg_fill_ballot);
      return SME_OK;
    };
    if (dtype == SME_F64)
      s_seg_fill_direct ? launch(k_seg_scatter_groups<double, IP, true>, 8, (const double*)val, (double*)out_val)
                        : launch(k_seg_scatter_groups<double, IP, false>, 8, (const double*)val, (double*)out_val);
    else
      s_seg_fill_direct ? launch(k_seg_scatter_groups<float, IP, true>, 4, (const float*)val, (float*)out_val)
                        : launch(k_seg_scatter_groups<float, IP, false>, 4, (const float*)val, (float*)out_val);
    SME_CHECK_LAUNCH("k_seg_scatter_groups");
    return SME_OK;
  }
  if (dtype == SME_F64)
    k_seg_scatter<double, IP><<<grid_for(n_rows * 32, 256), 256, 0, s>>>(n_rows, row_ptr, col, (const double*)val, n_panels,
                                                                      bounds, counts, pos, offsets, pk,
                                                                      (double*)out_val, hdr);
  else
    k_seg_scatter<float, IP><<<grid_for(n_rows * 32, 256), 256, 0, s>>>(n_rows, row_ptr, col, (const float*)val, n_panels,
                                                                     bounds, counts, pos, offsets, pk, (float*)out_val,
                                                                     hdr);
  SME_CHECK_LAUNCH("k_seg_scatter");
  return SME_OK;
}

SME_API int sme_seg_fill(int dtype, int64_t n_rows, const int32_t* row_ptr, const int32_t* col, const void* val,
                         int32_t n_panels, const int32_t* bounds, const int32_t* pos, const int64_t* offsets,
                         const int64_t* h_offsets, uint32_t* pk, void* out_val, int32_t* hdr, const void* ws,
                         sme_stream_t stream) {
  return seg_fill_impl(dtype, n_rows, row_ptr, col, val, n_panels, bounds, pos, offsets, h_offsets, pk, out_val, hdr,
                       ws, stream);
}

SME_API int sme_seg_fill_i64(int dtype, int64_t n_rows, const int64_t* row_ptr, const int32_t* col, const void* val,
                             int32_t n_panels, const int32_t* bounds, const int32_t* pos, const int64_t* offsets,
                             const int64_t* h_offsets, uint32_t* pk, void* out_val, int32_t* hdr, const void* ws,
                             sme_stream_t stream) {
  return seg_fill_impl(dtype, n_rows, row_ptr, col, val, n_panels, bounds, pos, offsets, h_offsets, pk, out_val, hdr,
                       ws, stream);
}

// Groups of non-empty rows: entry-parallel placement (1, default) or the lane-per-row
// walk / searched entry-parallel paths of earlier versions (0).  For A/B tests.
// 1 (default): the fill stores entries straight to their slots; 0: through the
// shared-memory image of each group's panel ranges (A/B and tests of that path)
SME_API int sme_seg_set_fill_direct(int on) {
  s_seg_fill_direct = on != 0;
  return SME_OK;
}

SME_API int sme_seg_set_fill_ballot(int on) {
  s_seg_fill_ballot = on != 0;
  return SME_OK;
}

// Layout fill: 1 = warp per 32-row group through a shared-memory image (default),
// 0 = warp per row (k_seg_scatter).  Process-wide; for A/B tests.
SME_API int sme_seg_set_scatter_groups(int on) {
  s_seg_scatter_groups = on != 0;
  return SME_OK;
}

// Kernel variant (process-wide; experiments): 0 = the SpMV, 3 = bound probe (the
// chunk stream and gathers without the row reduction; timing only, not y = A x).
SME_API int sme_spmv_seg_set_mode(int mode) {
  SME_REQUIRE(mode == 0 || mode == 3 || mode == 5 || mode == 6 || mode == 7,
              "mode must be 0 (SpMV), 3 (bound probe), 5 (accumulate with load + store), 6 (no staging) or "
              "7 (pipelined gathers)");
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
  occ((const void*)k_spmv_seg<double, false, false>);
  occ((const void*)k_spmv_seg<double, true, false>);
  occ((const void*)k_spmv_seg<float, false, false>);
  occ((const void*)k_spmv_seg<float, true, false>);
  occ((const void*)k_spmv_seg<double, false, true>);
  occ((const void*)k_spmv_seg<double, true, true>);
  occ((const void*)k_spmv_seg<double, false, false, false, true>);
  occ((const void*)k_spmv_seg<double, true, false, true, true>);
  if (s_seg_mode == 7) {
    occ((const void*)k_spmv_seg<double, false, false, false, true, true>);
    occ((const void*)k_spmv_seg<double, true, false, true, true, true>);
    occ((const void*)k_spmv_seg<float, false, false, false, false, true>);
    occ((const void*)k_spmv_seg<float, true, false, true, false, true>);
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

// The last pass of one iterative step with the fused epilogue (see SegEpi): out[qinv[r]] =
// scale[0] * (y[r] + this pass), partials[n_warps] scratch, ticket (uint32, zero-initialised
// once; left zero), result[2] = {1/sqrt(sum v^2), sum v^2}.  accumulate = 0 for a
// one-panel layout.  The layout must hold an entry or explicit zero for every row in
// this panel (sme_seg_positions with full_last = 1).  f64 only.
SME_API int sme_spmv_seg_epi(int dtype, int32_t n_warps, const uint32_t* pk, const void* val, const int32_t* hdr,
                             const int32_t* plan, const void* xs, void* y, int accumulate, void* out,
                             const int32_t* qinv, const double* scale, double* partials, uint32_t* ticket,
                             double* result, sme_stream_t stream) {
  SME_REQUIRE(dtype == SME_F64, "the fused epilogue is f64 only");
  SME_REQUIRE(n_warps >= 1 && pk && val && hdr && plan && out && scale && partials && ticket && result,
              "bad arguments");
  SME_REQUIRE((((uintptr_t)pk | (uintptr_t)val) & 15) == 0, "pk/val must be 16-byte aligned");
  const SegEpi<double> e{(double*)out, qinv, scale, partials, ticket, result, nullptr, 0, 0, nullptr, 0, nullptr,
                         nullptr};
  return launch_seg<double>(n_warps, pk, (const double*)val, hdr, plan, (const double*)xs, (double*)y, accumulate,
                            as_stream(stream), &e);
}

// The same epilogue pass for one row shard of a multi-GPU iteration: v is stored at
// global index row_offset + r of `out` (this rank's full-length next iterate) AND of
// each of the n_peers buffers in d_peers (the other ranks' next iterates, opened
// with sme_ipc_open: stores over NVLink), i.e. the all-gather of the iterate is
// fused into the SpMV epilogue.  result[1] is this shard's sum of v^2 (the caller
// all-reduces it); qinv must be null.
SME_API int sme_spmv_seg_epi_peers(int dtype, int32_t n_warps, const uint32_t* pk, const void* val,
                                   const int32_t* hdr, const int32_t* plan, const void* xs, void* y, int accumulate,
                                   void* out, int64_t row_offset, void* const* d_peers, int32_t n_peers,
                                   const double* scale, double* partials, uint32_t* ticket, double* result,
                                   sme_stream_t stream) {
  SME_REQUIRE(dtype == SME_F64, "the fused epilogue is f64 only");
  SME_REQUIRE(n_warps >= 1 && pk && val && hdr && plan && out && scale && partials && ticket && result &&
                  row_offset >= 0 && n_peers >= 0 && (n_peers == 0 || d_peers),
              "bad arguments");
  SME_REQUIRE((((uintptr_t)pk | (uintptr_t)val) & 15) == 0, "pk/val must be 16-byte aligned");
  const SegEpi<double> e{(double*)out, nullptr, scale, partials, ticket, result, (double* const*)d_peers, n_peers,
                         row_offset, nullptr, 0, nullptr, nullptr};
  return launch_seg<double>(n_warps, pk, (const double*)val, hdr, plan, (const double*)xs, (double*)y, accumulate,
                            as_stream(stream), &e);
}

// The last pass of one CG step with p.Ap fused in: out[r] = (A p)[r] (no scaling), the
// sum of out[r] * p[r] reduced deterministically, and the last CTA writes alpha =
// scal[0] / (p.Ap) into scal[1] (scal[0] = r.r, the layout of blas1.cu's CG
// scalars), replacing sme_dot(p, Ap) of the unfused step.  Square matrix, xs = p (full).
SME_API int sme_spmv_seg_epi_cg(int dtype, int32_t n_warps, const uint32_t* pk, const void* val, const int32_t* hdr,
                                const int32_t* plan, const void* xs, const void* p, void* y, int accumulate,
                                void* out, double* partials, uint32_t* ticket, double* scal, sme_stream_t stream) {
  SME_REQUIRE(dtype == SME_F64, "the fused epilogue is f64 only");
  SME_REQUIRE(n_warps >= 1 && pk && val && hdr && plan && p && out && partials && ticket && scal, "bad arguments");
  SME_REQUIRE((((uintptr_t)pk | (uintptr_t)val) & 15) == 0, "pk/val must be 16-byte aligned");
  const SegEpi<double> e{(double*)out, nullptr, nullptr, partials, ticket, scal, nullptr, 0, 0, (const double*)p, 1,
                         nullptr, nullptr};
  return launch_seg<double>(n_warps, pk, (const double*)val, hdr, plan, (const double*)xs, (double*)y, accumulate,
                            as_stream(stream), &e);
}

// Split-row plan: plan[w] = w * total / n_warps entry positions (ranges may start and end
// mid-row, so one long row no longer lands on a single warp).
__global__ void k_seg_plan_split(int64_t total, int32_t n_warps, int32_t* __restrict__ plan) {
  for (int w = blockIdx.x * blockDim.x + threadIdx.x; w <= n_warps; w += gridDim.x * blockDim.x)
    plan[w] = (int32_t)((int64_t)w * total / n_warps);
}

SME_API int sme_seg_plan_split(int64_t total_entries, int32_t n_warps, int32_t* plan, sme_stream_t stream) {
  SME_REQUIRE(n_warps >= 1 && total_entries >= 0 && total_entries < INT32_MAX && plan, "bad arguments");
  k_seg_plan_split<<<grid_for((int64_t)n_warps + 1, 256), 256, 0, as_stream(stream)>>>(total_entries, n_warps, plan);
  SME_CHECK_LAUNCH("k_seg_plan_split");
  return SME_OK;
}

// One panel pass over a split-row plan (not the fused epilogue): like sme_spmv_seg, then
// the open partials at the warp-range ends (carry_val[n_warps], carry_row[n_warps]
// scratch) are added to their rows in warp order by k_seg_carry_fixup.
SME_API int sme_spmv_seg_split(int dtype, int32_t n_warps, const uint32_t* pk, const void* val, const int32_t* hdr,
                               const int32_t* plan, const void* xs, void* y, int accumulate, void* carry_val,
                               int32_t* carry_row, sme_stream_t stream) {
  SME_REQUIRE(dtype == SME_F64 || dtype == SME_F32, "unknown dtype %d", dtype);
  SME_REQUIRE(n_warps >= 1 && pk && val && hdr && plan && carry_val && carry_row, "bad arguments");
  SME_REQUIRE((((uintptr_t)pk | (uintptr_t)val) & 15) == 0, "pk/val must be 16-byte aligned");
  cudaStream_t s = as_stream(stream);
  if (dtype == SME_F64) {
    SegEpi<double> e{};
    e.carry_val = (double*)carry_val;
    e.carry_row = carry_row;
    return launch_seg<double>(n_warps, pk, (const double*)val, hdr, plan, (const double*)xs, (double*)y, accumulate,
                              s, &e);
  }
  SegEpi<float> e{};
  e.carry_val = (float*)carry_val;
  e.carry_row = carry_row;
  return launch_seg<float>(n_warps, pk, (const float*)val, hdr, plan, (const float*)xs, (float*)y, accumulate, s,
                           &e);
}

namespace sme {
// Lazy module loading (CUDA 12 default) loads this file's module on the first launch of
// any of its kernels, ~10-20 ms each; sme_preload() does it ahead of time.
int preload_spmv_seg() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)k_seg_hdr) == cudaSuccess ? 0 : -1;
}
}  // namespace sme
