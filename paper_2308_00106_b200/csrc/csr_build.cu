// csr_build.cu — COO->CSR and the fused permuted-CSR build (K4 in SURVEY.md §2.2).
//
// Reference: coo_to_csr (matio.py:281-294) = lexsort((col,row)) + duplicate
// check + cumsum(bincount(row)); permute_matrix (permute.py:98-102) = index
// remap in entry order, after which the reference runs coo_to_csr again.
//
// GPU algorithm (same output bits):
//   1. row lengths of the result (COO: atomic count per row; CSR: gather of
//      the old row length through inv_r) -> exclusive scan -> row_ptr;
//   2. COO only: stable-free scatter of (mapped col, value) into the row's
//      slots (order inside a row is arbitrary here);
//   3. segmented sort inside every row by (mapped) column, values following
//      bit-exactly, adjacent-equal columns flagged as duplicates.  Rows are
//      dispatched by length: <= 32 -> a warp per 32 rows, transposed through shared
//      memory so one thread sorts one row with a register bitonic network
//      (G = next_pow2(max len in the warp's 32 rows) lanes per row);
//      <= SME_SORT_SMEM_MAX -> one CTA, bitonic in shared memory;
//      longer -> one CTA, shared-memory chunk sort + global merge passes.
// Because (row, col) pairs are unique the sorted CSR is unique, so the result
// is independent of the scatter order and bit-identical to the reference.
#include "common.cuh"
#include "scan.cuh"

namespace sme {

constexpr int LONG_CHUNK = SME_SORT_SMEM_MAX;  // keys per shared-memory chunk
constexpr int SORT_NT = 256;
constexpr int LONG_NT = 512;

struct SortLists {
  int32_t* med;       // [n_rows] row ids with 32 < len <= big_min (warp-wide register sort)
  int32_t* big;       // [n_rows] row ids with big_min < len <= SMEM_MAX (one CTA per row)
  int32_t* lng;       // [n_rows] row ids with len > SMEM_MAX
  int64_t* lng_off;   // [n_rows] offset of each long row in the long scratch
  int32_t* counters;  // [0] = #med, [1] = #long, [2] = #big
  int big_min;        // the warp sort's largest row (rows above go to `big`)
  unsigned long long* lng_cursor;  // running long scratch offset
  uint64_t* scratch_a;             // long_nnz keys
  uint64_t* scratch_b;             // long_nnz keys
  int mark_dups;                   // 1: duplicates become col = -1 (dedupe) instead of an error
};

inline size_t lists_bytes(int64_t n_rows, int64_t long_nnz) {
  return align_up(n_rows * 4) * 3 + align_up(n_rows * 8) + align_up(64) + align_up(long_nnz * 8) * 2;
}

inline SortLists carve_lists(char* p, int64_t n_rows, int64_t long_nnz) {
  SortLists L;
  L.med = (int32_t*)p;           p += align_up(n_rows * 4);
  L.big = (int32_t*)p;           p += align_up(n_rows * 4);
  L.lng = (int32_t*)p;           p += align_up(n_rows * 4);
  L.lng_off = (int64_t*)p;       p += align_up(n_rows * 8);
  L.counters = (int32_t*)p;
  L.lng_cursor = (unsigned long long*)(p + 16);
  p += align_up(64);
  L.scratch_a = (uint64_t*)p;    p += align_up(long_nnz * 8);
  L.scratch_b = (uint64_t*)p;
  L.mark_dups = 0;
  L.big_min = 32;
  return L;
}

// Where the entries of output row r are read from.
// start(r, dst) = where(r); split into the old row id (key, a coalesced load) and the
// dependent old_ptr gather (start_of) so the warp sort can issue them a phase apart.
// IP: the row_ptr element type (int32_t, or int64_t for nnz >= 2^31; entry offsets are
// carried as int64_t either way).
template <typename IP>
struct SrcGather {  // permuted CSR: old row inv[r] of the source CSR
  const IP* old_ptr;
  const int32_t* inv;
  __device__ __forceinline__ int32_t key(int32_t r) const { return inv ? inv[r] : r; }
  __device__ __forceinline__ int64_t start_of(int32_t k, int64_t /*dst*/) const { return (int64_t)old_ptr[k]; }
  __device__ __forceinline__ int64_t start(int32_t r, int64_t dst) const { return start_of(key(r), dst); }
};
struct SrcStaged {  // COO path: the row's slots in the staging arrays
  __device__ __forceinline__ int32_t key(int32_t /*r*/) const { return 0; }
  __device__ __forceinline__ int64_t start_of(int32_t /*k*/, int64_t dst) const { return dst; }
  __device__ __forceinline__ int64_t start(int32_t /*r*/, int64_t dst) const { return dst; }
};

__device__ __forceinline__ void report_dup(int32_t row, uint32_t col, int32_t* flag,
                                           unsigned long long* dup_key) {
  atomicOr(flag, SME_FLAG_DUPLICATE);
  atomicMin(dup_key, ((unsigned long long)(uint32_t)row << 32) | col);
}

// New column id of a source entry: cmap[c], or, for an entry the sliced pre-map
// (sme_map_cols_sliced_partial) already relabelled, its id with the bit-31 flag cleared.
__device__ __forceinline__ uint32_t map_col(const int32_t* __restrict__ cmap, int32_t c) {
  return (uint32_t)(cmap ? (c < 0 ? (c & 0x7fffffff) : __ldg(cmap + c)) : c);
}

// ---------------------------------------------------------------------------
// rows with len <= 32: thread-per-row register networks on a transposed tile
// ---------------------------------------------------------------------------
// 1: 32-bit keys whenever n_cols <= 2^27 (default); 0: always 64-bit keys (tests of that path)
static int g_sort_key32 = 1;
// 1: rows with 32 < len <= WMED_MAX are sorted warp-wide in registers (default); 0: by the
// CTA-wide shared-memory kernel (A/B and tests of that path)
static int g_sort_wmed = 3;  // rows 33..256 (C3 K4: 26.2 -> 20.0 ms; 512 spills: 27.8)
// 1: rows of 257..SME_SORT_SMEM_MAX entries sorted by the register/shuffle/smem hybrid
// network (default); 0: the all-shared-memory bitonic (A/B and tests of that path)
static int g_sort_cta = 1;

// Keys: 64-bit (mapped col << 32 | slot) in general; 32-bit (mapped col << 5 |
// slot) when every mapped column is < 2^27 (KEY32: one shuffle per exchange
// instead of two).  The column map (p_c, a random gather from an n_cols table) is
// read with an L2 evict-last hint and the streams (old rows in, new rows out)
// with evict-first, so the table keeps as much of L2 as it can.
template <bool KEY32>
struct SortKey {
  using K = uint64_t;
  static constexpr K NONE = ~0ull;
  __device__ static K make(uint32_t col, int slot) { return ((uint64_t)col << 32) | (uint32_t)slot; }
  __device__ static uint32_t col(K k) { return (uint32_t)(k >> 32); }
  __device__ static int slot(K k) { return (int)(uint32_t)k; }
};
template <>
struct SortKey<true> {
  using K = uint32_t;
  static constexpr K NONE = ~0u;
  __device__ static K make(uint32_t col, int slot) { return (col << 5) | (uint32_t)slot; }
  __device__ static uint32_t col(K k) { return k >> 5; }
  __device__ static int slot(K k) { return (int)(k & 31u); }
};

// Ascending bitonic network over N keys held in registers (all indices static: every
// compare-exchange is a min and a max, no shuffles).
template <int N, typename K>
__device__ __forceinline__ void bitonic_regs(K (&a)[N]) {
#pragma unroll
  for (int k = 2; k <= N; k <<= 1)
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1)
#pragma unroll
      for (int i = 0; i < N; ++i) {
        const int l = i ^ j;
        if (l > i) {
          const K x = a[i], y = a[l];
          const K lo = x < y ? x : y, hi = x < y ? y : x;
          const bool up = (i & k) == 0;
          a[i] = up ? lo : hi;
          a[l] = up ? hi : lo;
        }
      }
}

constexpr int SORT_STRIDE = 33;  // row pitch of the per-warp key tile (conflict-free rows and columns)
constexpr int SORT_UNROLL = 8;   // rows per unrolled load / store step (loads in flight per lane)
constexpr int TILE_NT = 128;     // k_sort_rows_warp block: 4 warps, 17 KB (32-bit keys) / 34 KB of tiles

// Rows of up to 32 entries, a warp per group of 32 rows, in three phases per group:
//   A. coalesced loads: the warp walks the group's rows, lane l reading entry l of each
//      (column id, relabelled through p_c), and writes the key (new column, entry slot)
//      into row r of a 32 x 33 shared-memory tile;
//   B. thread per row: lane t reads row t of the tile into registers, sorts it with an
//      N-key bitonic network (N = 8/16/32 by the group's longest row; keys past a row's
//      length are NONE) and writes it back;
//   C. coalesced stores: the warp walks the rows again, lane l writing entry l of the
//      sorted row (column, and the value its slot names, read from the source row),
//      flagging a key equal in column to its predecessor as a duplicate.
// About 40 warp instructions per row of 20, against ~160 for a shuffle network with a
// lane per entry, which left the kernel issue-bound (ncu, C4: 11 ms at 64 % issue).
template <typename T, class Src, bool KEY32, int N>
__device__ __forceinline__ void sort_group_tile(typename SortKey<KEY32>::K* tile, int lane, int64_t g,
                                                int32_t len, int64_t dst, int64_t from,
                                                const int32_t* __restrict__ src_col, const T* __restrict__ src_val,
                                                const int32_t* __restrict__ cmap, int32_t* __restrict__ out_col,
                                                T* __restrict__ out_val, const SortLists& L, int32_t* flag,
                                                unsigned long long* dup_key, uint64_t keep, uint64_t once) {
  using SK = SortKey<KEY32>;
  using K = typename SK::K;
  // A: keys into the tile, SORT_UNROLL rows per step (their loads in flight together)
#pragma unroll 1
  for (int r0 = 0; r0 < 32; r0 += SORT_UNROLL) {
    int32_t c[SORT_UNROLL];
    bool in[SORT_UNROLL];
#pragma unroll
    for (int u = 0; u < SORT_UNROLL; ++u) {
      const int32_t ml = __shfl_sync(0xffffffffu, len, r0 + u);
      const int64_t mf = __shfl_sync(0xffffffffu, from, r0 + u);
      in[u] = lane < ml;
      c[u] = in[u] ? ld_stream_i1(src_col + mf + lane, once) : 0;
    }
#pragma unroll
    for (int u = 0; u < SORT_UNROLL; ++u) {
      uint32_t mc = (uint32_t)c[u];
      if (cmap && in[u]) mc = c[u] < 0 ? (uint32_t)(c[u] & 0x7fffffff) : (uint32_t)ld_l1(cmap + c[u], keep);
      tile[(r0 + u) * SORT_STRIDE + lane] = in[u] ? SK::make(mc, lane) : SK::NONE;
    }
  }
  __syncwarp();
  // B: lane t sorts row t
  {
    K k[N];
#pragma unroll
    for (int i = 0; i < N; ++i) k[i] = tile[lane * SORT_STRIDE + i];
    bitonic_regs<N>(k);
#pragma unroll
    for (int i = 0; i < N; ++i) tile[lane * SORT_STRIDE + i] = k[i];
  }
  __syncwarp();
  // C: sorted rows out, values gathered by slot from the source row
#pragma unroll 1
  for (int r0 = 0; r0 < 32; r0 += SORT_UNROLL) {
    K key[SORT_UNROLL];
    T w[SORT_UNROLL];
    int64_t md[SORT_UNROLL];
    bool in[SORT_UNROLL];
#pragma unroll
    for (int u = 0; u < SORT_UNROLL; ++u) {
      const int32_t ml = __shfl_sync(0xffffffffu, len, r0 + u);
      const int64_t mf = __shfl_sync(0xffffffffu, from, r0 + u);
      md[u] = __shfl_sync(0xffffffffu, dst, r0 + u);
      in[u] = lane < ml;
      key[u] = tile[(r0 + u) * SORT_STRIDE + lane];
      w[u] = in[u] ? ld_stream(src_val + mf + SK::slot(key[u]), once) : T(0);
    }
#pragma unroll
    for (int u = 0; u < SORT_UNROLL; ++u) {
      if (in[u]) {
        const uint32_t col = SK::col(key[u]);
        const bool dup = lane > 0 && SK::col(tile[(r0 + u) * SORT_STRIDE + lane - 1]) == col;
        if (dup && !L.mark_dups) report_dup((int32_t)(g * 32 + r0 + u), col, flag, dup_key);
        // streaming stores: the outputs must not push the column map (cmap) out of L2
        st_stream(out_col + md[u] + lane, (dup && L.mark_dups) ? -1 : (int32_t)col);
        st_stream(out_val + md[u] + lane, w[u]);
      }
    }
  }
  __syncwarp();
}

template <typename T, class Src, bool KEY32, typename IP>
__global__ void __launch_bounds__(TILE_NT) k_sort_rows_warp(
    int32_t n_rows, const IP* __restrict__ new_ptr, Src src, const int32_t* __restrict__ src_col,
    const T* __restrict__ src_val, const int32_t* __restrict__ cmap, int32_t* __restrict__ out_col,
    T* __restrict__ out_val, SortLists L, int32_t* flag, unsigned long long* dup_key) {
  using SK = SortKey<KEY32>;
  using K = typename SK::K;
  __shared__ K s_tile[TILE_NT / 32][32 * SORT_STRIDE];
  K* tile = s_tile[threadIdx.x >> 5];
  const int lane = threadIdx.x & 31;
  const int64_t n_groups = ((int64_t)n_rows + 31) / 32;
  const int64_t warp_global = ((int64_t)blockIdx.x * TILE_NT + threadIdx.x) >> 5;
  const int64_t warps_total = ((int64_t)gridDim.x * TILE_NT) >> 5;
  const uint64_t keep = policy_evict_last(), once = policy_evict_first();
  // group metadata, one row per lane, fetched a group ahead: new_ptr and the old row id
  // (coalesced), then the old row's start (a gather) once the current group is running
  int64_t g = warp_global;
  IP n0 = 0, n1 = 0;
  int32_t k = 0;
  auto meta_raw = [&](int64_t gg) {
    const int32_t r = (int32_t)(gg * 32 + lane);
    n0 = n1 = k = 0;
    if (gg < n_groups && r < n_rows) {
      n0 = new_ptr[r];
      n1 = new_ptr[r + 1];
      k = src.key(r);
    }
  };
  meta_raw(g);
  int64_t from = n1 > n0 ? src.start_of(k, n0) : 0;
  for (; g < n_groups; g += warps_total) {
    const int32_t r = (int32_t)(g * 32 + lane);
    const int64_t dst = n0;
    int32_t len = (int32_t)(n1 - n0);
    const int64_t my_from = from;
    if (len > 32) {
      if (len <= L.big_min) {
        int slot = atomicAdd(&L.counters[0], 1);
        L.med[slot] = r;
      } else if (len <= SME_SORT_SMEM_MAX) {
        int slot = atomicAdd(&L.counters[2], 1);
        L.big[slot] = r;
      } else {
        int slot = atomicAdd(&L.counters[1], 1);
        L.lng[slot] = r;
        L.lng_off[slot] = (int64_t)atomicAdd(L.lng_cursor, (unsigned long long)len);
      }
      len = 0;
    }
    meta_raw(g + warps_total);
    int maxlen = len;
#pragma unroll
    for (int o = 16; o; o >>= 1) maxlen = max(maxlen, __shfl_xor_sync(0xffffffffu, maxlen, o));
    from = n1 > n0 ? src.start_of(k, n0) : 0;  // next group's starts: in flight during this one
    if (maxlen == 0) continue;
    if (maxlen <= 8)
      sort_group_tile<T, Src, KEY32, 8>(tile, lane, g, len, dst, my_from, src_col, src_val, cmap, out_col, out_val,
                                        L, flag, dup_key, keep, once);
    else if (maxlen <= 16)
      sort_group_tile<T, Src, KEY32, 16>(tile, lane, g, len, dst, my_from, src_col, src_val, cmap, out_col,
                                         out_val, L, flag, dup_key, keep, once);
    else
      sort_group_tile<T, Src, KEY32, 32>(tile, lane, g, len, dst, my_from, src_col, src_val, cmap, out_col,
                                         out_val, L, flag, dup_key, keep, once);
  }
}

// ---------------------------------------------------------------------------
// rows with 32 < len <= WMED_MAX: one warp per row, E = next_pow2(len) / 32 keys per
// lane in registers (blocked: lane l holds elements l*E .. l*E+E-1); bitonic steps
// with j < E are in-lane compare-exchanges, the others one shuffle per key.  Replaces
// a CTA-wide shared-memory bitonic (one __syncthreads per step) for these rows:
// R-MAT C3 (ragged rows up to the 1024 cap) K4 20.5 ms -> see DESIGN.md §5.
// ---------------------------------------------------------------------------
constexpr int WMED_MAX = 512;  // the largest row the warp sort handles (g_sort_wmed selects the cut)

template <int E>
__device__ __forceinline__ void warp_bitonic(uint64_t (&v)[E], int lane) {
  constexpr int N = 32 * E;
#pragma unroll
  for (int k = 2; k <= N; k <<= 1) {
#pragma unroll
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= E) {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = lane * E + e;
          const uint64_t o = __shfl_xor_sync(0xffffffffu, v[e], j / E);
          const bool asc = (i & k) == 0, lower = (i & j) == 0;
          const uint64_t mn = v[e] < o ? v[e] : o, mx = v[e] < o ? o : v[e];
          v[e] = (lower == asc) ? mn : mx;
        }
      } else {
#pragma unroll
        for (int e = 0; e < E; ++e) {
          if ((e & j) == 0) {
            const int i = lane * E + e;
            const bool asc = (i & k) == 0;
            const uint64_t a = v[e], b = v[e | j];
            if ((a > b) == asc) {
              v[e] = b;
              v[e | j] = a;
            }
          }
        }
      }
    }
  }
}

template <int E, typename T>
__device__ __forceinline__ void sort_row_warp(int32_t r, int64_t dst, int32_t len, int64_t from,
                                              const int32_t* __restrict__ src_col, const T* __restrict__ src_val,
                                              const int32_t* __restrict__ cmap, int32_t* __restrict__ out_col,
                                              T* __restrict__ out_val, const SortLists& L, int32_t* flag,
                                              unsigned long long* dup_key, int lane) {
  uint64_t v[E];
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = lane * E + e;
    v[e] = i < len ? (((uint64_t)map_col(cmap, src_col[from + i]) << 32) | (uint32_t)i) : ~0ull;
  }
  warp_bitonic<E>(v, lane);
  const uint64_t before = __shfl_up_sync(0xffffffffu, v[E - 1], 1);
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = lane * E + e;
    if (i < len) {
      const uint32_t key = (uint32_t)(v[e] >> 32);
      const uint64_t prev = e > 0 ? v[e > 0 ? e - 1 : 0] : before;
      const bool dup = i > 0 && (uint32_t)(prev >> 32) == key;
      if (dup && !L.mark_dups) report_dup(r, key, flag, dup_key);
      out_col[dst + i] = (dup && L.mark_dups) ? -1 : (int32_t)key;
      out_val[dst + i] = src_val[from + (uint32_t)v[e]];
    }
  }
}

template <typename T, class Src, typename IP>
__global__ void __launch_bounds__(SORT_NT) k_sort_rows_wmed(
    const IP* __restrict__ new_ptr, Src src, const int32_t* __restrict__ src_col,
    const T* __restrict__ src_val, const int32_t* __restrict__ cmap, int32_t* __restrict__ out_col,
    T* __restrict__ out_val, SortLists L, int32_t* flag, unsigned long long* dup_key, int wmed_max) {
  const int lane = threadIdx.x & 31;
  const int count = L.counters[0];
  const int64_t warp = ((int64_t)blockIdx.x * SORT_NT + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * SORT_NT) >> 5;
  for (int64_t it = warp; it < count; it += n_warps) {
    const int32_t r = L.med[it];
    const int64_t dst = new_ptr[r];
    const int32_t len = (int32_t)(new_ptr[r + 1] - dst);
    if (len > wmed_max) continue;  // k_sort_rows_block
    const int64_t from = src.start(r, dst);
    if (len <= 64)
      sort_row_warp<2, T>(r, dst, len, from, src_col, src_val, cmap, out_col, out_val, L, flag, dup_key, lane);
    else if (len <= 128)
      sort_row_warp<4, T>(r, dst, len, from, src_col, src_val, cmap, out_col, out_val, L, flag, dup_key, lane);
    else if (len <= 256)
      sort_row_warp<8, T>(r, dst, len, from, src_col, src_val, cmap, out_col, out_val, L, flag, dup_key, lane);
    else
      sort_row_warp<16, T>(r, dst, len, from, src_col, src_val, cmap, out_col, out_val, L, flag, dup_key, lane);
  }
}

// ---------------------------------------------------------------------------
// block-level bitonic sort of P (power of two) keys in shared memory
// ---------------------------------------------------------------------------
template <int NT>
__device__ void smem_bitonic(uint64_t* s, int P) {
  for (int k = 2; k <= P; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      for (int i = threadIdx.x; i < P; i += NT) {
        int p = i ^ j;
        if (p > i) {
          uint64_t a = s[i], b = s[p];
          bool asc = (i & k) == 0;
          if ((a > b) == asc) {
            s[i] = b;
            s[p] = a;
          }
        }
      }
      __syncthreads();
    }
  }
}

// CTA-wide bitonic sort of N = SORT_NT * E keys held E per thread in registers (blocked:
// thread t holds elements t*E .. t*E+E-1).  Steps with j < E are compare-exchanges inside a
// thread, j < 32*E one shuffle per key inside a warp, and only the j >= 32*E steps (6 of
// the 55 at N = 1024) go through shared memory with barriers — instead of a barrier after
// every one of the N log^2 N / 2 steps (smem_bitonic).
template <int E, int J>
__device__ __forceinline__ void cta_bitonic_local(uint64_t (&v)[E], int base, int k) {
#pragma unroll
  for (int e = 0; e < E; ++e) {
    if ((e & J) == 0) {
      const bool asc = ((base + e) & k) == 0;
      const uint64_t a = v[e], b = v[e | J];
      if ((a > b) == asc) {
        v[e] = b;
        v[e | J] = a;
      }
    }
  }
}

template <int E>
__device__ __forceinline__ void cta_bitonic(uint64_t (&v)[E], uint64_t* s) {
  constexpr int N = SORT_NT * E;
  const int tid = threadIdx.x, base = tid * E;
  for (int k = 2; k <= N; k <<= 1) {
    for (int j = k >> 1; j > 0; j >>= 1) {
      if (j >= 32 * E) {  // partner in another warp
#pragma unroll
        for (int e = 0; e < E; ++e) s[base + e] = v[e];
        __syncthreads();
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = base + e;
          const uint64_t o = s[i ^ j];
          const bool asc = (i & k) == 0, lower = (i & j) == 0;
          v[e] = (lower == asc) ? (v[e] < o ? v[e] : o) : (v[e] < o ? o : v[e]);
        }
        __syncthreads();
      } else if (j >= E) {  // partner in another lane of this warp
#pragma unroll
        for (int e = 0; e < E; ++e) {
          const int i = base + e;
          const uint64_t o = __shfl_xor_sync(0xffffffffu, v[e], j / E);
          const bool asc = (i & k) == 0, lower = (i & j) == 0;
          v[e] = (lower == asc) ? (v[e] < o ? v[e] : o) : (v[e] < o ? o : v[e]);
        }
      } else if (j == 1) {
        cta_bitonic_local<E, 1>(v, base, k);
      } else if (j == 2) {
        if constexpr (E > 2) cta_bitonic_local<E, 2>(v, base, k);
      } else if (j == 4) {
        if constexpr (E > 4) cta_bitonic_local<E, 4>(v, base, k);
      } else if (j == 8) {
        if constexpr (E > 8) cta_bitonic_local<E, 8>(v, base, k);
      }
    }
  }
}

template <int E, typename T>
__device__ __forceinline__ void sort_row_cta(int32_t len, int64_t from, const int32_t* __restrict__ src_col,
                                             const int32_t* __restrict__ cmap, uint64_t* s) {
  uint64_t v[E];
  const int base = threadIdx.x * E;
#pragma unroll
  for (int e = 0; e < E; ++e) {
    const int i = base + e;
    v[e] = i < len ? (((uint64_t)map_col(cmap, src_col[from + i]) << 32) | (uint32_t)i) : ~0ull;
  }
  cta_bitonic<E>(v, s);
#pragma unroll
  for (int e = 0; e < E; ++e) s[base + e] = v[e];
  __syncthreads();
}

// rows with 32 < len <= SME_SORT_SMEM_MAX: one CTA per row (rows of > 256 entries: the
// register / shuffle / shared-memory hybrid network; C3 R-MAT rows 257..1024)
template <typename T, class Src, typename IP>
__global__ void __launch_bounds__(SORT_NT) k_sort_rows_block(
    const IP* __restrict__ new_ptr, Src src, const int32_t* __restrict__ src_col,
    const T* __restrict__ src_val, const int32_t* __restrict__ cmap, int32_t* __restrict__ out_col,
    T* __restrict__ out_val, SortLists L, int32_t* flag, unsigned long long* dup_key, int wmed_max, int use_cta) {
  __shared__ uint64_t s[SME_SORT_SMEM_MAX];
  const int count = L.counters[2];
  for (int it = blockIdx.x; it < count; it += gridDim.x) {
    const int32_t r = L.big[it];
    const int64_t dst = new_ptr[r];
    const int32_t len = (int32_t)(new_ptr[r + 1] - dst);
    const int64_t from = src.start(r, dst);
    int P = 64;
    while (P < len) P <<= 1;
    if (P >= 2 * SORT_NT && use_cta) {
      if (P == 2 * SORT_NT) sort_row_cta<2, T>(len, from, src_col, cmap, s);
      else if (P == 4 * SORT_NT) sort_row_cta<4, T>(len, from, src_col, cmap, s);
      else if (P == 8 * SORT_NT) sort_row_cta<8, T>(len, from, src_col, cmap, s);
      else sort_row_cta<16, T>(len, from, src_col, cmap, s);
    } else {
      for (int i = threadIdx.x; i < P; i += SORT_NT)
        s[i] = i < len ? (((uint64_t)map_col(cmap, src_col[from + i]) << 32) | (uint32_t)i) : ~0ull;
      __syncthreads();
      smem_bitonic<SORT_NT>(s, P);
    }
    for (int i = threadIdx.x; i < len; i += SORT_NT) {
      uint64_t v = s[i];
      uint32_t key = (uint32_t)(v >> 32);
      const bool dup = i > 0 && (uint32_t)(s[i - 1] >> 32) == key;
      if (dup && !L.mark_dups) report_dup(r, key, flag, dup_key);
      out_col[dst + i] = (dup && L.mark_dups) ? -1 : (int32_t)key;
      out_val[dst + i] = src_val[from + (uint32_t)v];
    }
    __syncthreads();
  }
}

// rows with len > SME_SORT_SMEM_MAX: chunk sort in smem, then merge passes
// between two global scratch buffers; one CTA per row.
template <typename T, class Src, typename IP>
__global__ void __launch_bounds__(LONG_NT) k_sort_rows_long(
    const IP* __restrict__ new_ptr, Src src, const int32_t* __restrict__ src_col,
    const T* __restrict__ src_val, const int32_t* __restrict__ cmap, int32_t* __restrict__ out_col,
    T* __restrict__ out_val, SortLists L, int32_t* flag, unsigned long long* dup_key) {
  __shared__ uint64_t s[LONG_CHUNK];
  const int count = L.counters[1];
  for (int it = blockIdx.x; it < count; it += gridDim.x) {
    const int32_t r = L.lng[it];
    const int64_t dst = new_ptr[r];
    const int64_t len = new_ptr[r + 1] - dst;
    const int64_t from = src.start(r, dst);
    uint64_t* a = L.scratch_a + L.lng_off[it];
    uint64_t* b = L.scratch_b + L.lng_off[it];
    // 1. sorted chunks
    for (int64_t c0 = 0; c0 < len; c0 += LONG_CHUNK) {
      int n = (int)min((int64_t)LONG_CHUNK, len - c0);
      int P = 64;
      while (P < n) P <<= 1;
      for (int i = threadIdx.x; i < P; i += LONG_NT)
        s[i] = i < n ? (((uint64_t)map_col(cmap, src_col[from + c0 + i]) << 32) | (uint32_t)(c0 + i))
                     : ~0ull;
      __syncthreads();
      smem_bitonic<LONG_NT>(s, P);
      for (int i = threadIdx.x; i < n; i += LONG_NT) a[c0 + i] = s[i];
      __syncthreads();
    }
    // 2. merge passes a -> b, swap
    for (int64_t w = LONG_CHUNK; w < len; w <<= 1) {
      // thread t produces outputs [o0, o1) of the whole row
      int64_t o0 = len * threadIdx.x / LONG_NT, o1 = len * (threadIdx.x + 1) / LONG_NT;
      int64_t o = o0;
      while (o < o1) {
        int64_t ps = (o / (2 * w)) * (2 * w);  // pair start
        int64_t la = min(w, len - ps);
        int64_t lb = min(w, max((int64_t)0, len - ps - w));
        const uint64_t* A = a + ps;
        const uint64_t* B = a + ps + la;
        int64_t pend = min(o1, ps + la + lb);
        int64_t d = o - ps;
        int64_t lo = max((int64_t)0, d - lb), hi = min(d, la);
        while (lo < hi) {
          int64_t mid = (lo + hi) >> 1;
          if (A[mid] <= B[d - 1 - mid]) lo = mid + 1; else hi = mid;
        }
        int64_t ia = lo, ib = d - lo;
        for (; o < pend; ++o) {
          bool takeA = ib >= lb || (ia < la && A[ia] <= B[ib]);
          b[o] = takeA ? A[ia++] : B[ib++];
        }
      }
      __syncthreads();
      uint64_t* t = a; a = b; b = t;
      __syncthreads();
    }
    // 3. emit
    for (int64_t i = threadIdx.x; i < len; i += LONG_NT) {
      uint64_t v = a[i];
      uint32_t key = (uint32_t)(v >> 32);
      const bool dup = i > 0 && (uint32_t)(a[i - 1] >> 32) == key;
      if (dup && !L.mark_dups) report_dup(r, key, flag, dup_key);
      out_col[dst + i] = (dup && L.mark_dups) ? -1 : (int32_t)key;
      out_val[dst + i] = src_val[from + (uint32_t)v];
    }
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// COO phase kernels
// ---------------------------------------------------------------------------
__global__ void k_coo_count(int64_t nnz, int64_t n_rows, int64_t n_cols, const int32_t* __restrict__ row,
                            const int32_t* __restrict__ col, const int32_t* __restrict__ rmap,
                            int32_t* __restrict__ counts, int32_t* flag) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
    int32_t r = row[k], c = col[k];
    if (r < 0 || r >= n_rows || c < 0 || c >= n_cols) {
      atomicOr(flag, SME_FLAG_RANGE);
      continue;
    }
    if (rmap) r = rmap[r];
    atomicAdd(&counts[r], 1);
  }
}

__device__ __forceinline__ int32_t cursor_bump(int32_t* c) { return atomicAdd(c, 1); }
__device__ __forceinline__ int64_t cursor_bump(int64_t* c) {
  return (int64_t)atomicAdd(reinterpret_cast<unsigned long long*>(c), 1ull);
}

template <typename T, typename IP>
__global__ void k_coo_scatter(int64_t nnz, int64_t n_rows, int64_t n_cols, const int32_t* __restrict__ row,
                              const int32_t* __restrict__ col, const T* __restrict__ val,
                              const int32_t* __restrict__ rmap, IP* __restrict__ cursor,
                              int32_t* __restrict__ st_col, T* __restrict__ st_val) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
    int32_t r = row[k], c = col[k];
    if (r < 0 || r >= n_rows || c < 0 || c >= n_cols) continue;
    if (rmap) r = rmap[r];
    const IP pos = cursor_bump(&cursor[r]);
    st_col[pos] = c;  // column mapping is applied by the sort
    st_val[pos] = val[k];
  }
}

// The permuted row lengths, gathered once: stores the length and the source start of new
// row k (len_out[k], start_out[k]) while the scan's first pass sums them, so the second
// pass and the row sort read them sequentially instead of gathering old row_ptr again.
template <typename IP>
struct LenGatherStore {
  const IP* ptr;
  const int32_t* inv;
  int32_t* len_out;
  IP* start_out;
  __device__ __forceinline__ int64_t operator()(int64_t k) const {
    const int32_t o = inv ? inv[k] : (int32_t)k;
    const IP a = ptr[o], l = ptr[o + 1] - a;
    len_out[k] = (int32_t)l;
    start_out[k] = a;
    return (int64_t)l;
  }
};

struct LenFromCounts {
  const int32_t* counts;
  __device__ __forceinline__ int64_t operator()(int64_t k) const { return counts[k]; }
};
template <typename IP>
struct LenFromGather {
  const IP* ptr;
  const int32_t* inv;
  __device__ __forceinline__ int64_t operator()(int64_t k) const {
    int32_t o = inv ? inv[k] : (int32_t)k;
    return (int64_t)ptr[o + 1] - ptr[o];
  }
};

template <typename IP>
__global__ void k_long_row_nnz(int64_t n_rows, const IP* __restrict__ ptr, unsigned long long* out) {
  unsigned long long s = 0;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += stride) {
    const int64_t l = (int64_t)ptr[r + 1] - ptr[r];
    if (l > SME_SORT_SMEM_MAX) s += (unsigned long long)l;
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  if ((threadIdx.x & 31) == 0 && s) atomicAdd(out, s);
}

// out[0] = max row length, out[1] = number of empty rows (out zeroed by the caller)
template <typename IP>
__global__ void k_row_stats(int64_t n_rows, const IP* __restrict__ ptr, unsigned long long* out) {
  unsigned long long mx = 0, empty = 0;
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int64_t l = (int64_t)ptr[r + 1] - ptr[r];
    mx = max(mx, (unsigned long long)l);
    empty += l == 0;
  }
  for (int o = 16; o; o >>= 1) {
    mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    empty += __shfl_xor_sync(0xffffffffu, empty, o);
  }
  if ((threadIdx.x & 31) == 0) {
    atomicMax(out, mx);
    if (empty) atomicAdd(out + 1, empty);
  }
}

// Column span (last - first column) of n_samples evenly spaced rows (-1 for rows with < 2
// entries): the banded-structure probe of the kernel policy (kernels.banded).
template <typename IP>
__global__ void k_row_spans(int64_t n_rows, const IP* __restrict__ ptr, const int32_t* __restrict__ col,
                            int32_t n_samples, int32_t* __restrict__ out) {
  for (int32_t i = blockIdx.x * blockDim.x + threadIdx.x; i < n_samples; i += gridDim.x * blockDim.x) {
    const int64_t r = n_samples > 1 ? (int64_t)i * (n_rows - 1) / (n_samples - 1) : 0;
    const IP a = ptr[r], b = ptr[r + 1];
    out[i] = b - a >= 2 ? col[b - 1] - col[a] : -1;
  }
}

template <typename IP>
__global__ void k_csr_validate(int64_t n_rows, int64_t n_cols, int64_t nnz, const IP* __restrict__ ptr,
                               const int32_t* __restrict__ col, int32_t* flag) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int bits = 0;
  int64_t tid = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  if (tid == 0 && (ptr[0] != 0 || ptr[n_rows] != nnz)) bits |= SME_FLAG_ROWPTR;
  for (int64_t r = tid; r < n_rows; r += stride) {
    const IP a = ptr[r], b = ptr[r + 1];
    if (b < a) {
      bits |= SME_FLAG_ROWPTR;
      continue;
    }
    if (a < 0 || b > nnz) {
      bits |= SME_FLAG_ROWPTR;
      continue;
    }
    int32_t prev = -1;
    for (IP k = a; k < b; ++k) {
      int32_t c = col[k];
      if (c < 0 || c >= n_cols) bits |= SME_FLAG_RANGE;
      if (k > a && c <= prev) bits |= SME_FLAG_UNSORTED;
      prev = c;
    }
  }
  // also catch out-of-range columns outside any row span (corrupt row_ptr handled above)
  for (int o = 16; o; o >>= 1) bits |= __shfl_xor_sync(0xffffffffu, bits, o);
  if ((threadIdx.x & 31) == 0 && bits) atomicOr(flag, bits);
}

template <typename IP>
__global__ void k_csr_expand_rows(int64_t n_rows, const IP* __restrict__ ptr, int32_t* __restrict__ row_out) {
  // warp per row: rows are short on average, long rows are strided over lanes
  int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  int64_t nw = ((int64_t)gridDim.x * blockDim.x) >> 5;
  int lane = threadIdx.x & 31;
  for (int64_t r = warp; r < n_rows; r += nw) {
    const IP a = ptr[r], b = ptr[r + 1];
    for (IP k = a + lane; k < b; k += 32) row_out[k] = (int32_t)r;
  }
}

constexpr int SORT_WAVES = 16;

template <typename T, class Src, typename IP>
int launch_sorts(int64_t n_rows, const IP* new_ptr, Src src, const int32_t* src_col, const T* src_val,
                 const int32_t* cmap, int32_t* out_col, T* out_val, SortLists L, int32_t* flag,
                 uint64_t* dup_key, cudaStream_t s, int64_t n_cols = INT32_MAX) {
  int64_t groups = (n_rows + 31) / 32;
  // rows up to the warp sort's limit go to its list, longer ones (<= SMEM_MAX) to the CTA
  // sort's: each kernel walks only its own rows, in equal static shares over SORT_WAVES
  // occupancy-sized waves (grid_waves).
  L.big_min = g_sort_wmed > 0 ? 32 << g_sort_wmed : 32;
  if (n_cols <= ((int64_t)1 << 27) && g_sort_key32) {  // mapped columns < 2^27: 32-bit keys (col << 5 | slot)
    auto kern = k_sort_rows_warp<T, Src, true, IP>;
    kern<<<grid_waves(kern, groups * 32, TILE_NT, 0, SORT_WAVES, 16), TILE_NT, 0, s>>>(
        (int32_t)n_rows, new_ptr, src, src_col, src_val, cmap, out_col, out_val, L, flag, (unsigned long long*)dup_key);
  } else {
    auto kern = k_sort_rows_warp<T, Src, false, IP>;
    kern<<<grid_waves(kern, groups * 32, TILE_NT, 0, SORT_WAVES, 16), TILE_NT, 0, s>>>(
        (int32_t)n_rows, new_ptr, src, src_col, src_val, cmap, out_col, out_val, L, flag, (unsigned long long*)dup_key);
  }
  SME_CHECK_LAUNCH("k_sort_rows_warp");
  const int64_t any_work = (int64_t)1 << 40;  // the list lengths are on the device: grid = the resident cap
  const int wmed_max = g_sort_wmed > 0 ? 32 << g_sort_wmed : 0;  // 1: <= 64, 2: <= 128, 3: <= 256, 4: <= 512
  if (wmed_max) {
    auto kern = k_sort_rows_wmed<T, Src, IP>;
    kern<<<grid_waves(kern, any_work, SORT_NT, 0, SORT_WAVES, 8), SORT_NT, 0, s>>>(
        new_ptr, src, src_col, src_val, cmap, out_col, out_val, L, flag, (unsigned long long*)dup_key, wmed_max);
    SME_CHECK_LAUNCH("k_sort_rows_wmed");
  }
  {
    auto kern = k_sort_rows_block<T, Src, IP>;
    kern<<<grid_waves(kern, any_work, SORT_NT, 0, SORT_WAVES, 4), SORT_NT, 0, s>>>(
        new_ptr, src, src_col, src_val, cmap, out_col, out_val, L, flag, (unsigned long long*)dup_key, wmed_max,
        g_sort_cta);
  }
  SME_CHECK_LAUNCH("k_sort_rows_block");
  k_sort_rows_long<T, Src, IP><<<grid_waves(k_sort_rows_long<T, Src, IP>, any_work, LONG_NT, 0, SORT_WAVES, 1), LONG_NT, 0, s>>>(
      new_ptr, src, src_col, src_val, cmap, out_col, out_val, L, flag, (unsigned long long*)dup_key);
  SME_CHECK_LAUNCH("k_sort_rows_long");
  return SME_OK;
}

inline size_t coo_stage_bytes(int64_t n_rows, int64_t nnz) {  // cursor sized for int64 row_ptr
  return align_up(n_rows * 8) + align_up(nnz * 4) + align_up(nnz * 8);
}

}  // namespace sme

using namespace sme;

#define CHECK_DIMS(n_rows, n_cols)                                                               \
  SME_REQUIRE((n_rows) >= 0 && (n_rows) < INT32_MAX && (n_cols) >= 0 && (n_cols) < INT32_MAX,   \
              "matrix dimensions must be non-negative and < 2^31-1")
#define CHECK_SIZES(n_rows, n_cols, nnz)                                                         \
  CHECK_DIMS(n_rows, n_cols);                                                                    \
  SME_REQUIRE((nnz) >= 0 && (nnz) < INT32_MAX, "nnz %lld exceeds int32 offsets (use the _i64 entry point)", \
              (long long)(nnz))
// the _i64 entry points: int64 row_ptr, any nnz
#define CHECK_SIZES_WIDE(n_rows, n_cols, nnz)                                                    \
  CHECK_DIMS(n_rows, n_cols);                                                                    \
  SME_REQUIRE((nnz) >= 0, "negative nnz")

SME_API int sme_row_ptr_workspace_size(int64_t n_rows, size_t* bytes) {
  SME_REQUIRE(bytes, "null pointer");
  *bytes = align_up(n_rows * 4) + scan_workspace_bytes(n_rows);
  return SME_OK;
}

template <typename IP>
static int coo_row_ptr_impl(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* row, const int32_t* col,
                            const int32_t* row_map, IP* row_ptr_out, void* ws, size_t ws_bytes, int32_t* flag,
                            cudaStream_t s) {
  size_t need = align_up(n_rows * 4) + scan_workspace_bytes(n_rows);
  SME_REQUIRE(ws_bytes >= need, "workspace %zu < %zu", ws_bytes, need);
  int32_t* counts = (int32_t*)ws;
  void* scan_ws = (char*)ws + align_up(n_rows * 4);
  if (n_rows > 0) SME_CUDA(cudaMemsetAsync(counts, 0, n_rows * 4, s));
  if (nnz > 0) {
    k_coo_count<<<grid_for(nnz, 256), 256, 0, s>>>(nnz, n_rows, n_cols, row, col, row_map, counts, flag);
    SME_CHECK_LAUNCH("k_coo_count");
  }
  return exclusive_scan_lengths(n_rows, LenFromCounts{counts}, row_ptr_out, scan_ws, flag, s);
}

SME_API int sme_coo_row_ptr(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* row, const int32_t* col,
                            const int32_t* row_map, int32_t* row_ptr_out, void* ws, size_t ws_bytes,
                            int32_t* flag, sme_stream_t stream) {
  CHECK_SIZES(n_rows, n_cols, nnz);
  return coo_row_ptr_impl(n_rows, n_cols, nnz, row, col, row_map, row_ptr_out, ws, ws_bytes, flag,
                          as_stream(stream));
}

SME_API int sme_coo_row_ptr_i64(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* row, const int32_t* col,
                                const int32_t* row_map, int64_t* row_ptr_out, void* ws, size_t ws_bytes,
                                int32_t* flag, sme_stream_t stream) {
  CHECK_SIZES_WIDE(n_rows, n_cols, nnz);
  return coo_row_ptr_impl(n_rows, n_cols, nnz, row, col, row_map, row_ptr_out, ws, ws_bytes, flag,
                          as_stream(stream));
}

template <typename IP>
static int permute_row_ptr_impl(int64_t n_rows, const IP* row_ptr, const int32_t* inv_row, IP* row_ptr_out,
                                void* ws, size_t ws_bytes, sme_stream_t stream) {
  SME_REQUIRE(n_rows >= 0 && n_rows < INT32_MAX, "bad n_rows");
  size_t need = scan_workspace_bytes(n_rows);
  SME_REQUIRE(ws_bytes >= need, "workspace %zu < %zu", ws_bytes, need);
  return exclusive_scan_lengths(n_rows, LenFromGather<IP>{row_ptr, inv_row}, row_ptr_out, ws, nullptr,
                                as_stream(stream));
}

SME_API int sme_permute_csr_row_ptr(int64_t n_rows, const int32_t* row_ptr, const int32_t* inv_row,
                                    int32_t* row_ptr_out, void* ws, size_t ws_bytes, sme_stream_t stream) {
  return permute_row_ptr_impl(n_rows, row_ptr, inv_row, row_ptr_out, ws, ws_bytes, stream);
}

SME_API int sme_permute_csr_row_ptr_i64(int64_t n_rows, const int64_t* row_ptr, const int32_t* inv_row,
                                        int64_t* row_ptr_out, void* ws, size_t ws_bytes, sme_stream_t stream) {
  return permute_row_ptr_impl(n_rows, row_ptr, inv_row, row_ptr_out, ws, ws_bytes, stream);
}

template <typename IP>
static int long_row_nnz_impl(int64_t n_rows, const IP* row_ptr, int64_t* out, sme_stream_t stream) {
  cudaStream_t s = as_stream(stream);
  SME_CUDA(cudaMemsetAsync(out, 0, 8, s));
  if (n_rows == 0) return SME_OK;
  k_long_row_nnz<IP><<<grid_for(n_rows, 256, 4), 256, 0, s>>>(n_rows, row_ptr, (unsigned long long*)out);
  SME_CHECK_LAUNCH("k_long_row_nnz");
  return SME_OK;
}

// sme_permute_csr_row_ptr plus the source start of every new row (starts_out[r] =
// row_ptr[inv_row[r]]): the old row_ptr is gathered once, in the scan's first pass.  With
// starts as its row_ptr and inv_row = NULL, sme_permute_csr then reads the sources in order.
template <typename IP>
static int permute_row_ptr_starts_impl(int64_t n_rows, const IP* row_ptr, const int32_t* inv_row, IP* row_ptr_out,
                                       IP* starts_out, void* ws, size_t ws_bytes, sme_stream_t stream) {
  SME_REQUIRE(n_rows >= 0 && n_rows < INT32_MAX, "bad n_rows");
  const size_t need = align_up(n_rows * 4) + scan_workspace_bytes(n_rows);
  SME_REQUIRE(ws_bytes >= need, "workspace %zu < %zu", ws_bytes, need);
  cudaStream_t s = as_stream(stream);
  if (n_rows == 0) {
    SME_CUDA(cudaMemsetAsync(row_ptr_out, 0, sizeof(IP), s));
    return SME_OK;
  }
  int32_t* len = (int32_t*)ws;
  int64_t* sums = reinterpret_cast<int64_t*>((char*)ws + align_up(n_rows * 4));
  const int64_t tiles = scan_tiles(n_rows);
  k_scan_tile_sums<<<(unsigned)tiles, SCAN_NT, 0, s>>>(n_rows, LenGatherStore<IP>{row_ptr, inv_row, len, starts_out},
                                                      sums);
  SME_CHECK_LAUNCH("k_scan_tile_sums");
  k_scan_tile_offsets<<<1, 1024, 0, s>>>(tiles, sums);
  SME_CHECK_LAUNCH("k_scan_tile_offsets");
  k_scan_apply<<<(unsigned)tiles, SCAN_NT, 0, s>>>(n_rows, LenFromArray{len}, sums, row_ptr_out, (int32_t*)nullptr);
  SME_CHECK_LAUNCH("k_scan_apply");
  return SME_OK;
}

SME_API int sme_permute_csr_row_ptr_starts(int64_t n_rows, const int32_t* row_ptr, const int32_t* inv_row,
                                           int32_t* row_ptr_out, int32_t* starts_out, void* ws, size_t ws_bytes,
                                           sme_stream_t stream) {
  return permute_row_ptr_starts_impl(n_rows, row_ptr, inv_row, row_ptr_out, starts_out, ws, ws_bytes, stream);
}

SME_API int sme_permute_csr_row_ptr_starts_i64(int64_t n_rows, const int64_t* row_ptr, const int32_t* inv_row,
                                               int64_t* row_ptr_out, int64_t* starts_out, void* ws, size_t ws_bytes,
                                               sme_stream_t stream) {
  return permute_row_ptr_starts_impl(n_rows, row_ptr, inv_row, row_ptr_out, starts_out, ws, ws_bytes, stream);
}

SME_API int sme_long_row_nnz(int64_t n_rows, const int32_t* row_ptr, int64_t* out, sme_stream_t stream) {
  return long_row_nnz_impl(n_rows, row_ptr, out, stream);
}

SME_API int sme_long_row_nnz_i64(int64_t n_rows, const int64_t* row_ptr, int64_t* out, sme_stream_t stream) {
  return long_row_nnz_impl(n_rows, row_ptr, out, stream);
}

SME_API int sme_coo_to_csr_workspace_size(int64_t n_rows, int64_t nnz, int64_t long_nnz, size_t* bytes) {
  SME_REQUIRE(bytes && n_rows >= 0 && nnz >= 0 && long_nnz >= 0, "bad arguments");
  *bytes = coo_stage_bytes(n_rows, nnz) + lists_bytes(n_rows, long_nnz);
  return SME_OK;
}

template <typename IP>
static int coo_to_csr_impl(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* row,
                           const int32_t* col, const void* val, const int32_t* row_map, const int32_t* col_map,
                           const IP* row_ptr, int32_t* col_out, void* val_out, void* ws, size_t ws_bytes,
                           int64_t long_nnz, int32_t* flag, uint64_t* dup_key, sme_stream_t stream, int mark) {
  SME_REQUIRE(dtype == SME_F64 || dtype == SME_F32, "unknown dtype %d", dtype);
  size_t need = coo_stage_bytes(n_rows, nnz) + lists_bytes(n_rows, long_nnz);
  SME_REQUIRE(ws_bytes >= need, "workspace %zu < %zu", ws_bytes, need);
  if (nnz == 0 || n_rows == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  char* p = (char*)ws;
  IP* cursor = (IP*)p;            p += align_up(n_rows * 8);
  int32_t* st_col = (int32_t*)p;  p += align_up(nnz * 4);
  void* st_val = p;               p += align_up(nnz * 8);
  SortLists L = carve_lists(p, n_rows, long_nnz);
  L.mark_dups = mark;
  SME_CUDA(cudaMemsetAsync(L.counters, 0, 64, s));
  SME_CUDA(cudaMemcpyAsync(cursor, row_ptr, n_rows * sizeof(IP), cudaMemcpyDeviceToDevice, s));
  if (dtype == SME_F64) {
    k_coo_scatter<double, IP><<<grid_for(nnz, 256), 256, 0, s>>>(nnz, n_rows, n_cols, row, col, (const double*)val,
                                                                row_map, cursor, st_col, (double*)st_val);
    SME_CHECK_LAUNCH("k_coo_scatter");
    return launch_sorts<double>(n_rows, row_ptr, SrcStaged{}, st_col, (const double*)st_val, col_map, col_out,
                                (double*)val_out, L, flag, dup_key, s, n_cols);
  } else {
    k_coo_scatter<float, IP><<<grid_for(nnz, 256), 256, 0, s>>>(nnz, n_rows, n_cols, row, col, (const float*)val,
                                                               row_map, cursor, st_col, (float*)st_val);
    SME_CHECK_LAUNCH("k_coo_scatter");
    return launch_sorts<float>(n_rows, row_ptr, SrcStaged{}, st_col, (const float*)st_val, col_map, col_out,
                               (float*)val_out, L, flag, dup_key, s, n_cols);
  }
}

SME_API int sme_coo_to_csr(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* row,
                           const int32_t* col, const void* val, const int32_t* row_map, const int32_t* col_map,
                           const int32_t* row_ptr, int32_t* col_out, void* val_out, void* ws, size_t ws_bytes,
                           int64_t long_nnz, int32_t* flag, uint64_t* dup_key, sme_stream_t stream) {
  CHECK_SIZES(n_rows, n_cols, nnz);
  return coo_to_csr_impl(dtype, n_rows, n_cols, nnz, row, col, val, row_map, col_map, row_ptr, col_out, val_out, ws,
                         ws_bytes, long_nnz, flag, dup_key, stream, 0);
}

SME_API int sme_coo_to_csr_i64(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* row,
                               const int32_t* col, const void* val, const int32_t* row_map, const int32_t* col_map,
                               const int64_t* row_ptr, int32_t* col_out, void* val_out, void* ws, size_t ws_bytes,
                               int64_t long_nnz, int32_t* flag, uint64_t* dup_key, sme_stream_t stream) {
  CHECK_SIZES_WIDE(n_rows, n_cols, nnz);
  return coo_to_csr_impl(dtype, n_rows, n_cols, nnz, row, col, val, row_map, col_map, row_ptr, col_out, val_out, ws,
                         ws_bytes, long_nnz, flag, dup_key, stream, 0);
}

// Same, but duplicates are kept as col = -1 holes (no error) for sme_csr_compact:
// the dedupe step of generated graphs (R-MAT edge lists).
SME_API int sme_coo_to_csr_dedup(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* row,
                                 const int32_t* col, const void* val, const int32_t* row_ptr, int32_t* col_out,
                                 void* val_out, void* ws, size_t ws_bytes, int64_t long_nnz, int32_t* flag,
                                 sme_stream_t stream) {
  CHECK_SIZES(n_rows, n_cols, nnz);
  return coo_to_csr_impl(dtype, n_rows, n_cols, nnz, row, col, val, nullptr, nullptr, row_ptr, col_out, val_out, ws,
                         ws_bytes, long_nnz, flag, nullptr, stream, 1);
}

SME_API int sme_permute_csr_workspace_size(int64_t n_rows, int64_t nnz, int64_t long_nnz, size_t* bytes) {
  SME_REQUIRE(bytes && n_rows >= 0 && nnz >= 0 && long_nnz >= 0, "bad arguments");
  *bytes = lists_bytes(n_rows, long_nnz);
  return SME_OK;
}

template <typename IP>
static int permute_csr_impl(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz, const IP* row_ptr,
                            const int32_t* col, const void* val, const int32_t* inv_row, const int32_t* col_map,
                            const IP* row_ptr_out, int32_t* col_out, void* val_out, void* ws, size_t ws_bytes,
                            int64_t long_nnz, int32_t* flag, uint64_t* dup_key, sme_stream_t stream) {
  SME_REQUIRE(dtype == SME_F64 || dtype == SME_F32, "unknown dtype %d", dtype);
  size_t need = lists_bytes(n_rows, long_nnz);
  SME_REQUIRE(ws_bytes >= need, "workspace %zu < %zu", ws_bytes, need);
  if (nnz == 0 || n_rows == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  SortLists L = carve_lists((char*)ws, n_rows, long_nnz);
  SME_CUDA(cudaMemsetAsync(L.counters, 0, 64, s));
  SrcGather<IP> src{row_ptr, inv_row};
  if (dtype == SME_F64)
    return launch_sorts<double>(n_rows, row_ptr_out, src, col, (const double*)val, col_map, col_out,
                                (double*)val_out, L, flag, dup_key, s, n_cols);
  return launch_sorts<float>(n_rows, row_ptr_out, src, col, (const float*)val, col_map, col_out,
                             (float*)val_out, L, flag, dup_key, s, n_cols);
}

SME_API int sme_permute_csr(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* row_ptr,
                            const int32_t* col, const void* val, const int32_t* inv_row, const int32_t* col_map,
                            const int32_t* row_ptr_out, int32_t* col_out, void* val_out, void* ws,
                            size_t ws_bytes, int64_t long_nnz, int32_t* flag, uint64_t* dup_key,
                            sme_stream_t stream) {
  CHECK_SIZES(n_rows, n_cols, nnz);
  return permute_csr_impl(dtype, n_rows, n_cols, nnz, row_ptr, col, val, inv_row, col_map, row_ptr_out, col_out,
                          val_out, ws, ws_bytes, long_nnz, flag, dup_key, stream);
}

SME_API int sme_permute_csr_i64(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                                const int32_t* col, const void* val, const int32_t* inv_row, const int32_t* col_map,
                                const int64_t* row_ptr_out, int32_t* col_out, void* val_out, void* ws,
                                size_t ws_bytes, int64_t long_nnz, int32_t* flag, uint64_t* dup_key,
                                sme_stream_t stream) {
  CHECK_SIZES_WIDE(n_rows, n_cols, nnz);
  return permute_csr_impl(dtype, n_rows, n_cols, nnz, row_ptr, col, val, inv_row, col_map, row_ptr_out, col_out,
                          val_out, ws, ws_bytes, long_nnz, flag, dup_key, stream);
}

namespace sme {
// One pass of the column-sliced pre-map.  A random 4-byte gather from a column map
// larger than L2 costs a 64-byte DRAM access (tools/l2fetch_bench.cu: 73 B of DRAM and
// 86-90 G gathers/s from a 200 MB table, 287 G/s from a 50 MB one), so the map is
// applied in passes, pass q relabelling only the columns of slice [lo, hi) while that
// 1/n_slices of cmap stays L2-resident.  Every pass rewrites whole 16-byte vectors (no
// partial-sector writes): an entry already relabelled carries bit 31 (columns are
// < 2^31), and the last pass maps what is left and clears the flags.
//   PASS 0: first of several (read col, write out)   PASS 1: middle (out in place)
//   PASS 2: last (out in place)                       PASS 3: single pass (col -> out)
template <int PASS>
__device__ __forceinline__ int32_t map_one(int32_t v, const int32_t* __restrict__ cmap, int32_t lo, int32_t hi,
                                           uint64_t keep) {
  constexpr int32_t FLAG = (int32_t)0x80000000;
  if (PASS == 3) return ld_l1(cmap + v, keep);
  if (PASS == 2) return v < 0 ? (v & 0x7fffffff) : ld_l1(cmap + v, keep);
  // PASS 0/1: flagged (negative) entries fail the range test
  return (v >= lo && v < hi) ? (ld_l1(cmap + v, keep) | FLAG) : v;
}

template <int PASS>
__global__ void __launch_bounds__(256) k_map_cols_pass(int64_t nnz, const int32_t* __restrict__ src,
                                                       const int32_t* __restrict__ cmap, int32_t* __restrict__ out,
                                                       int32_t lo, int32_t hi) {
  const uint64_t once = policy_evict_first(), keep = policy_evict_last();
  const int64_t n4 = nnz / 4;
  const int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t q = (int64_t)blockIdx.x * blockDim.x + threadIdx.x;
  // two vectors per thread per iteration: 8 independent gathers in flight
  for (; q + stride < n4; q += 2 * stride) {
    int4 a = ld_stream_i4(reinterpret_cast<const int4*>(src) + q, once);
    int4 b = ld_stream_i4(reinterpret_cast<const int4*>(src) + q + stride, once);
    a.x = map_one<PASS>(a.x, cmap, lo, hi, keep); a.y = map_one<PASS>(a.y, cmap, lo, hi, keep);
    a.z = map_one<PASS>(a.z, cmap, lo, hi, keep); a.w = map_one<PASS>(a.w, cmap, lo, hi, keep);
    b.x = map_one<PASS>(b.x, cmap, lo, hi, keep); b.y = map_one<PASS>(b.y, cmap, lo, hi, keep);
    b.z = map_one<PASS>(b.z, cmap, lo, hi, keep); b.w = map_one<PASS>(b.w, cmap, lo, hi, keep);
    __stcs(reinterpret_cast<int4*>(out) + q, a);
    __stcs(reinterpret_cast<int4*>(out) + q + stride, b);
  }
  for (; q < n4; q += stride) {
    int4 a = ld_stream_i4(reinterpret_cast<const int4*>(src) + q, once);
    a.x = map_one<PASS>(a.x, cmap, lo, hi, keep); a.y = map_one<PASS>(a.y, cmap, lo, hi, keep);
    a.z = map_one<PASS>(a.z, cmap, lo, hi, keep); a.w = map_one<PASS>(a.w, cmap, lo, hi, keep);
    __stcs(reinterpret_cast<int4*>(out) + q, a);
  }
  if (blockIdx.x == 0)
    for (int64_t k = n4 * 4 + threadIdx.x; k < nnz; k += blockDim.x) out[k] = map_one<PASS>(src[k], cmap, lo, hi, keep);
}
}  // namespace sme

// The first n_passes of the n_slices-pass column relabelling mapped[k] = cmap[col[k]]
// (permute.py:98-102), pass q relabelling the columns of slice q with that slice of cmap
// L2-resident (evict-last gathers, evict-first streams, and an access-policy window on
// `stream` that pins the slice when the caller reserved persisting L2): the random cmap
// reads hit L2 instead of costing a 64-byte DRAM access each.  The first pass reads col
// and writes mapped, the others rewrite mapped in place.  With n_passes == n_slices the
// result is the plain relabelling; with fewer, relabelled entries carry bit 31 and the
// rest keep their old id, which the row sort of sme_permute_csr (given cmap) finishes:
// it maps unflagged entries and clears the flag of the others.  col and mapped must be
// 16-byte aligned; mapped may alias col only when n_slices == 1.
SME_API int sme_map_cols_sliced_partial(int64_t nnz, int64_t n_cols, const int32_t* col, const int32_t* cmap,
                                        int32_t* mapped, int32_t n_slices, int32_t n_passes,
                                        sme_stream_t stream) {
  SME_REQUIRE(nnz >= 0 && n_cols >= 1 && n_slices >= 1 && col && cmap && mapped, "bad arguments");
  SME_REQUIRE(n_passes >= 1 && n_passes <= n_slices, "n_passes must be in [1, n_slices]");
  SME_REQUIRE(n_cols <= INT32_MAX, "n_cols must be < 2^31");
  SME_REQUIRE(((uintptr_t)col & 15) == 0 && ((uintptr_t)mapped & 15) == 0, "col and mapped must be 16-byte aligned");
  if (nnz == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  const int grid = grid_for((nnz + 3) / 4, 256, 8);
  for (int32_t q = 0; q < n_passes; ++q) {
    const int64_t lo = n_cols * q / n_slices, hi = n_cols * (q + 1) / n_slices;
    cudaStreamAttrValue attr = {};
    attr.accessPolicyWindow.base_ptr = const_cast<int32_t*>(cmap + lo);
    attr.accessPolicyWindow.num_bytes = (size_t)(hi - lo) * 4;
    attr.accessPolicyWindow.hitRatio = 1.0f;
    attr.accessPolicyWindow.hitProp = cudaAccessPropertyPersisting;
    attr.accessPolicyWindow.missProp = cudaAccessPropertyStreaming;
    if (n_slices > 1) SME_CUDA(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &attr));
    const int32_t* in = q == 0 ? col : mapped;
    if (n_slices == 1)
      k_map_cols_pass<3><<<grid, 256, 0, s>>>(nnz, in, cmap, mapped, (int32_t)lo, (int32_t)hi);
    else if (q + 1 == n_slices)
      k_map_cols_pass<2><<<grid, 256, 0, s>>>(nnz, in, cmap, mapped, (int32_t)lo, (int32_t)hi);
    else if (q == 0)
      k_map_cols_pass<0><<<grid, 256, 0, s>>>(nnz, in, cmap, mapped, (int32_t)lo, (int32_t)hi);
    else
      k_map_cols_pass<1><<<grid, 256, 0, s>>>(nnz, in, cmap, mapped, (int32_t)lo, (int32_t)hi);
    SME_CHECK_LAUNCH("k_map_cols_pass");
  }
  if (n_slices > 1) {
    cudaStreamAttrValue clear = {};
    SME_CUDA(cudaStreamSetAttribute(s, cudaStreamAttributeAccessPolicyWindow, &clear));
  }
  return SME_OK;
}

// mapped[k] = cmap[col[k]]: all n_slices passes of the above.
SME_API int sme_map_cols_sliced(int64_t nnz, int64_t n_cols, const int32_t* col, const int32_t* cmap,
                                int32_t* mapped, int32_t n_slices, sme_stream_t stream) {
  return sme_map_cols_sliced_partial(nnz, n_cols, col, cmap, mapped, n_slices, n_slices, stream);
}

template <typename IP>
static int row_stats_impl(int64_t n_rows, const IP* row_ptr, int64_t* out, sme_stream_t stream) {
  cudaStream_t s = as_stream(stream);
  SME_CUDA(cudaMemsetAsync(out, 0, 16, s));
  if (n_rows == 0) return SME_OK;
  k_row_stats<IP><<<grid_for(n_rows, 256, 4), 256, 0, s>>>(n_rows, row_ptr, (unsigned long long*)out);
  SME_CHECK_LAUNCH("k_row_stats");
  return SME_OK;
}

template <typename IP>
static int row_spans_impl(int64_t n_rows, const IP* row_ptr, const int32_t* col, int32_t n_samples, int32_t* out,
                          sme_stream_t stream) {
  SME_REQUIRE(n_rows >= 1 && n_samples >= 1, "bad arguments");
  k_row_spans<IP><<<(n_samples + 255) / 256, 256, 0, as_stream(stream)>>>(n_rows, row_ptr, col, n_samples, out);
  SME_CHECK_LAUNCH("k_row_spans");
  return SME_OK;
}

SME_API int sme_row_spans(int64_t n_rows, const int32_t* row_ptr, const int32_t* col, int32_t n_samples, int32_t* out,
                          sme_stream_t stream) {
  return row_spans_impl(n_rows, row_ptr, col, n_samples, out, stream);
}

SME_API int sme_row_spans_i64(int64_t n_rows, const int64_t* row_ptr, const int32_t* col, int32_t n_samples,
                              int32_t* out, sme_stream_t stream) {
  return row_spans_impl(n_rows, row_ptr, col, n_samples, out, stream);
}

SME_API int sme_row_stats(int64_t n_rows, const int32_t* row_ptr, int64_t* out, sme_stream_t stream) {
  return row_stats_impl(n_rows, row_ptr, out, stream);
}

SME_API int sme_row_stats_i64(int64_t n_rows, const int64_t* row_ptr, int64_t* out, sme_stream_t stream) {
  return row_stats_impl(n_rows, row_ptr, out, stream);
}

template <typename IP>
static int csr_validate_impl(int64_t n_rows, int64_t n_cols, int64_t nnz, const IP* row_ptr, const int32_t* col,
                             int32_t* flag, sme_stream_t stream) {
  cudaStream_t s = as_stream(stream);
  k_csr_validate<IP><<<grid_for(n_rows + 1, 256), 256, 0, s>>>(n_rows, n_cols, nnz, row_ptr, col, flag);
  SME_CHECK_LAUNCH("k_csr_validate");
  return SME_OK;
}

SME_API int sme_csr_validate(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* row_ptr,
                             const int32_t* col, int32_t* flag, sme_stream_t stream) {
  CHECK_SIZES(n_rows, n_cols, nnz);
  return csr_validate_impl(n_rows, n_cols, nnz, row_ptr, col, flag, stream);
}

SME_API int sme_csr_validate_i64(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* row_ptr,
                                 const int32_t* col, int32_t* flag, sme_stream_t stream) {
  CHECK_SIZES_WIDE(n_rows, n_cols, nnz);
  return csr_validate_impl(n_rows, n_cols, nnz, row_ptr, col, flag, stream);
}

template <typename IP>
static int expand_rows_impl(int64_t n_rows, const IP* row_ptr, int32_t* row_out, sme_stream_t stream) {
  if (n_rows == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  k_csr_expand_rows<IP><<<grid_for(n_rows * 32, 256), 256, 0, s>>>(n_rows, row_ptr, row_out);
  SME_CHECK_LAUNCH("k_csr_expand_rows");
  return SME_OK;
}

SME_API int sme_csr_expand_rows(int64_t n_rows, const int32_t* row_ptr, int32_t* row_out, sme_stream_t stream) {
  return expand_rows_impl(n_rows, row_ptr, row_out, stream);
}

SME_API int sme_csr_expand_rows_i64(int64_t n_rows, const int64_t* row_ptr, int32_t* row_out,
                                    sme_stream_t stream) {
  return expand_rows_impl(n_rows, row_ptr, row_out, stream);
}

// ---------------------------------------------------------------------------
// compaction: drop col = -1 holes and keep at most `cap` entries per row (the
// first ones in column order) — the dedupe + degree cap of generated graphs
// ---------------------------------------------------------------------------
namespace sme {
struct LenCompact {
  const int32_t* ptr;
  const int32_t* col;
  int32_t cap;
  __device__ __forceinline__ int64_t operator()(int64_t r) const {
    int32_t n = 0;
    for (int32_t k = ptr[r]; k < ptr[r + 1] && n < cap; ++k) n += col[k] >= 0;
    return n;
  }
};

template <typename T>
__global__ void k_csr_compact(int64_t n_rows, const int32_t* __restrict__ ptr, const int32_t* __restrict__ col,
                              const T* __restrict__ val, int32_t cap, const int32_t* __restrict__ out_ptr,
                              int32_t* __restrict__ out_col, T* __restrict__ out_val) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    int32_t o = out_ptr[r];
    const int32_t end = out_ptr[r + 1];
    for (int32_t k = ptr[r]; k < ptr[r + 1] && o < end; ++k)
      if (col[k] >= 0) { out_col[o] = col[k]; out_val[o] = val[k]; ++o; }
  }
}
}  // namespace sme

SME_API int sme_csr_compact_row_ptr(int64_t n_rows, const int32_t* row_ptr, const int32_t* col, int32_t cap,
                                    int32_t* out_row_ptr, void* ws, size_t ws_bytes, sme_stream_t stream) {
  SME_REQUIRE(cap >= 1, "cap must be >= 1");
  SME_REQUIRE(ws_bytes >= scan_workspace_bytes(n_rows), "workspace too small");
  return exclusive_scan_lengths(n_rows, LenCompact{row_ptr, col, cap}, out_row_ptr, ws, nullptr, as_stream(stream));
}

SME_API int sme_csr_compact(int dtype, int64_t n_rows, const int32_t* row_ptr, const int32_t* col, const void* val,
                            int32_t cap, const int32_t* out_row_ptr, int32_t* out_col, void* out_val,
                            sme_stream_t stream) {
  if (n_rows == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == SME_F64)
    k_csr_compact<double><<<grid_for(n_rows, 256), 256, 0, s>>>(n_rows, row_ptr, col, (const double*)val, cap,
                                                               out_row_ptr, out_col, (double*)out_val);
  else if (dtype == SME_F32)
    k_csr_compact<float><<<grid_for(n_rows, 256), 256, 0, s>>>(n_rows, row_ptr, col, (const float*)val, cap,
                                                              out_row_ptr, out_col, (float*)out_val);
  else
    SME_REQUIRE(false, "unknown dtype %d", dtype);
  SME_CHECK_LAUNCH("k_csr_compact");
  return SME_OK;
}

// Test hook: 0 forces the 64-bit sort keys of k_sort_rows_warp (the path of n_cols > 2^27).
// Rows with 32 < len <= 32 << level: warp-wide register sort (level 1..4), longer ones
// the CTA-wide shared-memory sort; level 0: every row > 32 takes the CTA sort.
// Process-wide; for A/B tests.
SME_API int sme_sort_rows_set_wmed(int level) {
  SME_REQUIRE(level >= 0 && level <= 4, "level must lie in [0, 4]");
  g_sort_wmed = level;
  return SME_OK;
}

SME_API int sme_sort_rows_set_cta(int enable) {
  g_sort_cta = enable != 0;
  return SME_OK;
}

SME_API int sme_sort_rows_set_key32(int enable) {
  SME_REQUIRE(enable == 0 || enable == 1, "enable must be 0 or 1");
  g_sort_key32 = enable;
  return SME_OK;
}

namespace sme {
// Lazy module loading (CUDA 12 default) loads this file's module on the first launch of
// any of its kernels, ~10-20 ms each; sme_preload() does it ahead of time.
int preload_csr_build() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)k_coo_count) == cudaSuccess ? 0 : -1;
}
}  // namespace sme
