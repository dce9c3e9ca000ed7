// scan.cuh — exclusive prefix sum of per-row lengths into a row_ptr (int32, or int64
// for matrices with nnz >= 2^31).
//
// Reduce-then-scan in three launches (tile sums, one-block scan of tile sums,
// tile scan + offset).  The lengths come from a functor so the permuted row
// lengths (a gather through inv_r) never hit memory: bytes = 2 reads + 1 write
// of n int32 (the functor is evaluated twice).  Used for coo_to_csr's
// cumsum(bincount) (matio.py:292-293) and the permuted row_ptr.
#pragma once
#include "common.cuh"

namespace sme {

constexpr int SCAN_NT = 256;
constexpr int SCAN_IPT = 16;
constexpr int SCAN_TILE = SCAN_NT * SCAN_IPT;

inline int64_t scan_tiles(int64_t n) { return (n + SCAN_TILE - 1) / SCAN_TILE; }
inline size_t scan_workspace_bytes(int64_t n) { return align_up((size_t)(scan_tiles(n) + 1) * 8); }

// block-wide exclusive scan of one int64 per thread; returns the block total via *total
template <int NT>
__device__ __forceinline__ int64_t block_exclusive_scan(int64_t v, int64_t* total) {
  __shared__ int64_t s_warp[NT / 32];
  int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  int64_t incl = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    int64_t t = __shfl_up_sync(0xffffffffu, incl, o);
    if (lane >= o) incl += t;
  }
  if (lane == 31) s_warp[warp] = incl;
  __syncthreads();
  if (warp == 0) {
    int64_t w = lane < NT / 32 ? s_warp[lane] : 0;
    int64_t wi = w;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      int64_t t = __shfl_up_sync(0xffffffffu, wi, o);
      if (lane >= o) wi += t;
    }
    if (lane < NT / 32) s_warp[lane] = wi - w;  // exclusive warp offsets
    if (lane == NT / 32 - 1) *total = wi;
  }
  __syncthreads();
  int64_t r = s_warp[warp] + incl - v;
  __syncthreads();
  return r;
}

template <class LenFn>
__global__ void __launch_bounds__(SCAN_NT) k_scan_tile_sums(int64_t n, LenFn len, int64_t* tile_sums) {
  int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
  int64_t s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    int64_t k = base + (int64_t)i * SCAN_NT + threadIdx.x;
    if (k < n) s += len(k);
  }
  for (int o = 16; o; o >>= 1) s += __shfl_xor_sync(0xffffffffu, s, o);
  __shared__ int64_t sw[SCAN_NT / 32];
  if ((threadIdx.x & 31) == 0) sw[threadIdx.x >> 5] = s;
  __syncthreads();
  if (threadIdx.x == 0) {
    int64_t t = 0;
    for (int w = 0; w < SCAN_NT / 32; ++w) t += sw[w];
    tile_sums[blockIdx.x] = t;
  }
}

// one block: exclusive scan of tile sums in place; tile_sums[n_tiles] = grand total
static __global__ void __launch_bounds__(1024) k_scan_tile_offsets(int64_t n_tiles, int64_t* tile_sums) {
  __shared__ int64_t s_total;
  int64_t carry = 0;
  for (int64_t b = 0; b < n_tiles; b += 1024) {
    int64_t k = b + threadIdx.x;
    int64_t v = k < n_tiles ? tile_sums[k] : 0;
    int64_t t;
    int64_t ex = block_exclusive_scan<1024>(v, &s_total);
    __syncthreads();
    t = s_total;
    if (k < n_tiles) tile_sums[k] = carry + ex;
    carry += t;
    __syncthreads();
  }
  if (threadIdx.x == 0) tile_sums[n_tiles] = carry;
}

// out[k] = exclusive prefix (k < n); out[n] = total.  The tile's items are loaded coalesced
// (item i of thread t is k = base + i*NT + t) into shared memory, each thread then scans its
// SCAN_IPT consecutive items in registers, one block-wide scan adds the thread offsets, and
// the positions leave through shared memory with coalesced stores.  (The previous version
// ran SCAN_IPT block-wide scans per tile, each with its barriers: 219 us per 50M-row scan at
// 1.6 TB/s, latency-bound.)
__device__ __forceinline__ int scan_pad(int i) { return i + (i >> 5); }  // bank-conflict padding

template <class LenFn, typename OutT>
__global__ void __launch_bounds__(SCAN_NT) k_scan_apply(int64_t n, LenFn len, const int64_t* tile_offsets,
                                                        OutT* out, int32_t* flag) {
  constexpr bool NARROW = sizeof(OutT) == 4;
  constexpr int SLOTS = SCAN_TILE + SCAN_TILE / 32;
  __shared__ __align__(16) unsigned char s_buf[SLOTS * sizeof(OutT) > SLOTS * 4 ? SLOTS * sizeof(OutT) : SLOTS * 4];
  __shared__ int64_t s_total;
  int32_t* s_len = reinterpret_cast<int32_t*>(s_buf);
  OutT* s_out = reinterpret_cast<OutT*>(s_buf);
  const int t = threadIdx.x;
  const int64_t base = (int64_t)blockIdx.x * SCAN_TILE;
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    const int64_t k = base + (int64_t)i * SCAN_NT + t;
    s_len[scan_pad(i * SCAN_NT + t)] = k < n ? (int32_t)len(k) : 0;
  }
  __syncthreads();
  int32_t v[SCAN_IPT];
  int64_t tot = 0;
#pragma unroll
  for (int j = 0; j < SCAN_IPT; ++j) {
    v[j] = s_len[scan_pad(t * SCAN_IPT + j)];
    tot += v[j];
  }
  const int64_t off = tile_offsets[blockIdx.x] + block_exclusive_scan<SCAN_NT>(tot, &s_total);
  __syncthreads();  // every s_len read is done before s_out overwrites the buffer
  int64_t run = off;
  bool over = false;
#pragma unroll
  for (int j = 0; j < SCAN_IPT; ++j) {
    over |= NARROW && run > INT32_MAX;
    s_out[scan_pad(t * SCAN_IPT + j)] = (OutT)run;
    run += v[j];
  }
  if (over && flag) atomicOr(flag, SME_FLAG_RANGE);
  __syncthreads();
#pragma unroll
  for (int i = 0; i < SCAN_IPT; ++i) {
    const int64_t k = base + (int64_t)i * SCAN_NT + t;
    if (k < n) out[k] = s_out[scan_pad(i * SCAN_NT + t)];
  }
  if (blockIdx.x == gridDim.x - 1 && t == SCAN_NT - 1) {
    // the last thread's run is the grand total (items past n contribute 0)
    if (NARROW && run > INT32_MAX && flag) atomicOr(flag, SME_FLAG_RANGE);
    out[n] = (OutT)run;
  }
}

struct LenFromArray {
  const int32_t* a;
  __device__ __forceinline__ int64_t operator()(int64_t k) const { return a[k]; }
};

// Launch the three phases.  ws must hold scan_workspace_bytes(n).
template <class LenFn, typename OutT>
int exclusive_scan_lengths(int64_t n, LenFn len, OutT* out, void* ws, int32_t* flag, cudaStream_t s) {
  if (n == 0) {
    SME_CUDA(cudaMemsetAsync(out, 0, sizeof(OutT), s));
    return SME_OK;
  }
  int64_t tiles = scan_tiles(n);
  int64_t* sums = reinterpret_cast<int64_t*>(ws);
  k_scan_tile_sums<<<(unsigned)tiles, SCAN_NT, 0, s>>>(n, len, sums);
  SME_CHECK_LAUNCH("k_scan_tile_sums");
  k_scan_tile_offsets<<<1, 1024, 0, s>>>(tiles, sums);
  SME_CHECK_LAUNCH("k_scan_tile_offsets");
  k_scan_apply<<<(unsigned)tiles, SCAN_NT, 0, s>>>(n, len, sums, out, flag);
  SME_CHECK_LAUNCH("k_scan_apply");
  return SME_OK;
}

}  // namespace sme
