// shuffle.cu — the swaps of a Fisher–Yates shuffle, applied in parallel (the APPLY
// half of Generator(PCG64).permutation, permute.py:71-81; the swap partners come
// from the host, sme_host_pcg64_swap_partners, bit-exact with numpy's draws).
//
// numpy runs  a = arange(n); for i = n-1 .. 1: swap(a[i], a[j_i])  (j_i <= i).
// Position i is final after step i (later steps only touch positions < i), so
//   a[i] = value at position j_i just before step i.
// That value was last written by the smallest step s > i with j_s = j_i (it moved
// a[s]'s then-value there), or is j_i itself if no such step exists; and a[s]'s
// value just before step s is, recursively, G(s):
//   next(p) = smallest step s > p with j_s = p      (the last writer of position p
//                                                     before step p)
//   G(s)    = G(next(s)) if next(s) exists, else s  (follow the chain upwards)
//   a[i]    = G(succ(i)) if succ(i) exists, else j_i,  succ(i) = smallest s > i with
//             j_s = j_i (the successor of i in bucket j_i);   a[0] = G(next(0)) or 0.
// So the shuffle is a bucket sort of the steps by partner, one link pass and a
// chain walk per position — O(n) parallel work instead of n dependent swaps.
// Buckets are small (bucket p holds ~ln(n/p) steps) and chains short, so the
// sort is an insertion sort per bucket and the walk a plain loop.
// Verified against the sequential shuffle by tests/test_gpu_shuffle.py.
#include "common.cuh"
#include "scan.cuh"

namespace sme {

__global__ void k_fy_count(int64_t n, const uint32_t* __restrict__ j, int32_t* __restrict__ counts) {
  for (int64_t s = 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x)
    atomicAdd(&counts[j[s]], 1);
}

// cursor[p] starts at off[p]: one random atomic per step instead of a read of off[p] plus an
// atomic on a zeroed counter
__global__ void k_fy_fill(int64_t n, const uint32_t* __restrict__ j, int32_t* __restrict__ cursor,
                          int32_t* __restrict__ bucket) {
  for (int64_t s = 1 + (int64_t)blockIdx.x * blockDim.x + threadIdx.x; s < n; s += (int64_t)gridDim.x * blockDim.x) {
    const uint32_t p = j[s];
    bucket[atomicAdd(&cursor[p], 1)] = (int32_t)s;
  }
}

// per bucket p: sort its steps ascending, link each to its successor, and
// next[p] = the first step > p
__global__ void k_fy_links(int64_t n, const int32_t* __restrict__ off, int32_t* __restrict__ bucket,
                           int32_t* __restrict__ succ, int32_t* __restrict__ nxt) {
  for (int64_t p = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; p < n; p += (int64_t)gridDim.x * blockDim.x) {
    const int32_t b = off[p], e = off[p + 1];
    for (int32_t m = b + 1; m < e; ++m) {  // insertion sort (buckets hold a few steps)
      const int32_t v = bucket[m];
      int32_t q = m - 1;
      while (q >= b && bucket[q] > v) {
        bucket[q + 1] = bucket[q];
        --q;
      }
      bucket[q + 1] = v;
    }
    int32_t first_gt = -1;
    for (int32_t m = b; m < e; ++m) {
      const int32_t v = bucket[m];
      succ[v] = m + 1 < e ? bucket[m + 1] : -1;
      if (first_gt < 0 && v > p) first_gt = v;
    }
    nxt[p] = first_gt;
  }
}

__global__ void k_fy_final(int64_t n, const uint32_t* __restrict__ j, const int32_t* __restrict__ succ,
                           const int32_t* __restrict__ nxt, int32_t* __restrict__ perm) {
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (int64_t)gridDim.x * blockDim.x) {
    const int32_t s = i == 0 ? nxt[0] : succ[i];
    int32_t v;
    if (s < 0) {
      v = i == 0 ? 0 : (int32_t)j[i];
    } else {
      v = s;
      for (int32_t t = nxt[v]; t >= 0; t = nxt[v]) v = t;
    }
    perm[i] = v;
  }
}

inline size_t fy_ws_bytes(int64_t n) {  // counts (later succ), bucket, nxt, off, scan scratch
  return align_up((size_t)n * 4) * 3 + align_up((size_t)(n + 1) * 4) + scan_workspace_bytes(n);
}

}  // namespace sme

using namespace sme;

SME_API int sme_fy_apply_workspace_size(int64_t n, size_t* bytes) {
  SME_REQUIRE(bytes && n >= 1 && n < INT32_MAX, "bad arguments");
  *bytes = fy_ws_bytes(n);
  return SME_OK;
}

// perm = the permutation numpy's Fisher-Yates builds from the swap partners
// d_j[1..n-1] (d_j[0] ignored): perm[i] = a[i] after  a = arange(n);
// for i = n-1..1: swap(a[i], a[j_i]).
SME_API int sme_fy_apply(int64_t n, const uint32_t* d_j, int32_t* d_perm, void* ws, size_t ws_bytes,
                         sme_stream_t stream) {
  SME_REQUIRE(n >= 1 && n < INT32_MAX && d_j && d_perm, "bad arguments");
  SME_REQUIRE(ws_bytes >= fy_ws_bytes(n), "workspace %zu < %zu", ws_bytes, fy_ws_bytes(n));
  cudaStream_t s = as_stream(stream);
  char* p = (char*)ws;
  int32_t* counts = (int32_t*)p;  p += align_up((size_t)n * 4);
  int32_t* succ = counts;         // the counts / fill cursors are dead once the buckets are filled
  int32_t* bucket = (int32_t*)p;  p += align_up((size_t)n * 4);
  int32_t* nxt = (int32_t*)p;     p += align_up((size_t)n * 4);
  int32_t* off = (int32_t*)p;     p += align_up((size_t)(n + 1) * 4);
  void* scan_ws = p;
  SME_CUDA(cudaMemsetAsync(counts, 0, (size_t)n * 4, s));
  const int grid = grid_for(n, 256);
  k_fy_count<<<grid, 256, 0, s>>>(n, d_j, counts);
  SME_CHECK_LAUNCH("k_fy_count");
  int rc = exclusive_scan_lengths(n, LenFromArray{counts}, off, scan_ws, nullptr, s);
  if (rc != SME_OK) return rc;
  SME_CUDA(cudaMemcpyAsync(counts, off, (size_t)n * 4, cudaMemcpyDeviceToDevice, s));  // the fill cursors
  k_fy_fill<<<grid, 256, 0, s>>>(n, d_j, counts, bucket);
  SME_CHECK_LAUNCH("k_fy_fill");
  k_fy_links<<<grid, 256, 0, s>>>(n, off, bucket, succ, nxt);
  SME_CHECK_LAUNCH("k_fy_links");
  k_fy_final<<<grid, 256, 0, s>>>(n, d_j, succ, nxt, d_perm);
  SME_CHECK_LAUNCH("k_fy_final");
  return SME_OK;
}

namespace sme {
// Lazy module loading (CUDA 12 default) loads this file's module on the first launch of
// any of its kernels, ~10-20 ms each; sme_preload() does it ahead of time.
int preload_shuffle() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)k_fy_count) == cudaSuccess ? 0 : -1;
}
}  // namespace sme
