// panel.cu — column-panel split of a CSR matrix (x-locality layout for SpMV).
//
// When x (8 B x n_cols) is larger than the L2 share it can keep (C4: 400 MB
// against a 126 MB L2), every random x gather misses to DRAM and costs ~100 B
// of DRAM traffic (measured: 112 GB per C4 SpMV for 13 GB of algorithmic
// bytes).  Splitting the columns into P panels and running P accumulating
// SpMV passes keeps each pass's x slice L2-resident; the price is P-1 extra
// y read+write passes and P row_ptr arrays.  The split is a stable partition
// of every (column-sorted) row by panel, so each panel is itself a valid CSR
// (global column ids, columns ascending) and y = sum_p A_p x bit-for-bit
// reproduces the same products; only the association of row sums changes.
//
// Layout: one col/val buffer; panel p occupies [off_p, off_p + nnz_p) with
// off_p a multiple of 128 elements (so panel arrays stay 16-byte aligned and
// global 128-element chunk boundaries coincide with local ones); row_ptr_p is
// relative to off_p.
#include "common.cuh"
#include "scan.cuh"

namespace sme {

// counts[p * n_rows + r] = entries of row r with panel boundary b_p <= col < b_{p+1}
__global__ void k_panel_count(int64_t n_rows, const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                              int32_t n_panels, const int32_t* __restrict__ bounds, int32_t* __restrict__ counts) {
  for (int64_t r = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; r < n_rows; r += (int64_t)gridDim.x * blockDim.x) {
    const int32_t a = row_ptr[r], b = row_ptr[r + 1];
    int32_t k = a;
    for (int p = 0; p < n_panels; ++p) {
      const int32_t hi = bounds[p + 1];
      int32_t k0 = k;
      while (k < b && col[k] < hi) ++k;
      counts[(int64_t)p * n_rows + r] = k - k0;
    }
  }
}

__global__ void k_panel_scatter(int64_t n_rows, const int32_t* __restrict__ row_ptr, const int32_t* __restrict__ col,
                                const void* __restrict__ val, int vbytes, int32_t n_panels,
                                const int32_t* __restrict__ bounds, const int32_t* __restrict__ panel_ptr,
                                const int64_t* __restrict__ offsets, int32_t* __restrict__ out_col,
                                void* __restrict__ out_val) {
  // warp per row keeps the reads of a row coalesced
  const int lane = threadIdx.x & 31;
  const int64_t warp = ((int64_t)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int64_t n_warps = ((int64_t)gridDim.x * blockDim.x) >> 5;
  for (int64_t r = warp; r < n_rows; r += n_warps) {
    const int32_t a = row_ptr[r], b = row_ptr[r + 1];
    for (int32_t k = a + lane; k < b; k += 32) {
      const int32_t c = col[k];
      int p = 0;
      while (p + 1 < n_panels && c >= bounds[p + 1]) ++p;
      // first entry of panel p in this row = a + sum of the row's counts in panels < p
      // = a + (panel_ptr_q[r+1]-panel_ptr_q[r]) summed over q < p
      int32_t first = a;
      for (int qq = 0; qq < p; ++qq) {
        const int32_t* pp = panel_ptr + (int64_t)qq * (n_rows + 1);
        first += pp[r + 1] - pp[r];
      }
      const int32_t* pp = panel_ptr + (int64_t)p * (n_rows + 1);
      const int64_t dst = offsets[p] + pp[r] + (k - first);
      out_col[dst] = c;
      if (vbytes == 8)
        reinterpret_cast<double*>(out_val)[dst] = reinterpret_cast<const double*>(val)[k];
      else
        reinterpret_cast<float*>(out_val)[dst] = reinterpret_cast<const float*>(val)[k];
    }
  }
}

}  // namespace sme

using namespace sme;

SME_API int sme_panel_count_workspace_size(int64_t n_rows, int32_t n_panels, size_t* bytes) {
  SME_REQUIRE(bytes && n_rows >= 0 && n_panels >= 1, "bad arguments");
  *bytes = align_up((size_t)n_panels * n_rows * 4) + scan_workspace_bytes(n_rows);
  return SME_OK;
}

// Step 1: per-panel row pointers (relative), panel_ptr = n_panels x (n_rows + 1) int32.
SME_API int sme_panel_row_ptrs(int64_t n_rows, const int32_t* row_ptr, const int32_t* col, int32_t n_panels,
                               const int32_t* bounds, int32_t* panel_ptr, void* ws, size_t ws_bytes,
                               sme_stream_t stream) {
  SME_REQUIRE(n_rows >= 0 && n_rows < INT32_MAX && n_panels >= 1, "bad arguments");
  size_t need = align_up((size_t)n_panels * n_rows * 4) + scan_workspace_bytes(n_rows);
  SME_REQUIRE(ws_bytes >= need, "workspace %zu < %zu", ws_bytes, need);
  if (n_rows == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  int32_t* counts = (int32_t*)ws;
  void* scan_ws = (char*)ws + align_up((size_t)n_panels * n_rows * 4);
  k_panel_count<<<grid_for(n_rows, 256), 256, 0, s>>>(n_rows, row_ptr, col, n_panels, bounds, counts);
  SME_CHECK_LAUNCH("k_panel_count");
  for (int p = 0; p < n_panels; ++p) {
    int rc = exclusive_scan_lengths(n_rows, LenFromArray{counts + (int64_t)p * n_rows},
                                    panel_ptr + (int64_t)p * (n_rows + 1), scan_ws, nullptr, s);
    if (rc != SME_OK) return rc;
  }
  return SME_OK;
}

// Step 2: scatter entries into the panel buffers at offsets[p] (int64, multiples of 128).
SME_API int sme_panel_scatter(int dtype, int64_t n_rows, const int32_t* row_ptr, const int32_t* col, const void* val,
                              int32_t n_panels, const int32_t* bounds, const int32_t* panel_ptr,
                              const int64_t* offsets, int32_t* out_col, void* out_val, sme_stream_t stream) {
  SME_REQUIRE(dtype == SME_F64 || dtype == SME_F32, "unknown dtype %d", dtype);
  if (n_rows == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  k_panel_scatter<<<grid_for(n_rows * 32, 256), 256, 0, s>>>(n_rows, row_ptr, col, val, dtype == SME_F64 ? 8 : 4,
                                                              n_panels, bounds, panel_ptr, offsets, out_col, out_val);
  SME_CHECK_LAUNCH("k_panel_scatter");
  return SME_OK;
}

namespace sme {
// Lazy module loading (CUDA 12 default) loads this file's module on the first launch of
// any of its kernels, ~10-20 ms each; sme_preload() does it ahead of time.
int preload_panel() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)k_panel_count) == cudaSuccess ? 0 : -1;
}
}  // namespace sme
