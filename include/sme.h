/*
 * sme.h — C-ABI of the B200 max_E SpMV hot path (libsme.so, sm_100a).
 *
 * "sme" = SpMV-Entropy.  Every entry point replaces one numpy expression of the
 * reference package `spmv_entropy` (/root/reference/pkg/src/spmv_entropy/...).
 * The reference file:line each call stands in for is cited next to it.
 *
 * Conventions:
 *   - plain pointers and sizes only, no torch types;
 *   - every pointer argument named d_* is DEVICE memory owned by the caller;
 *   - no allocation inside: scratch comes from a caller buffer sized by the
 *     matching *_workspace_size() query;
 *   - every call is stream-ordered on the passed stream and never synchronises
 *     the host; device-side validation results are written to device flags the
 *     caller reads when it chooses;
 *   - return value: SME_OK (0) or a negative SME_E* code; sme_last_error()
 *     returns a thread-local message for the last failure on this thread.
 *   - indices are int32 (n_rows, n_cols, nnz < 2^31); values are f64 or f32,
 *     selected by an sme_dtype argument.  The reference is int64/f64
 *     (matio.py:42-44, 97-99); parity compares after widening.
 */
#ifndef SME_H
#define SME_H

#include <stdint.h>
#include <stddef.h>

#ifdef __cplusplus
extern "C" {
#endif

typedef void* sme_stream_t; /* a cudaStream_t / CUstream; NULL = legacy default stream */

enum sme_status {
  SME_OK = 0,
  SME_EINVAL = -1,   /* bad argument: maps to ValueError at the Python boundary     */
  SME_ECUDA = -2,    /* CUDA launch/runtime error: maps to RuntimeError              */
  SME_ENOSPACE = -3, /* workspace smaller than *_workspace_size() said               */
};

enum sme_dtype { SME_F64 = 0, SME_F32 = 1 };

/* Device-side validation flag bits written by the CSR/COO/perm calls. */
enum sme_flag_bits {
  SME_FLAG_RANGE = 1,        /* an index lies outside [0, n)                                  */
  SME_FLAG_NOT_BIJECTION = 2,/* permutation is not a bijection (permute.py:34-36)              */
  SME_FLAG_DUPLICATE = 4,    /* duplicate (row, col) pair (matio.py:59-64, 288-291)            */
  SME_FLAG_ROWPTR = 8,       /* row_ptr decreasing / bad endpoints (matio.py:109-112)          */
  SME_FLAG_UNSORTED = 16,    /* columns not strictly increasing within a row (matio.py:116-122)*/
};

const char* sme_last_error(void);
int sme_version(void);
/* Number of SMs of the current device (grid sizing is done inside; exported for the host). */
int sme_device_sm_count(void);
/* Test hook (A/B timing only): -1 (default) the row sorts of the CSR builds run their
 * tuned number of occupancy-sized waves; 0 = fixed per-SM caps; k > 0 = k waves. */
int sme_set_resident_grids(int mode);
/* out[6]: L2 bytes, max persisting L2 bytes, max access-policy window bytes, SMs,
 * shared memory per SM, max opt-in shared memory per block. */
int sme_device_info(int64_t* out);
/* L2 residency control for the x slice of a column-panel pass: reserve persisting
 * L2 (device-wide) and set/clear the access-policy window of a stream. */
int sme_l2_set_persisting(size_t bytes);
int sme_l2_window(const void* d_ptr, size_t bytes, float hit_ratio, sme_stream_t stream);
/* Demote every persisting L2 line to normal (cudaCtxResetPersistingL2Cache).  Not
 * stream-ordered: it waits for the whole device, so pipelines call it once at the end,
 * not per step.  sme_l2_window(bytes = 0) only clears the stream's window. */
int sme_l2_reset_persisting(void);
/* Sequential L2 prefetch (evict-last) of a device range: warms a panel's x slice
 * before its random gathers (stream-ordered). */
int sme_l2_prefetch(const void* d_ptr, size_t bytes, sme_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Matrix Market I/O — matio.py (HOST calls: host buffers, no stream)        */
/* ------------------------------------------------------------------------ */

/* Entry body of parse_matrix_market (matio.py:196-239), multithreaded: buf/len
 * = the bytes after the size line, whose first line is number first_line_no.
 * field 0 real / 1 integer / 2 pattern; rows/cols int32[declared] (0-based),
 * vals f64[declared].  cr_newline: '\r' and "\r\n" also end lines.  threads <= 0:
 * all hardware threads.  status[4] = {error code (0 ok, 1 more than declared,
 * 2 field count, 3 malformed index, 4/5 row/col out of range, 6/7 malformed
 * integer/real value, 8 non-ASCII), 1-based error line, entries found, byte
 * offset of the error line in buf}.  Malformed content is reported through
 * status (return SME_OK); bad arguments return SME_EINVAL. */
int sme_host_mm_parse(const char* buf, int64_t len, int field, int64_t n_rows, int64_t n_cols, int64_t declared,
                      int64_t first_line_no, int cr_newline, int threads, int32_t* rows, int32_t* cols,
                      double* vals, int64_t* status);

/* Entry lines of _write_mm (matio.py:270-274): "i+1 j+1 %.17g\n" per entry into
 * out (cap >= 72 * n bytes), *out_len = bytes written; multithreaded. */
int sme_host_mm_format(const int64_t* rows, const int64_t* cols, const double* vals, int64_t n, char* out,
                       int64_t cap, int threads, int64_t* out_len);

/* ------------------------------------------------------------------------ */
/* Permutations — permute.py                                                 */
/* ------------------------------------------------------------------------ */

/* HOST call (no device memory, no stream): Generator(PCG64).permutation(n) of
 * numpy, bit-exact — the generation step of random_permutation (permute.py:71-81)
 * and of each part of riffle_shuffle_permutation (permute.py:150-156).
 * st[6] = {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger}, i.e.
 * numpy's PCG64.state; updated in place to the generator state after the
 * shuffle (the riffle draws two permutations from one generator).
 * h_out = int32[n] host buffer, 1 <= n <= 2^31 - 1.  Swap partners are drawn
 * ahead of the swaps and prefetched (pcg64_host.cpp). */
int sme_host_pcg64_permutation(uint64_t* st, int64_t n, int32_t* h_out);
/* HOST call: only the swap partners of that shuffle, h_j[i] = random_interval(i)
 * for i = n-1 .. 1 (h_j[0] = 0), st updated exactly as numpy's shuffle leaves it.
 * Raw outputs are generated in parallel (LCG jump-ahead per thread), the masked
 * rejection replayed sequentially and branch-free.  threads <= 0: up to 8. */
int sme_host_pcg64_swap_partners(uint64_t* st, int64_t n, uint32_t* h_j, int threads);
/* The same partners written straight to DEVICE memory d_j (int32[n]): the replay
 * fills a small pinned ring (4 x 4 MB) and each slot is copied with cudaMemcpyAsync on
 * `stream` as soon as the replay has moved below it, so the upload hides behind the
 * draws and no n-sized host buffer is touched.  HOST call; returns after the copies
 * have completed (it synchronises `stream`). */
int sme_pcg64_swap_partners_to_device(uint64_t* st, int64_t n, int32_t* d_j, int threads, sme_stream_t stream);
/* The same partners drawn on the GPU (shuffle_gen.cu): the PCG64 stream is generated in
 * parallel, every draw whose step provably lies in a narrow statistical window is
 * decided in parallel, the few others in order on the host, and a final pass checks
 * the windows and writes d_j.  n >= 2.  Returns SME_OK, or 1 if a window check failed
 * (odds ~1e-30; st untouched, replay on the host instead).  HOST call that
 * synchronises `stream`. */
int sme_pcg64_swap_partners_gpu_workspace_size(int64_t n, size_t* bytes);
/* d_ws: optional caller scratch of sme_pcg64_swap_partners_gpu_workspace_size bytes (NULL:
 * allocated stream-ordered inside). */
int sme_pcg64_swap_partners_gpu(uint64_t* st, int64_t n, int32_t* d_j, void* d_ws, size_t ws_bytes,
                                sme_stream_t stream);
/* The swaps of that shuffle on the GPU (shuffle.cu): d_perm = the permutation
 * a = arange(n); for i = n-1..1: swap(a[i], a[d_j[i]]) builds — computed as a
 * bucket sort of the steps by partner, a link pass and a chain walk (no dependent
 * swaps).  Bit-exact with numpy's Generator.permutation given the partners. */
int sme_fy_apply_workspace_size(int64_t n, size_t* bytes);
int sme_fy_apply(int64_t n, const uint32_t* d_j, int32_t* d_perm, void* d_ws, size_t ws_bytes,
                 sme_stream_t stream);

/* Permutation.inverse: inv[fwd[i]] = i.  Replaces permute.py:42-45 and the
 * bijection check of Permutation.__post_init__ (permute.py:29-36): bit
 * SME_FLAG_RANGE / SME_FLAG_NOT_BIJECTION is OR-ed into *d_flag (int32). */
int sme_perm_inverse(int64_t n, const int32_t* d_fwd, int32_t* d_inv, int32_t* d_flag,
                     sme_stream_t stream);

/* permute_vector: out[p[i]] = x[i]  (permute.py:105-112).  Bit-exact value moves. */
int sme_permute_vector(int dtype, int64_t n, const int32_t* d_p, const void* d_x, void* d_out,
                       sme_stream_t stream);

/* Gather: out[i] = x[idx[i]].  With idx = inverse(p) this equals permute_vector;
 * with int32 data it is compose(after, first) = after.forward[first.forward]
 * (permute.py:64-68) — pass dtype = -1 for int32 payloads. */
int sme_gather(int dtype, int64_t n, const int32_t* d_idx, const void* d_x, void* d_out,
               sme_stream_t stream);

/* permute_matrix on COO: (p_r[row], p_c[col], v) in ORIGINAL entry order
 * (permute.py:98-102, permute_rows/permute_cols :84-95).  Either map may be NULL
 * (identity).  Values are not touched (the caller shares or copies them). */
int sme_coo_remap(int64_t nnz, const int32_t* d_row, const int32_t* d_col, const int32_t* d_row_map,
                  const int32_t* d_col_map, int32_t* d_row_out, int32_t* d_col_out,
                  sme_stream_t stream);

/* ------------------------------------------------------------------------ */
/* CSR construction — matio.py:281-300 and permute.py:98 (fused)              */
/* ------------------------------------------------------------------------ */

/* Scratch for the two row_ptr builders (row counts + scan partials). */
int sme_row_ptr_workspace_size(int64_t n_rows, size_t* bytes);

/* Step 1 of coo_to_csr (matio.py:292-293, cumsum(bincount(row))): row counts of
 * the (optionally row-mapped) COO and their exclusive scan -> row_ptr[n_rows+1].
 * Range violations of row/col are OR-ed into *d_flag as SME_FLAG_RANGE. */
int sme_coo_row_ptr(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* d_row,
                    const int32_t* d_col, const int32_t* d_row_map, int32_t* d_row_ptr_out,
                    void* d_ws, size_t ws_bytes, int32_t* d_flag, sme_stream_t stream);

/* Step 2 of coo_to_csr (matio.py:281-294), optionally through row/col maps so
 * that coo_to_csr(permute_matrix(m, p_r, p_c)) is one pipeline: scatter into
 * the rows of d_row_ptr (from step 1), then a segmented column sort inside each
 * row; values move bit-exactly.  Duplicates are OR-ed into *d_flag; the
 * smallest duplicate (row << 32 | col) in row-major order goes to *d_dup_key
 * (uint64, caller initialises it to UINT64_MAX) — the first duplicate the
 * reference's lexsort reports (matio.py:288-291).  long_nnz = sum of the
 * lengths of rows longer than SME_SORT_SMEM_MAX (sme_long_row_nnz). */
int sme_coo_to_csr_workspace_size(int64_t n_rows, int64_t nnz, int64_t long_nnz, size_t* bytes);
int sme_coo_to_csr(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* d_row,
                   const int32_t* d_col, const void* d_val, const int32_t* d_row_map,
                   const int32_t* d_col_map, const int32_t* d_row_ptr, int32_t* d_col_out,
                   void* d_val_out, void* d_ws, size_t ws_bytes, int64_t long_nnz,
                   int32_t* d_flag, uint64_t* d_dup_key, sme_stream_t stream);

/* Permuted CSR directly from CSR (K4): new row r is old
 * row inv_r[r], columns mapped through col_map (old -> new; NULL = identity),
 * then sorted within the row; bit-identical to
 * coo_to_csr(permute_matrix(csr_to_coo(A), p_r, p_c)).  d_inv_row may be NULL
 * (identity rows). */
int sme_permute_csr_row_ptr(int64_t n_rows, const int32_t* d_row_ptr, const int32_t* d_inv_row,
                            int32_t* d_row_ptr_out, void* d_ws, size_t ws_bytes,
                            sme_stream_t stream); /* ws: sme_row_ptr_workspace_size */
/* The same row_ptr plus d_starts_out[r] = d_row_ptr[d_inv_row[r]], the source start of
 * every new row, with the old row_ptr gathered once (the scan's second pass reads the
 * lengths back sequentially).  Passing d_starts_out as sme_permute_csr's d_row_ptr with
 * d_inv_row = NULL then reads the sources in order (K4 without a second random gather).
 * ws: sme_row_ptr_workspace_size. */
int sme_permute_csr_row_ptr_starts(int64_t n_rows, const int32_t* d_row_ptr, const int32_t* d_inv_row,
                                   int32_t* d_row_ptr_out, int32_t* d_starts_out, void* d_ws, size_t ws_bytes,
                                   sme_stream_t stream);
int sme_permute_csr_workspace_size(int64_t n_rows, int64_t nnz, int64_t long_nnz, size_t* bytes);
int sme_permute_csr(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz,
                    const int32_t* d_row_ptr, const int32_t* d_col, const void* d_val,
                    const int32_t* d_inv_row, const int32_t* d_col_map,
                    const int32_t* d_row_ptr_out /* from sme_permute_csr_row_ptr */,
                    int32_t* d_col_out, void* d_val_out, void* d_ws, size_t ws_bytes,
                    int64_t long_nnz, int32_t* d_flag, uint64_t* d_dup_key, sme_stream_t stream);
/* mapped[k] = cmap[col[k]] (permute.py:98-102's column relabelling) in n_slices passes,
 * pass s relabelling slice s of the columns while that slice of cmap stays L2-resident
 * (the first pass reads col and writes mapped, the others rewrite mapped in place,
 * whole 16-byte vectors; an access-policy window pins the slice when the caller
 * reserved persisting L2).  col and mapped 16-byte aligned, n_cols < 2^31. */
int sme_map_cols_sliced(int64_t nnz, int64_t n_cols, const int32_t* d_col, const int32_t* d_cmap,
                        int32_t* d_mapped, int32_t n_slices, sme_stream_t stream);
/* The first n_passes (1..n_slices) of those passes: relabelled entries carry bit 31, the
 * others keep their old id.  The K4 pre-pass when cmap exceeds L2: sme_permute_csr, given
 * col = mapped and the same cmap, maps the unflagged entries (the last slice, L2-resident
 * by then) and clears the flags inside its row sort. */
int sme_map_cols_sliced_partial(int64_t nnz, int64_t n_cols, const int32_t* d_col, const int32_t* d_cmap,
                                int32_t* d_mapped, int32_t n_slices, int32_t n_passes, sme_stream_t stream);

/* Rows longer than this are sorted through global scratch (long-row path). */
#define SME_SORT_SMEM_MAX 4096
/* Sum of the lengths of rows longer than SME_SORT_SMEM_MAX -> *d_out (int64). */
int sme_long_row_nnz(int64_t n_rows, const int32_t* d_row_ptr, int64_t* d_out, sme_stream_t stream);

/* Dedupe variant of sme_coo_to_csr (no maps): duplicate (row, col) pairs stay as
 * col = -1 holes instead of an error; sme_csr_compact then removes the holes and
 * keeps at most `cap` entries per row (the smallest columns).  Used to build
 * graphs from generated edge lists (C3 R-MAT: dedupe + degree cap). */
int sme_coo_to_csr_dedup(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* d_row,
                         const int32_t* d_col, const void* d_val, const int32_t* d_row_ptr,
                         int32_t* d_col_out, void* d_val_out, void* d_ws, size_t ws_bytes, int64_t long_nnz,
                         int32_t* d_flag, sme_stream_t stream);
int sme_csr_compact_row_ptr(int64_t n_rows, const int32_t* d_row_ptr, const int32_t* d_col, int32_t cap,
                            int32_t* d_out_row_ptr, void* d_ws, size_t ws_bytes, sme_stream_t stream);
int sme_csr_compact(int dtype, int64_t n_rows, const int32_t* d_row_ptr, const int32_t* d_col, const void* d_val,
                    int32_t cap, const int32_t* d_out_row_ptr, int32_t* d_out_col, void* d_out_val,
                    sme_stream_t stream);

/* Column span col[last] - col[first] of n_samples evenly spaced rows (row i*(n_rows-1)/(n_samples-1)),
 * -1 for rows with fewer than 2 entries: the banded-structure probe of the kernel policy. */
int sme_row_spans(int64_t n_rows, const int32_t* d_row_ptr, const int32_t* d_col, int32_t n_samples,
                  int32_t* d_out, sme_stream_t stream);
/* Row-length statistics for kernel selection: out[0] = max row length, out[1] = empty rows. */
int sme_row_stats(int64_t n_rows, const int32_t* d_row_ptr, int64_t* d_out, sme_stream_t stream);

/* CsrMatrix.__post_init__ checks (matio.py:105-122) on device: OR-s
 * SME_FLAG_ROWPTR / SME_FLAG_RANGE / SME_FLAG_UNSORTED into *d_flag. */
int sme_csr_validate(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* d_row_ptr,
                     const int32_t* d_col, int32_t* d_flag, sme_stream_t stream);

/* csr_to_coo row expansion (matio.py:297-300): row_idx[k] = row of entry k. */
int sme_csr_expand_rows(int64_t n_rows, const int32_t* d_row_ptr, int32_t* d_row_out,
                        sme_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Entropy histogram — entropy.py                                            */
/* ------------------------------------------------------------------------ */

/* histogram_2d (entropy.py:91-101) from CSR: counts[br*bc] (int64, row-major),
 * bins per _bin_index (entropy.py:65-67): width = n // bins, last bin absorbs
 * the remainder.  ACCUMULATES into d_counts (caller zeroes it). */
int sme_hist2d_csr(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* d_row_ptr,
                   const int32_t* d_col, int32_t bins_r, int32_t bins_c, int64_t* d_counts,
                   sme_stream_t stream);
/* Same from COO triplets in any order (the reference's own input type). */
/* Kernel selection of sme_hist2d_csr (process-wide; tests and experiments):
 * 0 = lane-private u16 counters when bins_c <= 128 (default), 1 = the
 * shared-memory window with warp-aggregated atomics, 2 = lane counters on one CTA. */
int sme_hist2d_set_mode(int mode);
/* Row-sort keys of the CSR builds (process-wide; tests): 1 = 32-bit (mapped col << 5 |
 * slot) whenever n_cols <= 2^27 (default), 0 = always 64-bit (col << 32 | slot). */
int sme_sort_rows_set_key32(int enable);
/* Test hook: 1 (default) sorts rows of 257..SME_SORT_SMEM_MAX entries with the CTA-wide
 * register / shuffle / shared-memory bitonic network; 0 = all in shared memory. */
int sme_sort_rows_set_cta(int enable);
/* Rows with 32 < len <= 512 of the CSR builds (process-wide; tests): 1 = one warp per
 * row, keys in registers (default), 0 = one CTA per row, bitonic in shared memory. */
int sme_sort_rows_set_wmed(int enable);
/* Tiling of the lane-counter kernel (experiments): 0 = 864 threads x 4 int4 loads per
 * lane (default; 768 x 4 when bins_r > ~1500), 1 = 768 x 4, 2 = 512 x 4 + next-iteration
 * prefetch, 3 = 768 x 2 + prefetch, 4 = 640 x 4 + prefetch, 5 = 864 x 4, 6 = 864 x 2,
 * 7 = 512 x 8. */
int sme_hist2d_set_variant(int variant);
int sme_hist2d_coo(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* d_row,
                   const int32_t* d_col, int32_t bins_r, int32_t bins_c, int64_t* d_counts,
                   sme_stream_t stream);
/* row_histogram from CSR (entropy.py:77-81): counts[b] = row_ptr[e_{b+1}] - row_ptr[e_b]. */
int sme_row_hist_csr(int64_t n_rows, const int32_t* d_row_ptr, int32_t bins, int64_t* d_counts,
                     sme_stream_t stream);

/* shannon_entropy / _entropy_of_counts (entropy.py:104-119):
 * -sum_{c>0} p log_base p, p = c / total, one deterministic block reduction.
 * *d_out (double) receives the entropy; *d_total (int64, may be NULL) the total. */
int sme_entropy(int64_t n_bins, const int64_t* d_counts, double base, double* d_out,
                int64_t* d_total, sme_stream_t stream);

/* ------------------------------------------------------------------------ */
/* SpMV — kernels.py                                                        */
/* ------------------------------------------------------------------------ */

/* Merge-path (nnz+row balanced) CSR SpMV, the drop-in for spmv_csr
 * (kernels.py:59-78).  A per-matrix plan (tile coordinates on the merge path
 * of row ends and nonzeros) is built once and reused across calls:
 *   plan: (n_tiles + 1) int2 = (row, nnz) split points; carry: n_tiles x
 *   (int32 row + value) scratch.
 * accumulate = 0: y = A x;  accumulate = 1: y += A x (column-panel passes). */
int sme_spmv_merge_tiles(int64_t n_rows, int64_t nnz, int64_t* n_tiles);
int sme_spmv_merge_plan(int64_t n_rows, int64_t nnz, const int32_t* d_row_ptr, int32_t* d_plan,
                        sme_stream_t stream);
int sme_spmv_merge_carry_bytes(int dtype, int64_t n_tiles, size_t* bytes);
int sme_spmv_merge(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz,
                   const int32_t* d_row_ptr, const int32_t* d_col, const void* d_val,
                   const void* d_x, void* d_y, const int32_t* d_plan, int64_t n_tiles,
                   void* d_carry, int accumulate, sme_stream_t stream);

/* Warp-streaming CSR SpMV (the fast path for regular and moderately ragged rows):
 * every resident warp of a persistent grid owns a contiguous row range holding
 * ~nnz/W nonzeros (per-matrix plan, W from sme_spmv_stream_warps), streams it in
 * 128-element chunks aligned to GLOBAL positions (align_off in [0,128) = global
 * position of local element 0 mod 128, so row shards reduce exactly like the
 * whole matrix) and reduces rows with a flag-segmented warp scan.  No fix-up
 * pass.  plan: (W + 1) int32.  accumulate = 1: y += A x. */
int sme_spmv_stream_warps(int64_t n_rows, int64_t nnz, int32_t* n_warps);
/* Chunk-stream source: 0 = 128-bit register loads one chunk ahead (default),
 * 1 = per-lane cp.async (LDGSTS) shared-memory ring, 3 chunks ahead. */
int sme_spmv_stream_set_mode(int mode);
/* Plan weight of a row in nonzero units (default 2): warp ranges balance nnz + cost * rows. */
int sme_spmv_stream_set_row_cost(int cost);
int sme_spmv_stream_plan(int64_t n_rows, int64_t nnz, const int32_t* d_row_ptr, int32_t n_warps,
                         int32_t* d_plan, sme_stream_t stream);
int sme_spmv_stream(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* d_row_ptr,
                    const int32_t* d_col, const void* d_val, const void* d_x, void* d_y,
                    const int32_t* d_plan, int32_t n_warps, int accumulate, int32_t align_off,
                    sme_stream_t stream);

/* Column panels (x-locality layout, panel.cu): split a column-sorted CSR into
 * n_panels CSRs by column ranges [bounds[p], bounds[p+1]) so that the SpMV can
 * run one accumulating pass per panel with that panel's x slice L2-resident.
 * Step 1 writes panel_ptr (n_panels x (n_rows+1), relative row pointers);
 * step 2 scatters entries to out_col/out_val at offsets[p] (int64 device,
 * multiples of 128 elements).  Columns stay global and ascending per row. */
int sme_panel_count_workspace_size(int64_t n_rows, int32_t n_panels, size_t* bytes);
int sme_panel_row_ptrs(int64_t n_rows, const int32_t* d_row_ptr, const int32_t* d_col, int32_t n_panels,
                       const int32_t* d_bounds, int32_t* d_panel_ptr, void* d_ws, size_t ws_bytes,
                       sme_stream_t stream);
int sme_panel_scatter(int dtype, int64_t n_rows, const int32_t* d_row_ptr, const int32_t* d_col,
                      const void* d_val, int32_t n_panels, const int32_t* d_bounds,
                      const int32_t* d_panel_ptr, const int64_t* d_offsets, int32_t* d_out_col,
                      void* d_out_val, sme_stream_t stream);

/* Segmented-chunk layout (spmv_seg.cu): the fast path for randomly permuted
 * matrices.  Per column panel p, entries keep CSR order in 32-bit words
 * (col - bounds[p]) << 9 | end_of_row << 8 | (row - hdr[chunk]) with a row
 * header per 128-entry chunk, so no row_ptr is streamed; a warp sums the rows
 * of a chunk from the end flags (in-lane runs + one shuffle per lane).  Replaces spmv_csr / _accumulate_rows (kernels.py:59-78)
 * on the column-panel passes (y = A_0 x_0; y += A_p x_p).
 * Build: sme_seg_positions (padded per-panel entry positions, n_panels x
 * (n_rows+1) int32; ws sized by sme_seg_workspace_size keeps row counts),
 * sme_seg_fill (pk/val/hdr at the 128-aligned panel offsets; offsets given on
 * device and host), sme_seg_plan (per panel: n_warps+1 entry positions on row
 * boundaries, n_warps from sme_spmv_seg_warps).  Panel width < 2^23 - 1.
 * full_last = 1 also gives every row without entries in the LAST panel an
 * explicit zero there (needed by the fused epilogue of sme_spmv_seg_epi). */
int sme_seg_workspace_size(int64_t n_rows, int32_t n_panels, size_t* bytes);
int sme_seg_positions(int64_t n_rows, const int32_t* d_row_ptr, const int32_t* d_col, int32_t n_panels,
                      const int32_t* d_bounds, int full_last, int32_t* d_pos, void* d_ws, size_t ws_bytes,
                      sme_stream_t stream);
int sme_seg_fill(int dtype, int64_t n_rows, const int32_t* d_row_ptr, const int32_t* d_col,
                 const void* d_val, int32_t n_panels, const int32_t* d_bounds, const int32_t* d_pos,
                 const int64_t* d_offsets, const int64_t* h_offsets, uint32_t* d_pk, void* d_out_val,
                 int32_t* d_hdr, const void* d_ws, sme_stream_t stream);
/* Test hook: 1 (default) fills the layout with a warp per 32-row group through a
 * shared-memory image of the group's panel ranges (coalesced writes); 0 = warp per row. */
int sme_seg_set_scatter_groups(int on);
/* Test hook: 1 (default) places the entries of groups without empty rows entry-parallel
 * (row from a mask of the row starts in each 32-entry window); 0 = the per-row walk. */
int sme_seg_set_fill_ballot(int on);
/* Test hook: 1 (default) the grouped fill stores every entry straight to its slot; 0 =
 * through the shared-memory image of the group's panel ranges (same layout bits). */
int sme_seg_set_fill_direct(int on);
int sme_spmv_seg_warps(int32_t* n_warps);
/* Kernel variant (process-wide): 0 = the SpMV (default; accumulating passes add
 * with RED.ADD at L2), 3 = bound probe (the chunk stream and gathers without the
 * row reduction; timing only, not y = A x), 5 = accumulating passes load y, add,
 * store (same bits, 3-4 % slower on C4). */
int sme_spmv_seg_set_mode(int mode);
int sme_seg_plan(int64_t n_rows, const int32_t* d_pos_panel, int32_t n_warps, int32_t* d_plan,
                 sme_stream_t stream);
/* Split-row plan (power-law rows): plan[w] = w * total / n_warps, ranges may start and
 * end mid-row; passes over it use sme_spmv_seg_split. */
int sme_seg_plan_split(int64_t total_entries, int32_t n_warps, int32_t* d_plan, sme_stream_t stream);
/* One pass over a split-row plan: the pass, then the open row partials at the range ends
 * (d_carry_val[n_warps] of the value type, d_carry_row[n_warps] int32 scratch) added to
 * their rows in warp order (deterministic). */
int sme_spmv_seg_split(int dtype, int32_t n_warps, const uint32_t* d_pk, const void* d_val, const int32_t* d_hdr,
                       const int32_t* d_plan, const void* d_xs, void* d_y, int accumulate, void* d_carry_val,
                       int32_t* d_carry_row, sme_stream_t stream);
/* y (+)= A_p x_p for one panel: d_xs = x + bounds[p]; accumulate = 0 for panel 0. */
int sme_spmv_seg(int dtype, int32_t n_warps, const uint32_t* d_pk, const void* d_val, const int32_t* d_hdr,
                 const int32_t* d_plan, const void* d_xs, void* d_y, int accumulate, sme_stream_t stream);
/* The last pass of one power-iteration step with its BLAS-1 work fused in (f64):
 * v_r = scale[0] * (y[r] (+ this panel's row sum)), written to d_out[qinv[r]]
 * (qinv NULL: d_out[r]) — the permuted-coordinate gather z = (B z)[q] of
 * iterative.py becomes this scatter — while the sum of v_r^2 is reduced
 * deterministically (warp partials in d_partials[n_warps], last CTA in fixed
 * order; d_ticket: one uint32, zero-initialised once) into d_result[1], and
 * d_result[0] = 1/sqrt(d_result[1]) is the next step's scale.  Replaces the
 * numpy loop x = A x / ||A x|| over spmv_csr (kernels.py:73-78) of the C5
 * oracle.  Needs a layout built with full_last = 1. */
int sme_spmv_seg_epi(int dtype, int32_t n_warps, const uint32_t* d_pk, const void* d_val, const int32_t* d_hdr,
                     const int32_t* d_plan, const void* d_xs, void* d_y, int accumulate, void* d_out,
                     const int32_t* d_qinv, const double* d_scale, double* d_partials, uint32_t* d_ticket,
                     double* d_result, sme_stream_t stream);
/* The same epilogue for one row shard of a multi-GPU power iteration (rowshard.py):
 * v is stored at global index row_offset + r of d_out (this rank's full-length
 * next iterate) and of every buffer in d_peers[n_peers] (the other ranks' next
 * iterates, opened with sme_ipc_open — stores over NVLink): the all-gather of the
 * iterate (ncclAllGather in the unfused path) rides in the SpMV
 * epilogue.  d_result[1] = this shard's sum of v^2 (the caller all-reduces it). */
int sme_spmv_seg_epi_peers(int dtype, int32_t n_warps, const uint32_t* d_pk, const void* d_val,
                           const int32_t* d_hdr, const int32_t* d_plan, const void* d_xs, void* d_y,
                           int accumulate, void* d_out, int64_t row_offset, void* const* d_peers, int32_t n_peers,
                           const double* d_scale, double* d_partials, uint32_t* d_ticket, double* d_result,
                           sme_stream_t stream);

/* The last pass of one CG step (iterative.py) with p.Ap fused in: d_out[r] = (A p)[r],
 * sum d_out[r] * d_p[r] reduced deterministically, and the last CTA writes
 * alpha = d_scal[0] / (p.Ap) into d_scal[1] (d_scal[0] = r.r, blas1.cu's CG
 * scalars) — replaces sme_dot(p, Ap) after the SpMV.  d_xs = d_p + bounds of the
 * last panel; needs a layout built with full_last = 1. */
int sme_spmv_seg_epi_cg(int dtype, int32_t n_warps, const uint32_t* d_pk, const void* d_val, const int32_t* d_hdr,
                        const int32_t* d_plan, const void* d_xs, const void* d_p, void* d_y, int accumulate,
                        void* d_out, double* d_partials, uint32_t* d_ticket, double* d_scal, sme_stream_t stream);

/* The CSR-vector twin of the fused iteration epilogue (banded / unpermuted operators):
 * d_out = scale[0] * (A x) (scale NULL: 1) with sum d_out * (d_dotv ? d_dotv : d_out)
 * reduced deterministically over a fixed grid of sme_spmv_vector_epi_blocks() blocks
 * (d_partials holds one double per block; d_ticket one uint32, zero-initialised once);
 * finish 0: d_result = {1/sqrt(sum), sum} (power iteration), finish 1: d_result[1] =
 * d_result[0] / sum (CG alpha).  f64.  Replaces spmv_csr + the oracle loop's norm / dot
 * (kernels.py:73-78). */
int sme_spmv_vector_epi_blocks(int64_t n_rows, int lanes, int64_t* blocks);
int sme_spmv_vector_epi(int lanes, int64_t n_rows, const int32_t* d_row_ptr, const int32_t* d_col,
                        const double* d_val, const double* d_x, double* d_out, const double* d_scale,
                        const double* d_dotv, double* d_partials, uint32_t* d_ticket, double* d_result,
                        int finish, sme_stream_t stream);

/* The epilogue alone (split-row seg layouts, whose passes end mid-row): d_out[qinv[r]] =
 * scale[0] * d_y[r] with the same deterministic reduction and d_result semantics as
 * sme_spmv_vector_epi; d_partials holds sme_rows_epi_blocks() doubles. */
int sme_rows_epi_blocks(int64_t n_rows, int64_t* blocks);
int sme_rows_epi(int64_t n_rows, const double* d_y, double* d_out, const int32_t* d_qinv, const double* d_scale,
                 const double* d_dotv, double* d_partials, uint32_t* d_ticket, double* d_result, int finish,
                 sme_stream_t stream);

/* CUDA IPC buffers for the fused exchange (ipc.cu): whole cudaMalloc allocations
 * whose handles (SME_IPC_HANDLE_BYTES bytes) are exchanged between the ranks of a
 * node (torch.distributed all_gather_object) and opened by the peers. */
#define SME_IPC_HANDLE_BYTES 64
int sme_ipc_malloc(size_t bytes, void** d_ptr);
int sme_ipc_free(void* d_ptr);
int sme_ipc_get_handle(void* d_ptr, uint8_t* handle);
int sme_ipc_open(const uint8_t* handle, void** d_ptr);
int sme_ipc_close(void* d_ptr);

/* Merge kernel selection (process-wide; tests and experiments): 1 = persistent
 * TMA-pipelined kernel (needs 16-byte aligned row_ptr/col_idx/values), 0 = one
 * CTA per tile with plain global loads, -1 = auto (TMA when aligned). */
int sme_spmv_merge_set_mode(int mode);

/* CSR-vector ("warp-per-row") SpMV: `lanes` in {1,2,4,8,16,32} threads per row,
 * lane-strided partial sums combined by a butterfly shuffle.  The per-row
 * reduction order depends only on `lanes`, so any row partition
 * (spmv_csr_parallel, kernels.py:102-128; multi-GPU row shards) is bitwise
 * equal to the unpartitioned call. */
int sme_spmv_vector(int dtype, int lanes, int64_t n_rows, int64_t n_cols,
                    const int32_t* d_row_ptr, const int32_t* d_col, const void* d_val,
                    const void* d_x, void* d_y, int accumulate, sme_stream_t stream);

/* Bit-exact restatement of the reference reduction on the GPU: y_i =
 * prod[s] + numpy_pairwise_sum(prod[s+1:e]) with separately rounded multiplies
 * and adds (kernels.py:59-70; numpy's add.reduceat order, SURVEY.md App. A
 * item 1).  f64 only.  Slow (thread per row); parity tool. */
int sme_spmv_reduceat_exact(int64_t n_rows, const int32_t* d_row_ptr, const int32_t* d_col,
                            const double* d_val, const double* d_x, double* d_y,
                            sme_stream_t stream);

/* COO SpMV (spmv_coo, kernels.py:81-86): y = 0; y[row[k]] += v[k] * x[col[k]].
 * Fixed-point-free floating atomics: order-dependent in the last ulps. */
int sme_spmv_coo(int dtype, int64_t n_rows, int64_t nnz, const int32_t* d_row, const int32_t* d_col,
                 const void* d_val, const void* d_x, void* d_y, sme_stream_t stream);

/* Deterministic COO SpMV, bitwise equal to the reference's np.add.at (kernels.py:81-86:
 * y = 0, then y[row[k]] += v[k] * x[col[k]] in stored entry order).  Plan: d_row_ptr
 * (n_rows + 1) and d_order[p] = the entry ids of each row in ascending entry order,
 * d_val[p] = values[d_order[p]] (built once by sme_coo_to_csr with entry ids as the
 * sort key).  One thread per row sums its products in that order with round-to-
 * nearest multiply and add (no FMA), starting from 0. */
int sme_spmv_coo_ordered(int dtype, int64_t n_rows, const int32_t* d_row_ptr, const int32_t* d_order,
                         const void* d_val, const int32_t* d_col, const void* d_x, void* d_y,
                         sme_stream_t stream);

/* relative_error (kernels.py:131-142) helper: d_out[0] = max|got - exp|,
 * d_out[1] = max|exp| (f64, caller zeroes). */
int sme_maxabs_diff(int dtype, int64_t n, const void* d_got, const void* d_exp, double* d_out,
                    sme_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Iterative drivers (C5: power iteration / CG on the permuted matrix)       */
/* ------------------------------------------------------------------------ */

/* Deterministic BLAS-1 with device-resident scalars (graph-capturable).
 * scal = [rr, alpha, beta, inv_norm] (4 doubles, device); partial: sme_blas_partials doubles.
 * sme_dot mode: 0 plain, 1 alpha = scal[0]/dot, 2 beta = dot/scal[0] & scal[0] = dot,
 * 3 scal[3] = 1/sqrt(dot).  sme_cg_update: x += a p; r -= a Ap; rr' = r.r; b = rr'/rr; p = r + b p. */
int sme_blas_partials(int64_t* n_partials);
int sme_dot(int dtype, int64_t n, const void* d_x, const void* d_y, double* d_partial, double* d_out,
            double* d_scal, int mode, sme_stream_t stream);
int sme_cg_update(int dtype, int64_t n, void* d_x, void* d_r, void* d_p, const void* d_ap, double* d_scal,
                  double* d_partial, sme_stream_t stream);
int sme_scale(int dtype, int64_t n, void* d_y, const void* d_x, const double* d_scal, int idx,
              sme_stream_t stream);
int sme_axpby(int dtype, int64_t n, double a, const void* d_x, double b, void* d_y, sme_stream_t stream);

/* ------------------------------------------------------------------------ */
/* Row sharding (multi-GPU) — kernels.py:38-49 make_row_partition           */
/* ------------------------------------------------------------------------ */

/* Column ids -> positions in the padded all-gathered x of `parts` equal slots of
 * `pad` entries: rank k owns the make_row_partition range [b_k, b_{k+1}) and its
 * slice lands at k * pad.  col_out may alias col_in. */
int sme_rowshard_remap_cols(int64_t nnz, int64_t n_cols, int32_t parts, int64_t pad,
                            const int32_t* d_col_in, int32_t* d_col_out, sme_stream_t stream);

/* 64-bit content hash of a device array (the key of the on-disk permuted-CSR cache,
 * cache.py; the reference persists permuted matrices through cmd_permute ->
 * write_matrix_market, cli.py:173-230, matio.py:262-278).  Over the 32-bit words w_i:
 * *d_out = sum_i mix64((mix64(seed ^ C) + i * G) ^ (w_i * K)) mod 2^64 — deterministic
 * for any launch shape.  n_bytes % 4 == 0, d_data 4-byte aligned. */
int sme_hash64(const void* d_data, int64_t n_bytes, uint64_t seed, uint64_t* d_out, sme_stream_t stream);

/* Load every kernel module of libsme.so now (CUDA lazy loading would load each on the
 * first launch of one of its kernels, ~10-20 ms apiece, inside the first permuted-matrix
 * setup of a process).  Call once after the context exists; idempotent. */
int sme_preload(void);

/* ------------------------------------------------------------------------ */
/* int64 row_ptr ("wide" CSR): matrices with nnz >= 2^31 - 1                 */
/* ------------------------------------------------------------------------ */
/* The reference stores row_ptr as int64 at every size (matio.py:97-99); the GPU
 * layout keeps int32 row_ptr while nnz < 2^31 - 1 and switches to int64 above
 * (SURVEY.md §7, §8(d) s_p = 8): a 180 GB B200 holds f64 CSRs of ~10^10 nonzeros.
 * Column ids stay int32 (n_cols < 2^31), and so do the per-panel slot positions of
 * the seg layout (each panel < 2^31 slots: the caller picks enough panels).  Each
 * entry point below is its int32 namesake with int64 row_ptr arguments and no
 * nnz < 2^31 limit; semantics, flags and errors are identical. */
int sme_coo_row_ptr_i64(int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* d_row,
                        const int32_t* d_col, const int32_t* d_row_map, int64_t* d_row_ptr_out,
                        void* d_ws, size_t ws_bytes, int32_t* d_flag, sme_stream_t stream);
int sme_coo_to_csr_i64(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz, const int32_t* d_row,
                       const int32_t* d_col, const void* d_val, const int32_t* d_row_map,
                       const int32_t* d_col_map, const int64_t* d_row_ptr, int32_t* d_col_out,
                       void* d_val_out, void* d_ws, size_t ws_bytes, int64_t long_nnz,
                       int32_t* d_flag, uint64_t* d_dup_key, sme_stream_t stream);
int sme_permute_csr_row_ptr_i64(int64_t n_rows, const int64_t* d_row_ptr, const int32_t* d_inv_row,
                                int64_t* d_row_ptr_out, void* d_ws, size_t ws_bytes, sme_stream_t stream);
int sme_permute_csr_i64(int dtype, int64_t n_rows, int64_t n_cols, int64_t nnz,
                        const int64_t* d_row_ptr, const int32_t* d_col, const void* d_val,
                        const int32_t* d_inv_row, const int32_t* d_col_map, const int64_t* d_row_ptr_out,
                        int32_t* d_col_out, void* d_val_out, void* d_ws, size_t ws_bytes,
                        int64_t long_nnz, int32_t* d_flag, uint64_t* d_dup_key, sme_stream_t stream);
int sme_permute_csr_row_ptr_starts_i64(int64_t n_rows, const int64_t* d_row_ptr, const int32_t* d_inv_row,
                                       int64_t* d_row_ptr_out, int64_t* d_starts_out, void* d_ws, size_t ws_bytes,
                                       sme_stream_t stream);
int sme_long_row_nnz_i64(int64_t n_rows, const int64_t* d_row_ptr, int64_t* d_out, sme_stream_t stream);
int sme_row_stats_i64(int64_t n_rows, const int64_t* d_row_ptr, int64_t* d_out, sme_stream_t stream);
int sme_row_spans_i64(int64_t n_rows, const int64_t* d_row_ptr, const int32_t* d_col, int32_t n_samples,
                      int32_t* d_out, sme_stream_t stream);
int sme_csr_validate_i64(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* d_row_ptr,
                         const int32_t* d_col, int32_t* d_flag, sme_stream_t stream);
int sme_csr_expand_rows_i64(int64_t n_rows, const int64_t* d_row_ptr, int32_t* d_row_out,
                            sme_stream_t stream);
int sme_hist2d_csr_i64(int64_t n_rows, int64_t n_cols, int64_t nnz, const int64_t* d_row_ptr,
                       const int32_t* d_col, int32_t bins_r, int32_t bins_c, int64_t* d_counts,
                       sme_stream_t stream);
int sme_row_hist_csr_i64(int64_t n_rows, const int64_t* d_row_ptr, int32_t bins, int64_t* d_counts,
                         sme_stream_t stream);
int sme_seg_positions_i64(int64_t n_rows, const int64_t* d_row_ptr, const int32_t* d_col, int32_t n_panels,
                          const int32_t* d_bounds, int full_last, int32_t* d_pos, void* d_ws, size_t ws_bytes,
                          sme_stream_t stream);
int sme_seg_fill_i64(int dtype, int64_t n_rows, const int64_t* d_row_ptr, const int32_t* d_col,
                     const void* d_val, int32_t n_panels, const int32_t* d_bounds, const int32_t* d_pos,
                     const int64_t* d_offsets, const int64_t* h_offsets, uint32_t* d_pk, void* d_out_val,
                     int32_t* d_hdr, const void* d_ws, sme_stream_t stream);
int sme_spmv_vector_i64(int dtype, int lanes, int64_t n_rows, int64_t n_cols, const int64_t* d_row_ptr,
                        const int32_t* d_col, const void* d_val, const void* d_x, void* d_y, int accumulate,
                        sme_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif /* SME_H */
