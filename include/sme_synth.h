/*
 * sme_synth.h — device generators for the synthetic matrices of BASELINE.json
 * (SURVEY.md §8d).  Benchmark/test inputs only; not part of the reference path.
 * Bit-identical numpy restatements live in paper_2308_00106_b200/synth.py.
 */
#ifndef SME_SYNTH_H
#define SME_SYNTH_H
#include "sme.h"
#ifdef __cplusplus
extern "C" {
#endif

/* 5-point Laplacian on a g x g grid (C2: g = 2000, C5: g = 2828): row r = i*g + j
 * holds r-g, r-1, r, r+1, r+g (those inside the grid), values -1, -1, 4, -1, -1.
 * row_ptr: g*g + 1 int32; col/val: 5g^2 - 4g entries. */
int sme_synth_laplacian5(int dtype, int64_t g, int32_t* d_row_ptr, int32_t* d_col, void* d_val,
                         sme_stream_t stream);

/* Random-structured rows (C4): every row has k (<= 32) distinct columns, the first
 * k distinct draws of hash3(seed, r, t) mapped to [0, n_cols), sorted ascending;
 * value of sorted slot s = U[-1,1) from hash3(seed ^ 0x5DEECE66D, r, s).
 * d_row_ptr may be NULL (it is r * k; required for nnz >= 2^31, int64 row_ptr). */
int sme_synth_random_rows(int dtype, int64_t n_rows, int64_t n_cols, int32_t k, uint64_t seed,
                          int32_t* d_row_ptr, int32_t* d_col, void* d_val, sme_stream_t stream);

/* The same generator for selected rows: output row i is generator row d_rows[i]
 * (row_ptr[i] = i*k).  A row shard of the permuted C4 generates only the original
 * rows inverse(p_r)[lo:hi] it owns (bench.py multi-GPU setup). */
int sme_synth_random_rows_sel(int dtype, int64_t n_sel, const int32_t* d_rows, int64_t n_cols, int32_t k,
                              uint64_t seed, int32_t* d_row_ptr, int32_t* d_col, void* d_val,
                              sme_stream_t stream);

/* R-MAT edges (C3): edge e, level l: u = U[0,1)(hash3(seed, e, l)); quadrant (0,0) if
 * u < a, (0,1) if u < a+b, (1,0) if u < a+b+c, else (1,1); bits appended MSB first.
 * Dedupe/cap through sme_coo_to_csr_dedup + sme_csr_compact; values per (row, slot)
 * by sme_synth_row_values: U[-1,1)(hash3(seed ^ 0x5DEECE66D, row, slot)). */
int sme_synth_rmat_edges(int64_t n_edges, int32_t scale, double a, double b, double c, uint64_t seed,
                         int32_t* d_row, int32_t* d_col, sme_stream_t stream);
int sme_synth_row_values(int dtype, int64_t n_rows, const int32_t* d_row_ptr, uint64_t seed, void* d_val,
                         sme_stream_t stream);

/* Diagnostic (roofline) microbenchmark: blocks x 256 threads each gather
 * per_thread (multiple of 8) hash-random elements of x[n] (keep = L2 evict-last)
 * and write one sum to out[thread]. */
int sme_diag_gather(const double* d_x, int64_t n, int32_t blocks, int32_t per_thread, int32_t keep,
                    double* d_out, sme_stream_t stream);

#ifdef __cplusplus
}
#endif
#endif
