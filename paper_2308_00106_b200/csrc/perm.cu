// perm.cu — permutation kernels (permute.py:23-112 of the reference).
//
// All of these are HBM-bound index moves: one coalesced stream plus one random
// stream (the scatter/gather side).  Grids are grid-stride loops sized to a
// multiple of the SM count.
#include "common.cuh"

namespace sme {

// inv[fwd[i]] = i, with range check (Permutation.__post_init__, permute.py:29-36)
__global__ void k_inverse_scatter(int64_t n, const int32_t* __restrict__ fwd,
                                  int32_t* __restrict__ inv, int32_t* __restrict__ flag) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    int32_t f = fwd[i];
    if (f < 0 || (int64_t)f >= n) {
      atomicOr(flag, SME_FLAG_RANGE | SME_FLAG_NOT_BIJECTION);
      continue;
    }
    inv[f] = (int32_t)i;
  }
}

// every slot written exactly once <=> bijection (n writes into n slots, all in range)
__global__ void k_inverse_verify(int64_t n, const int32_t* __restrict__ fwd,
                                 const int32_t* __restrict__ inv, int32_t* __restrict__ flag) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  bool bad = false;
  for (int64_t j = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; j < n; j += stride) {
    int32_t i = inv[j];
    if (i < 0 || (int64_t)i >= n || fwd[i] != (int32_t)j) bad = true;
  }
  if (__any_sync(0xffffffffu, bad) && lane_id() == 0) atomicOr(flag, SME_FLAG_NOT_BIJECTION);
}

template <typename T>
__global__ void k_scatter(int64_t n, const int32_t* __restrict__ p, const T* __restrict__ x,
                          T* __restrict__ out) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[p[i]] = x[i];
}

template <typename T>
__global__ void k_gather(int64_t n, const int32_t* __restrict__ idx, const T* __restrict__ x,
                         T* __restrict__ out) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    out[i] = x[idx[i]];
}

__global__ void k_coo_remap(int64_t nnz, const int32_t* __restrict__ row,
                            const int32_t* __restrict__ col, const int32_t* __restrict__ rmap,
                            const int32_t* __restrict__ cmap, int32_t* __restrict__ row_out,
                            int32_t* __restrict__ col_out) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
    if (row_out) row_out[k] = rmap ? rmap[row[k]] : row[k];
    if (col_out) col_out[k] = cmap ? cmap[col[k]] : col[k];
  }
}

// make_row_partition (kernels.py:38-49): first `extra` parts have base+1 entries.
__global__ void k_rowshard_remap(int64_t nnz, int64_t base, int64_t extra, int64_t pad,
                                 const int32_t* __restrict__ cin, int32_t* __restrict__ cout) {
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  int64_t big = extra * (base + 1);
  for (int64_t k = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; k < nnz; k += stride) {
    int64_t j = cin[k];
    int64_t part, off;
    if (j < big) {
      part = j / (base + 1);
      off = j - part * (base + 1);
    } else {
      part = extra + (j - big) / base;
      off = (j - big) - (part - extra) * base;
    }
    cout[k] = (int32_t)(part * pad + off);
  }
}

template <typename T>
__global__ void k_maxabs_diff(int64_t n, const T* __restrict__ got, const T* __restrict__ exp,
                              double* __restrict__ out) {
  double md = 0.0, me = 0.0;
  int64_t stride = (int64_t)gridDim.x * blockDim.x;
  for (int64_t i = (int64_t)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    double g = (double)got[i], e = (double)exp[i];
    double d = fabs(g - e), a = fabs(e);
    // NaN-propagating max, like np.max in relative_error (kernels.py:136-137)
    md = (d > md || d != d) ? d : md;
    me = (a > me || a != a) ? a : me;
  }
  for (int o = 16; o; o >>= 1) {
    double od = __shfl_xor_sync(0xffffffffu, md, o), oe = __shfl_xor_sync(0xffffffffu, me, o);
    md = (od > md || od != od) ? od : md;
    me = (oe > me || oe != oe) ? oe : me;
  }
  if (lane_id() == 0) {
    // non-negative doubles (and +NaN above +inf) order like their bit patterns
    atomicMax(reinterpret_cast<unsigned long long*>(out), (unsigned long long)__double_as_longlong(md));
    atomicMax(reinterpret_cast<unsigned long long*>(out + 1), (unsigned long long)__double_as_longlong(me));
  }
}

}  // namespace sme

using namespace sme;

SME_API int sme_perm_inverse(int64_t n, const int32_t* fwd, int32_t* inv, int32_t* flag,
                             sme_stream_t stream) {
  SME_REQUIRE(n >= 1 && n < INT32_MAX, "permutation size %lld out of range", (long long)n);
  SME_REQUIRE(fwd && inv && flag, "null pointer");
  cudaStream_t s = as_stream(stream);
  SME_CUDA(cudaMemsetAsync(inv, 0xff, (size_t)n * sizeof(int32_t), s));
  k_inverse_scatter<<<grid_for(n, 256), 256, 0, s>>>(n, fwd, inv, flag);
  SME_CHECK_LAUNCH("k_inverse_scatter");
  k_inverse_verify<<<grid_for(n, 256), 256, 0, s>>>(n, fwd, inv, flag);
  SME_CHECK_LAUNCH("k_inverse_verify");
  return SME_OK;
}

SME_API int sme_permute_vector(int dtype, int64_t n, const int32_t* p, const void* x, void* out,
                               sme_stream_t stream) {
  SME_REQUIRE(n >= 0, "negative length");
  if (n == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == SME_F64)
    k_scatter<double><<<grid_for(n, 256), 256, 0, s>>>(n, p, (const double*)x, (double*)out);
  else if (dtype == SME_F32)
    k_scatter<float><<<grid_for(n, 256), 256, 0, s>>>(n, p, (const float*)x, (float*)out);
  else if (dtype == -1)
    k_scatter<int32_t><<<grid_for(n, 256), 256, 0, s>>>(n, p, (const int32_t*)x, (int32_t*)out);
  else
    SME_REQUIRE(false, "unknown dtype %d", dtype);
  SME_CHECK_LAUNCH("k_scatter");
  return SME_OK;
}

SME_API int sme_gather(int dtype, int64_t n, const int32_t* idx, const void* x, void* out,
                       sme_stream_t stream) {
  SME_REQUIRE(n >= 0, "negative length");
  if (n == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == SME_F64)
    k_gather<double><<<grid_for(n, 256), 256, 0, s>>>(n, idx, (const double*)x, (double*)out);
  else if (dtype == SME_F32)
    k_gather<float><<<grid_for(n, 256), 256, 0, s>>>(n, idx, (const float*)x, (float*)out);
  else if (dtype == -1)
    k_gather<int32_t><<<grid_for(n, 256), 256, 0, s>>>(n, idx, (const int32_t*)x, (int32_t*)out);
  else
    SME_REQUIRE(false, "unknown dtype %d", dtype);
  SME_CHECK_LAUNCH("k_gather");
  return SME_OK;
}

SME_API int sme_coo_remap(int64_t nnz, const int32_t* row, const int32_t* col,
                          const int32_t* row_map, const int32_t* col_map, int32_t* row_out,
                          int32_t* col_out, sme_stream_t stream) {
  SME_REQUIRE(nnz >= 0, "negative nnz");
  if (nnz == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  k_coo_remap<<<grid_for(nnz, 256), 256, 0, s>>>(nnz, row, col, row_map, col_map, row_out, col_out);
  SME_CHECK_LAUNCH("k_coo_remap");
  return SME_OK;
}

SME_API int sme_rowshard_remap_cols(int64_t nnz, int64_t n_cols, int32_t parts, int64_t pad,
                                    const int32_t* col_in, int32_t* col_out, sme_stream_t stream) {
  SME_REQUIRE(parts >= 1 && parts <= n_cols, "parts %d outside [1, n_cols]", parts);
  int64_t base = n_cols / parts, extra = n_cols % parts;
  SME_REQUIRE(pad >= base + (extra ? 1 : 0), "pad %lld too small", (long long)pad);
  SME_REQUIRE(pad * parts < INT32_MAX, "padded x exceeds int32 indexing");
  if (nnz == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  k_rowshard_remap<<<grid_for(nnz, 256), 256, 0, s>>>(nnz, base, extra, pad, col_in, col_out);
  SME_CHECK_LAUNCH("k_rowshard_remap");
  return SME_OK;
}

SME_API int sme_maxabs_diff(int dtype, int64_t n, const void* got, const void* exp, double* out,
                            sme_stream_t stream) {
  if (n == 0) return SME_OK;
  cudaStream_t s = as_stream(stream);
  if (dtype == SME_F64)
    k_maxabs_diff<double><<<grid_for(n, 256, 4), 256, 0, s>>>(n, (const double*)got, (const double*)exp, out);
  else if (dtype == SME_F32)
    k_maxabs_diff<float><<<grid_for(n, 256, 4), 256, 0, s>>>(n, (const float*)got, (const float*)exp, out);
  else
    SME_REQUIRE(false, "unknown dtype %d", dtype);
  SME_CHECK_LAUNCH("k_maxabs_diff");
  return SME_OK;
}

namespace sme {
// Lazy module loading (CUDA 12 default) loads this file's module on the first launch of
// any of its kernels, ~10-20 ms each; sme_preload() does it ahead of time.
int preload_perm() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)k_inverse_scatter) == cudaSuccess ? 0 : -1;
}
}  // namespace sme
