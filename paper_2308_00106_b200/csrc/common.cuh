// common.cuh — shared helpers for the sm_100a kernels of libsme.so.
#pragma once
#include <cuda_runtime.h>
#include <stdint.h>
#include <stddef.h>

#include "../../include/sme.h"

#define SME_API extern "C" __attribute__((visibility("default")))

namespace sme {

// thread-local error message (sme_abi.cu)
void set_error(const char* fmt, ...);

inline cudaStream_t as_stream(sme_stream_t s) { return reinterpret_cast<cudaStream_t>(s); }

int sm_count();

// Grid for a grid-stride loop: enough CTAs to fill every SM `per_sm` times, never more
// than the work needs.
inline int grid_for(int64_t work_items, int threads, int per_sm = 8) {
  int64_t need = (work_items + threads - 1) / threads;
  int64_t cap = (int64_t)sm_count() * per_sm;
  if (need < 1) need = 1;
  return (int)(need < cap ? need : cap);
}

// sme_set_resident_grids: -1 (default) each site's tuned wave count, 0 = the fixed per-SM
// caps, k > 0 = k resident waves everywhere (sweeps)
extern int g_resident_grids;

// Grid for a grid-stride loop with equal static shares, in waves of the kernel's
// occupancy at this block size and dynamic shared memory (the CTAs one pass of the
// device holds), never more than the work needs.  A fixed per-SM cap ignores the
// occupancy: the C4 tile sort ran 2.29 waves of 7 CTAs per SM and its last, partial
// wave a full share at a third of the occupancy; several whole waves also let the SMs
// that run ahead take more shares (C4 K4 16.6 -> 15.5 ms, C3 14.9 -> 13.8 ms at 16 waves,
// profiles/round2/resident_grids.txt).  `legacy_per_sm`: the fixed cap (A/B only).
template <typename K>
inline int grid_waves(K kernel, int64_t work_items, int threads, size_t smem, int waves, int legacy_per_sm) {
  if (g_resident_grids == 0) return grid_for(work_items, threads, legacy_per_sm);
  if (g_resident_grids > 0) waves = g_resident_grids;
  int occ = 0;
  if (cudaOccupancyMaxActiveBlocksPerMultiprocessor(&occ, kernel, threads, smem) != cudaSuccess || occ < 1) {
    (void)cudaGetLastError();
    occ = 1;
  }
  return grid_for(work_items, threads, occ * waves);
}

inline size_t align_up(size_t x, size_t a = 256) { return (x + a - 1) / a * a; }

}  // namespace sme

#define SME_CHECK_LAUNCH(what)                                                        \
  do {                                                                                \
    cudaError_t _e = cudaGetLastError();                                              \
    if (_e != cudaSuccess) {                                                          \
      sme::set_error("%s: %s", what, cudaGetErrorString(_e));                         \
      return SME_ECUDA;                                                               \
    }                                                                                 \
  } while (0)

#define SME_CUDA(call)                                                                \
  do {                                                                                \
    cudaError_t _e = (call);                                                          \
    if (_e != cudaSuccess) {                                                          \
      sme::set_error("%s: %s", #call, cudaGetErrorString(_e));                        \
      return SME_ECUDA;                                                               \
    }                                                                                 \
  } while (0)

#define SME_REQUIRE(cond, ...)                                                        \
  do {                                                                                \
    if (!(cond)) {                                                                    \
      sme::set_error(__VA_ARGS__);                                                    \
      return SME_EINVAL;                                                              \
    }                                                                                 \
  } while (0)

namespace sme {

// ---------------------------------------------------------------------------
// cache-policy loads (PTX createpolicy + L2::cache_hint)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint64_t policy_evict_first() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_first.b64 %0, 1.0;" : "=l"(p));
  return p;
}
__device__ __forceinline__ uint64_t policy_evict_last() {
  uint64_t p;
  asm volatile("createpolicy.fractional.L2::evict_last.b64 %0, 1.0;" : "=l"(p));
  return p;
}

// streaming 128-bit loads: no L1 allocation, L2 evict-first
__device__ __forceinline__ int4 ld_stream_i4(const int4* p, uint64_t pol) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.s32 {%0,%1,%2,%3}, [%4], %5;"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ double2 ld_stream_d2(const double2* p, uint64_t pol) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v2.f64 {%0,%1}, [%2], %3;"
               : "=d"(r.x), "=d"(r.y)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ float4 ld_stream_f4(const float4* p, uint64_t pol) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.v4.f32 {%0,%1,%2,%3}, [%4], %5;"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ int ld_stream_i1(const int* p, uint64_t pol) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.s32 %0, [%1], %2;"
               : "=r"(r)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ double ld_stream(const double* p, uint64_t pol) {
  double r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f64 %0, [%1], %2;"
               : "=d"(r)
               : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ float ld_stream(const float* p, uint64_t pol) {
  float r;
  asm volatile("ld.global.nc.L1::no_allocate.L2::cache_hint.f32 %0, [%1], %2;"
               : "=f"(r)
               : "l"(p), "l"(pol));
  return r;
}

// streaming loads without an L2 policy operand (a per-thread policy register costs an
// R2UR + constant load per access when the compiler cannot keep it uniform)
__device__ __forceinline__ int4 ld_nc_na_i4(const int4* p) {
  int4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.s32 {%0,%1,%2,%3}, [%4];"
               : "=r"(r.x), "=r"(r.y), "=r"(r.z), "=r"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ double2 ld_nc_na_d2(const double2* p) {
  double2 r;
  asm volatile("ld.global.nc.L1::no_allocate.v2.f64 {%0,%1}, [%2];" : "=d"(r.x), "=d"(r.y) : "l"(p));
  return r;
}
__device__ __forceinline__ float4 ld_nc_na_f4(const float4* p) {
  float4 r;
  asm volatile("ld.global.nc.L1::no_allocate.v4.f32 {%0,%1,%2,%3}, [%4];"
               : "=f"(r.x), "=f"(r.y), "=f"(r.z), "=f"(r.w)
               : "l"(p));
  return r;
}
__device__ __forceinline__ int ld_nc_na_i1(const int* p) {
  int r;
  asm volatile("ld.global.nc.L1::no_allocate.s32 %0, [%1];" : "=r"(r) : "l"(p));
  return r;
}

// read-only loads that allocate in L1 (lines re-read by neighbouring lanes), L2 hint
__device__ __forceinline__ double ld_l1(const double* p, uint64_t pol) {
  double r;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ float ld_l1(const float* p, uint64_t pol) {
  float r;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ int ld_l1(const int* p, uint64_t pol) {
  int r;
  asm volatile("ld.global.nc.L2::cache_hint.s32 %0, [%1], %2;" : "=r"(r) : "l"(p), "l"(pol));
  return r;
}

// gathers of x: read-only path, L2 evict-last so the vector stays resident
__device__ __forceinline__ double ld_keep(const double* p, uint64_t pol) {
  double r;
  asm volatile("ld.global.nc.L2::cache_hint.f64 %0, [%1], %2;" : "=d"(r) : "l"(p), "l"(pol));
  return r;
}
__device__ __forceinline__ float ld_keep(const float* p, uint64_t pol) {
  float r;
  asm volatile("ld.global.nc.L2::cache_hint.f32 %0, [%1], %2;" : "=f"(r) : "l"(p), "l"(pol));
  return r;
}

// streaming store (evict-first)
__device__ __forceinline__ void st_stream(double* p, double v) {
  asm volatile("st.global.cs.f64 [%0], %1;" ::"l"(p), "d"(v));
}
__device__ __forceinline__ void st_stream(float* p, float v) {
  asm volatile("st.global.cs.f32 [%0], %1;" ::"l"(p), "f"(v));
}
__device__ __forceinline__ void st_stream(int32_t* p, int32_t v) {
  asm volatile("st.global.cs.s32 [%0], %1;" ::"l"(p), "r"(v));
}

// ---------------------------------------------------------------------------
// exact division by an invariant divisor: q = (n * m) >> s, exact for
// 0 <= n < 2^31 and 1 <= d < 2^31 (m = ceil(2^s / d), s = 32 + ceil(log2 d)).
// ---------------------------------------------------------------------------
struct FastDiv {
  uint64_t m;
  uint32_t s;
};
inline FastDiv make_fastdiv(uint32_t d) {
  uint32_t l = 0;
  while ((1ull << l) < d) ++l;
  uint32_t s = 32 + l;
  unsigned __int128 num = ((unsigned __int128)1) << s;
  uint64_t m = (uint64_t)((num + d - 1) / d);
  return FastDiv{m, s};
}
__device__ __forceinline__ uint32_t fastdiv(uint32_t n, FastDiv f) {
  return (uint32_t)(((uint64_t)n * f.m) >> f.s);
}

// _bin_index (entropy.py:65-67): min(idx // (n // bins), bins - 1)
struct Binner {
  FastDiv div;
  int32_t last;
};
inline Binner make_binner(int64_t n, int32_t bins) {
  int64_t width = n / bins;
  return Binner{make_fastdiv((uint32_t)width), bins - 1};
}
__device__ __forceinline__ int32_t bin_of(int32_t idx, Binner b) {
  int32_t q = (int32_t)fastdiv((uint32_t)idx, b.div);
  return q < b.last ? q : b.last;
}

__device__ __forceinline__ int lane_id() { return threadIdx.x & 31; }

// ---------------------------------------------------------------------------
// mbarrier + 1-D bulk async copies (TMA engine, cp.async.bulk; sm_90+)
// ---------------------------------------------------------------------------
__device__ __forceinline__ uint32_t smem_u32(const void* p) {
  return (uint32_t)__cvta_generic_to_shared(p);
}
__device__ __forceinline__ void mbar_init(uint64_t* bar, uint32_t count) {
  asm volatile("mbarrier.init.shared::cta.b64 [%0], %1;" ::"r"(smem_u32(bar)), "r"(count));
}
__device__ __forceinline__ void fence_mbar_init() {
  asm volatile("fence.mbarrier_init.release.cluster;" ::: "memory");
}
__device__ __forceinline__ void fence_proxy_async_smem() {
  asm volatile("fence.proxy.async.shared::cta;" ::: "memory");
}
__device__ __forceinline__ void mbar_arrive_expect_tx(uint64_t* bar, uint32_t bytes) {
  asm volatile("mbarrier.arrive.expect_tx.shared::cta.b64 _, [%0], %1;" ::"r"(smem_u32(bar)), "r"(bytes)
               : "memory");
}
__device__ __forceinline__ void mbar_wait(uint64_t* bar, uint32_t parity) {
  asm volatile(
      "{\n"
      ".reg .pred p;\n"
      "WAIT_%=:\n"
      "mbarrier.try_wait.parity.shared::cta.b64 p, [%0], %1;\n"
      "@!p bra WAIT_%=;\n"
      "}\n" ::"r"(smem_u32(bar)),
      "r"(parity)
      : "memory");
}
// per-thread 16-byte async copy global -> shared (LDGSTS), L1 bypass, L2 hint;
// src_bytes < 16 zero-fills the rest
__device__ __forceinline__ void cp_async16(void* dst, const void* src, uint32_t src_bytes, uint64_t policy) {
  asm volatile("cp.async.cg.shared.global.L2::cache_hint [%0], [%1], 16, %2, %3;" ::"r"(smem_u32(dst)), "l"(src),
               "r"(src_bytes), "l"(policy)
               : "memory");
}
__device__ __forceinline__ void cp_async_commit() { asm volatile("cp.async.commit_group;" ::: "memory"); }
template <int N>
__device__ __forceinline__ void cp_async_wait() {
  asm volatile("cp.async.wait_group %0;" ::"n"(N) : "memory");
}

// global -> shared bulk copy completing on `bar`; size and both addresses 16-B aligned
__device__ __forceinline__ void bulk_g2s(void* dst, const void* src, uint32_t bytes, uint64_t* bar,
                                         uint64_t policy) {
  asm volatile(
      "cp.async.bulk.shared::cluster.global.mbarrier::complete_tx::bytes.L2::cache_hint [%0], [%1], %2, [%3], %4;" ::"r"(
          smem_u32(dst)),
      "l"(src), "r"(bytes), "r"(smem_u32(bar)), "l"(policy)
      : "memory");
}

}  // namespace sme
