// shuffle_gen.cu — the swap partners of Generator(PCG64).permutation(n) drawn on the GPU,
// bit-exact with numpy (the GENERATION half of random_permutation, permute.py:71-81;
// the swaps are sme_fy_apply, shuffle.cu).
//
// numpy: for i = n-1 .. 1: draw v = next_uint32() & mask(i) until v <= i; j_i = v.
// Over the uint32 stream U_t (t = 0, 1, ...; a buffered high half first when
// has_uint32), draw t is made for step i_t = n-1 - t + R_t, where R_t counts the
// rejections before t, and is rejected iff (U_t & mask(i_t)) > i_t.  R_t is a sequential
// counter, but it is confined to a narrow band: the draws before step i are a sum of
// independent geometric variables, whose mean D(i) and variance V(i) have closed forms,
// so every block of draws gets a window [ilo, ihi] of steps it can be serving
// (D ± 6 sqrt(V) + slack).  Inside it, almost every draw is decided without knowing
// R_t exactly: accept when U & mask <= ilo, reject when U & mask > ihi (one mask for the
// whole window).  Only the rest ("ambiguous": values inside the window, windows that
// straddle a power of two, and every draw for steps below 2^16) need the exact count,
// and the host resolves those in order with the certain rejections before each of them
// (~2 % of the ~1.47 n draws).  A final pass recomputes every R_t, checks that each
// certain draw's step really lay inside its window (if not — odds ~1e-30 — the caller
// falls back to the sequential host replay), and writes j[i_t] for the accepted draws.
// Measured at n = 50M: 1.16M of the 73M draws are ambiguous (6-sigma windows); ~15 ms
// per axis warm, against 50 ms for the sequential host replay.
#include "common.cuh"
#include "scan.cuh"

#include <algorithm>
#include <chrono>
#include <cmath>
#include <cstdio>
#include <cstdlib>
#include <memory>
#include <vector>

namespace sme {
namespace {

typedef unsigned __int128 u128;

constexpr int GG_NT = 256;
constexpr int GG_PER = 16;                  // draws per thread
constexpr int64_t GG_BLK = GG_NT * GG_PER;  // draws per CTA (one window each)
constexpr int64_t GG_AMB_FLOOR = 1 << 16;   // steps below this are always resolved on the host
constexpr double GG_SIGMAS = 6.0;   // a wider excursion (p ~ 1e-8) fails the window check -> host replay
constexpr double GG_SLACK = 1024.0;

__host__ __device__ inline u128 pcg_mult() {
  return ((u128)2549297995355413924ULL << 64) | (u128)4865540595714422341ULL;
}

__host__ __device__ inline u128 pcg_advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = pcg_mult(), cur_plus = inc;
  while (delta > 0) {
    if (delta & 1) {
      acc_mult *= cur_mult;
      acc_plus = acc_plus * cur_mult + cur_plus;
    }
    cur_plus = (cur_mult + 1) * cur_plus;
    cur_mult *= cur_mult;
    delta >>= 1;
  }
  return acc_mult * state + acc_plus;
}

__host__ __device__ inline uint64_t pcg_out(u128 s) {
  const uint64_t hi = (uint64_t)(s >> 64), lo = (uint64_t)s;
  const unsigned rot = (unsigned)(hi >> 58);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

__host__ __device__ inline uint32_t smear(uint32_t x) {
  x |= x >> 1;
  x |= x >> 2;
  x |= x >> 4;
  x |= x >> 8;
  x |= x >> 16;
  return x;
}

struct GenState {
  u128 state, inc;  // before the first fresh output
  int lead;         // 1: U_0 is the buffered high half buf32
  uint32_t buf32;
  int64_t n;        // permutation size
  int64_t T;        // draws generated
};

// this thread's 16 draws U[t0 .. t0+15]; the CTA's thread 0 jumps to the block's first
// output (O(log t) steps) and the others jump from there (< 2^11 outputs)
__device__ inline void gen_draws(const GenState& g, int64_t t0, uint32_t (&u)[GG_PER]) {
  __shared__ u128 s_base;
  const int64_t f0 = t0 - g.lead;  // fresh index of the first draw (-1: the buffered half)
  uint64_t next = f0 > 0 ? (uint64_t)(f0 >> 1) : 0;  // next output to produce
  const int64_t fb = (int64_t)blockIdx.x * GG_BLK - g.lead;
  const uint64_t base = fb > 0 ? (uint64_t)(fb >> 1) : 0;
  if (threadIdx.x == 0) s_base = pcg_advance(g.state, g.inc, base);
  __syncthreads();
  u128 x = pcg_advance(s_base, g.inc, next - base);
  uint64_t v = 0;
#pragma unroll
  for (int k = 0; k < GG_PER; ++k) {
    const int64_t f = f0 + k;
    if (f < 0) {
      u[k] = g.buf32;
      continue;
    }
    const uint64_t o = (uint64_t)(f >> 1);
    while (next <= o) {
      x = x * pcg_mult() + g.inc;
      v = pcg_out(x);
      ++next;
    }
    u[k] = (f & 1) ? (uint32_t)(v >> 32) : (uint32_t)v;
  }
}

// 0: accepted for sure, 1: rejected for sure, 2: needs the exact step
__device__ inline int classify(uint32_t u, int64_t ilo, int64_t ihi) {
  if (ilo < GG_AMB_FLOOR) return 2;
  const uint32_t m = smear((uint32_t)ilo);
  if (m != smear((uint32_t)ihi)) return 2;
  const int64_t d = (int64_t)(u & m);
  return d <= ilo ? 0 : d > ihi ? 1 : 2;
}

__global__ void __launch_bounds__(GG_NT) k_gg_draw_classify(GenState g, const int64_t* __restrict__ wlo,
                                                              const int64_t* __restrict__ whi, uint32_t* __restrict__ U,
                                                              int32_t* __restrict__ cr_cnt, int32_t* __restrict__ amb_cnt) {
  const int64_t blk = blockIdx.x;
  const int64_t t0 = blk * GG_BLK + (int64_t)threadIdx.x * GG_PER;
  uint32_t u[GG_PER];
  gen_draws(g, t0, u);
  uint4* dst = reinterpret_cast<uint4*>(U + t0);
#pragma unroll
  for (int q = 0; q < GG_PER / 4; ++q) dst[q] = make_uint4(u[4 * q], u[4 * q + 1], u[4 * q + 2], u[4 * q + 3]);
  const int64_t ilo = wlo[blk], ihi = whi[blk];
  int cr = 0, amb = 0;
#pragma unroll
  for (int k = 0; k < GG_PER; ++k) {
    const int c = classify(u[k], ilo, ihi);
    cr += c == 1;
    amb += c == 2;
  }
  __shared__ int64_t s_tot;
  block_exclusive_scan<GG_NT>(cr, &s_tot);
  if (threadIdx.x == 0) cr_cnt[blk] = (int32_t)s_tot;
  __syncthreads();
  block_exclusive_scan<GG_NT>(amb, &s_tot);
  if (threadIdx.x == 0) amb_cnt[blk] = (int32_t)s_tot;
}

// the ambiguous draws in order: t, U_t and the certain rejections before t
__global__ void __launch_bounds__(GG_NT) k_gg_compact(const uint32_t* __restrict__ U, const int64_t* __restrict__ wlo,
                                                        const int64_t* __restrict__ whi, const int64_t* __restrict__ cr_base,
                                                        const int64_t* __restrict__ amb_base, uint32_t* __restrict__ amb_t,
                                                        uint32_t* __restrict__ amb_u, uint32_t* __restrict__ amb_cr) {
  const int64_t blk = blockIdx.x;
  const int64_t t0 = blk * GG_BLK + (int64_t)threadIdx.x * GG_PER;
  const uint4* src = reinterpret_cast<const uint4*>(U + t0);
  uint32_t u[GG_PER];
#pragma unroll
  for (int q = 0; q < GG_PER / 4; ++q) {
    const uint4 v = src[q];
    u[4 * q] = v.x; u[4 * q + 1] = v.y; u[4 * q + 2] = v.z; u[4 * q + 3] = v.w;
  }
  const int64_t ilo = wlo[blk], ihi = whi[blk];
  int cls[GG_PER];
  int cr = 0, amb = 0;
#pragma unroll
  for (int k = 0; k < GG_PER; ++k) {
    cls[k] = classify(u[k], ilo, ihi);
    cr += cls[k] == 1;
    amb += cls[k] == 2;
  }
  __shared__ int64_t s_tot;
  int64_t cr_run = cr_base[blk] + block_exclusive_scan<GG_NT>(cr, &s_tot);
  __syncthreads();
  int64_t idx = amb_base[blk] + block_exclusive_scan<GG_NT>(amb, &s_tot);
#pragma unroll
  for (int k = 0; k < GG_PER; ++k) {
    if (cls[k] == 2) {
      amb_t[idx] = (uint32_t)(t0 + k);
      amb_u[idx] = u[k];
      amb_cr[idx] = (uint32_t)cr_run;
      ++idx;
    }
    cr_run += cls[k] == 1;
  }
}

// every R_t, the window check, and j[i_t] = U_t & mask(i_t) for the accepted draws t <= t_last
__global__ void __launch_bounds__(GG_NT) k_gg_write(const uint32_t* __restrict__ U, const int64_t* __restrict__ wlo,
                                                      const int64_t* __restrict__ whi, const int64_t* __restrict__ rej_base,
                                                      const int64_t* __restrict__ amb_base, const uint8_t* __restrict__ dec,
                                                      int64_t t_last, int64_t n, int32_t* __restrict__ j,
                                                      int* __restrict__ bad) {
  const int64_t blk = blockIdx.x;
  const int64_t t0 = blk * GG_BLK + (int64_t)threadIdx.x * GG_PER;
  const uint4* src = reinterpret_cast<const uint4*>(U + t0);
  uint32_t u[GG_PER];
#pragma unroll
  for (int q = 0; q < GG_PER / 4; ++q) {
    const uint4 v = src[q];
    u[4 * q] = v.x; u[4 * q + 1] = v.y; u[4 * q + 2] = v.z; u[4 * q + 3] = v.w;
  }
  const int64_t ilo = wlo[blk], ihi = whi[blk];
  int cls[GG_PER];
  int amb = 0;
#pragma unroll
  for (int k = 0; k < GG_PER; ++k) {
    cls[k] = classify(u[k], ilo, ihi);
    amb += cls[k] == 2;
  }
  __shared__ int64_t s_tot;
  int64_t aidx = amb_base[blk] + block_exclusive_scan<GG_NT>(amb, &s_tot);
  __syncthreads();
  unsigned rejm = 0;  // this thread's rejected draws (ambiguous ones as the host decided)
  int rej = 0;
#pragma unroll
  for (int k = 0; k < GG_PER; ++k) {
    bool r = cls[k] == 1;
    if (cls[k] == 2) {
      r = t0 + k <= t_last && dec[aidx] != 0;
      ++aidx;
    }
    rejm |= r ? (1u << k) : 0u;
    rej += r;
  }
  int64_t R = rej_base[blk] + block_exclusive_scan<GG_NT>(rej, &s_tot);
  bool violated = false;
#pragma unroll
  for (int k = 0; k < GG_PER; ++k) {
    const int64_t t = t0 + k;
    if (t > t_last) break;
    const int64_t i = n - 1 - t + R;
    if (cls[k] != 2) violated |= i < ilo || i > ihi;
    if ((rejm >> k) & 1u) {
      ++R;
    } else if (i >= 1 && i < n) {
      j[i] = (int32_t)(u[k] & smear((uint32_t)i));
    } else {
      violated = true;
    }
  }
  if (violated) atomicOr(bad, 1);
}

// harmonic sums H(x) = sum_{k<=x} 1/k and H2(x) = sum 1/k^2 (exact below 2^16,
// asymptotic above — the windows carry a 12-sigma margin, so 1e-9 is plenty)
struct Harmonic {
  std::vector<double> h, h2;
  Harmonic() : h(1 << 16 | 1), h2(1 << 16 | 1) {
    for (size_t k = 1; k < h.size(); ++k) {
      h[k] = h[k - 1] + 1.0 / (double)k;
      h2[k] = h2[k - 1] + 1.0 / ((double)k * (double)k);
    }
  }
  double H(double x) const {
    if (x < (double)h.size()) return h[(size_t)x];
    return std::log(x) + 0.57721566490153286 + 0.5 / x - 1.0 / (12.0 * x * x);
  }
  double H2(double x) const {
    if (x < (double)h2.size()) return h2[(size_t)x];
    return 1.6449340668482264 - 1.0 / x + 0.5 / (x * x) - 1.0 / (6.0 * x * x * x);
  }
};

// the step grid: ig[g] (descending) with the earliest / latest draw index at which step
// ig[g] can start (increasing)
struct StepGrid {
  std::vector<int64_t> ig;
  std::vector<double> tlo, thi;
};

StepGrid step_grid(int64_t n) {
  static const Harmonic hm;
  constexpr int64_t G = 2048;
  StepGrid sg;
  double D = 0.0, V = 0.0;  // mean / variance of the draws before step i
  int64_t i = n - 1;
  auto push = [&]() {
    const double w = GG_SIGMAS * std::sqrt(V) + GG_SLACK;
    sg.ig.push_back(i);
    sg.tlo.push_back(D - w);
    sg.thi.push_back(D + w);
  };
  push();
  while (i > 0) {
    const int64_t i_next = std::max<int64_t>(0, i - G);
    // steps k = i, i-1, ..., i_next+1 complete before step i_next starts
    int64_t hi = i;
    while (hi > i_next) {
      const uint32_t M = smear((uint32_t)hi);
      const int64_t lo = std::max<int64_t>(i_next + 1, (int64_t)(M >> 1) + 1);  // same mask on [lo, hi]
      const double m1 = (double)M + 1.0;
      const double s1 = hm.H((double)hi + 1.0) - hm.H((double)lo);  // sum 1/(k+1)
      const double s2 = hm.H2((double)hi + 1.0) - hm.H2((double)lo);
      D += m1 * s1;
      V += m1 * m1 * s2 - m1 * s1;
      hi = lo - 1;
    }
    i = i_next;
    push();
  }
  return sg;
}

// per block of draws: the steps [ilo, ihi] it can be serving
void block_windows(const StepGrid& sg, int64_t n, int64_t n_blocks, std::vector<int64_t>& wlo,
                   std::vector<int64_t>& whi) {
  wlo.resize((size_t)n_blocks);
  whi.resize((size_t)n_blocks);
  for (int64_t b = 0; b < n_blocks; ++b) {
    const double t_first = (double)(b * GG_BLK), t_lastd = (double)(b * GG_BLK + GG_BLK - 1);
    // i_t >= ig[g*] with g* the first grid point whose earliest start lies after t
    const size_t gs = (size_t)(std::upper_bound(sg.tlo.begin(), sg.tlo.end(), t_lastd) - sg.tlo.begin());
    wlo[(size_t)b] = gs < sg.ig.size() ? sg.ig[gs] : 0;
    // i_t <= ig[h] with h the last grid point whose latest start is not after t
    const size_t h1 = (size_t)(std::upper_bound(sg.thi.begin(), sg.thi.end(), t_first) - sg.thi.begin());
    whi[(size_t)b] = h1 == 0 ? n - 1 : sg.ig[h1 - 1];
  }
}

}  // namespace
}  // namespace sme

using namespace sme;

// numpy's swap partners straight into d_j (int32[n], d_j[0] = 0), drawn on the GPU;
// st (numpy PCG64.state as six words, see sme_host_pcg64_permutation) is advanced as
// the full shuffle leaves it.  Returns SME_OK, or 1 when a window check failed (nothing
// usable written; st untouched) so the caller replays on the host.  HOST call that
// synchronises `stream` (the ambiguous draws go to the host and back).
namespace sme {
namespace {
// bytes of the n-dependent scratch (the draws, windows, bases, counts)
size_t gg_scratch_bytes(int64_t n, int64_t* n_blocks_out) {
  const StepGrid sg = step_grid(n);
  const int64_t t_max = (int64_t)std::ceil(sg.thi.back()) + GG_BLK;
  const int64_t n_blocks = (t_max + GG_BLK - 1) / GG_BLK;
  if (n_blocks_out) *n_blocks_out = n_blocks;
  const size_t b_U = align_up((size_t)(n_blocks * GG_BLK) * 4), b_w = align_up((size_t)n_blocks * 8),
               b_c = align_up((size_t)n_blocks * 4);
  const int64_t amb_cap = n_blocks * GG_BLK / 16;  // ambiguous draws held in the caller's scratch
  return b_U + 4 * b_w + 2 * b_c + 256 + 3 * align_up((size_t)amb_cap * 4 + 4) + align_up((size_t)amb_cap + 1);
}
}  // namespace
}  // namespace sme

// Scratch of sme_pcg64_swap_partners_gpu for size n (pass a buffer this large to skip
// the stream-ordered allocation inside; the few ambiguous draws still use one).
SME_API int sme_pcg64_swap_partners_gpu_workspace_size(int64_t n, size_t* bytes) {
  SME_REQUIRE(bytes && n >= 2 && n < INT32_MAX, "bad arguments (n=%lld)", (long long)n);
  *bytes = gg_scratch_bytes(n, nullptr);
  return SME_OK;
}

SME_API int sme_pcg64_swap_partners_gpu(uint64_t* st, int64_t n, int32_t* d_j, void* d_ws, size_t ws_bytes,
                                        sme_stream_t stream) {
  SME_REQUIRE(st && d_j && n >= 2 && n < INT32_MAX, "bad arguments (n=%lld)", (long long)n);
  cudaStream_t s = as_stream(stream);
  const bool dbg = std::getenv("SME_GG_DEBUG") != nullptr;
  auto now = [] { return std::chrono::steady_clock::now(); };
  auto ms = [](auto a, auto b) { return std::chrono::duration<double, std::milli>(b - a).count(); };
  const auto c0 = now();
  GenState g;
  g.state = ((u128)st[0] << 64) | st[1];
  g.inc = ((u128)st[2] << 64) | st[3];
  g.lead = st[4] != 0 ? 1 : 0;
  g.buf32 = (uint32_t)st[5];
  g.n = n;
  // windows first (they fix how many draws to make)
  const StepGrid sg = step_grid(n);
  const int64_t t_max = (int64_t)std::ceil(sg.thi.back()) + GG_BLK;  // draws of the latest plausible end
  SME_REQUIRE(t_max < (int64_t)UINT32_MAX, "too many draws for 32-bit draw indices");
  const int64_t n_blocks = (t_max + GG_BLK - 1) / GG_BLK;
  std::vector<int64_t> wlo, whi;
  block_windows(sg, n, n_blocks, wlo, whi);
  g.T = n_blocks * GG_BLK;
  const auto c1 = now();
  // device buffers (one allocation)
  const size_t b_U = align_up((size_t)g.T * 4), b_w = align_up((size_t)n_blocks * 8), b_c = align_up((size_t)n_blocks * 4);
  char* ws = nullptr;
  const size_t ws_need = b_U + 4 * b_w + 2 * b_c + 256;
  const bool own_ws = !(d_ws && ws_bytes >= ws_need);
  if (own_ws)
    SME_CUDA(cudaMallocAsync((void**)&ws, ws_need, s));
  else
    ws = (char*)d_ws;
  uint32_t* U = (uint32_t*)ws;
  int64_t* d_wlo = (int64_t*)(ws + b_U);
  int64_t* d_whi = (int64_t*)(ws + b_U + b_w);
  int64_t* d_base1 = (int64_t*)(ws + b_U + 2 * b_w);  // certain-rejection bases, later all-rejection bases
  int64_t* d_base2 = (int64_t*)(ws + b_U + 3 * b_w);  // ambiguous bases
  int32_t* d_cr = (int32_t*)(ws + b_U + 4 * b_w);
  int32_t* d_amb = (int32_t*)(ws + b_U + 4 * b_w + b_c);
  int* d_bad = (int*)(ws + b_U + 4 * b_w + 2 * b_c);
  auto fail = [&](int rc) {
    if (own_ws) cudaFreeAsync(ws, s);
    return rc;
  };
  SME_CUDA(cudaMemcpyAsync(d_wlo, wlo.data(), (size_t)n_blocks * 8, cudaMemcpyHostToDevice, s));
  SME_CUDA(cudaMemcpyAsync(d_whi, whi.data(), (size_t)n_blocks * 8, cudaMemcpyHostToDevice, s));
  SME_CUDA(cudaMemsetAsync(d_bad, 0, 4, s));
  k_gg_draw_classify<<<(unsigned)n_blocks, GG_NT, 0, s>>>(g, d_wlo, d_whi, U, d_cr, d_amb);
  SME_CHECK_LAUNCH("k_gg_draw_classify");
  std::vector<int32_t> cr((size_t)n_blocks), amb((size_t)n_blocks);
  SME_CUDA(cudaMemcpyAsync(cr.data(), d_cr, (size_t)n_blocks * 4, cudaMemcpyDeviceToHost, s));
  SME_CUDA(cudaMemcpyAsync(amb.data(), d_amb, (size_t)n_blocks * 4, cudaMemcpyDeviceToHost, s));
  SME_CUDA(cudaStreamSynchronize(s));
  const auto c2 = now();
  std::vector<int64_t> cr_base((size_t)n_blocks), amb_base((size_t)n_blocks);
  int64_t n_amb = 0, c_acc = 0;
  for (int64_t b = 0; b < n_blocks; ++b) {
    cr_base[(size_t)b] = c_acc;
    amb_base[(size_t)b] = n_amb;
    c_acc += cr[(size_t)b];
    n_amb += amb[(size_t)b];
  }
  char* aws = nullptr;
  const size_t b_a = align_up((size_t)n_amb * 4 + 4), b_ad = align_up((size_t)n_amb + 1);
  const bool own_aws = own_ws || ws_bytes < ws_need + 3 * b_a + b_ad;  // the caller's scratch holds them
  if (own_aws)
    SME_CUDA(cudaMallocAsync((void**)&aws, 3 * b_a + b_ad, s));
  else
    aws = ws + ws_need;
  uint32_t* d_at = (uint32_t*)aws;
  uint32_t* d_acr = (uint32_t*)(aws + b_a);
  uint32_t* d_au = (uint32_t*)(aws + 2 * b_a);
  uint8_t* d_dec = (uint8_t*)(aws + 3 * b_a);
  auto fail2 = [&](int rc) {
    if (own_aws) cudaFreeAsync(aws, s);
    return fail(rc);
  };
  SME_CUDA(cudaMemcpyAsync(d_base1, cr_base.data(), (size_t)n_blocks * 8, cudaMemcpyHostToDevice, s));
  SME_CUDA(cudaMemcpyAsync(d_base2, amb_base.data(), (size_t)n_blocks * 8, cudaMemcpyHostToDevice, s));
  k_gg_compact<<<(unsigned)n_blocks, GG_NT, 0, s>>>(U, d_wlo, d_whi, d_base1, d_base2, d_at, d_au, d_acr);
  SME_CHECK_LAUNCH("k_gg_compact");
  // one host block for the three arrays (uninitialised: the copies fill it) + decisions
  std::unique_ptr<uint32_t[]> hbuf(new uint32_t[(size_t)(3 * n_amb + 1)]);
  uint32_t* at = hbuf.get();
  uint32_t* acr = at + n_amb;
  uint32_t* au = acr + n_amb;
  std::unique_ptr<uint8_t[]> dec(new uint8_t[(size_t)n_amb + 1]);
  if (n_amb) {
    SME_CUDA(cudaMemcpyAsync(at, d_at, (size_t)n_amb * 4, cudaMemcpyDeviceToHost, s));
    SME_CUDA(cudaMemcpyAsync(acr, d_acr, (size_t)n_amb * 4, cudaMemcpyDeviceToHost, s));
    SME_CUDA(cudaMemcpyAsync(au, d_au, (size_t)n_amb * 4, cudaMemcpyDeviceToHost, s));
  }
  SME_CUDA(cudaStreamSynchronize(s));
  const auto c3 = now();
  // the ambiguous draws, in order, with their exact step
  int64_t amb_rej = 0, t_last = -1;
  std::vector<int64_t> blk_rej((size_t)n_blocks, 0);
  int64_t k_end = n_amb;
  uint32_t M = 0;  // the current mask (recomputed only when i leaves (M/2, M])
  for (int64_t k = 0; k < n_amb; ++k) {
    const int64_t t = at[k];
    const int64_t i = n - 1 - t + (int64_t)acr[k] + amb_rej;
    if (i < 1 || i >= n) {  // the end went by on a draw classified as certain: fall back
      k_end = -1;
      break;
    }
    if (i > (int64_t)M || i <= (int64_t)(M >> 1)) M = smear((uint32_t)i);
    const int rej = (int64_t)(au[k] & M) > i;
    dec[k] = (uint8_t)rej;
    amb_rej += rej;
    if (__builtin_expect((i == 1) & (rej == 0), 0)) {  // one combined test: rej is random
      t_last = t;
      k_end = k + 1;
      break;
    }
  }
  for (int64_t k = 0; k < k_end; ++k) blk_rej[(size_t)(at[k] / GG_BLK)] += dec[k];
  const auto c4 = now();
  if (t_last < 0) return fail2(1);
  std::vector<int64_t> rej_base((size_t)n_blocks);
  for (int64_t b = 0, acc = 0; b < n_blocks; ++b) {
    rej_base[(size_t)b] = cr_base[(size_t)b] + acc;
    acc += blk_rej[(size_t)b];
  }
  if (k_end > 0) SME_CUDA(cudaMemcpyAsync(d_dec, dec.get(), (size_t)k_end, cudaMemcpyHostToDevice, s));
  SME_CUDA(cudaMemcpyAsync(d_base1, rej_base.data(), (size_t)n_blocks * 8, cudaMemcpyHostToDevice, s));
  SME_CUDA(cudaMemsetAsync(d_j, 0, 4, s));  // j[0] = 0
  const unsigned used_blocks = (unsigned)(t_last / GG_BLK + 1);
  k_gg_write<<<used_blocks, GG_NT, 0, s>>>(U, d_wlo, d_whi, d_base1, d_base2, d_dec, t_last, n, d_j, d_bad);
  SME_CHECK_LAUNCH("k_gg_write");
  int bad = 0;
  SME_CUDA(cudaMemcpyAsync(&bad, d_bad, 4, cudaMemcpyDeviceToHost, s));
  SME_CUDA(cudaStreamSynchronize(s));
  fail2(SME_OK);  // release the scratch
  if (dbg)
    std::fprintf(stderr,
                 "[gg] n=%lld draws=%lld ambiguous=%lld | windows %.2f ms, draw+classify %.2f, compact+D2H %.2f, "
                 "host resolve %.2f, write %.2f\n",
                 (long long)n, (long long)(t_last + 1), (long long)n_amb, ms(c0, c1), ms(c1, c2), ms(c2, c3), ms(c3, c4),
                 ms(c4, now()));
  if (bad) return 1;
  // generator state after t_last + 1 draws (the buffered half counts as one)
  const int64_t fresh = t_last + 1 - g.lead;
  const uint64_t outputs = (uint64_t)((fresh + 1) / 2);
  const u128 ns = pcg_advance(g.state, g.inc, outputs);
  st[0] = (uint64_t)(ns >> 64);
  st[1] = (uint64_t)ns;
  if (fresh > 0) {
    st[4] = (fresh & 1) ? 1 : 0;
    st[5] = (uint32_t)(pcg_out(ns) >> 32);  // the high half of the last output drawn
  } else {
    st[4] = 0;  // only the buffered half was used
  }
  return SME_OK;
}

namespace sme {
// Lazy module loading (CUDA 12 default) loads this file's module on the first launch of
// any of its kernels, ~10-20 ms each; sme_preload() does it ahead of time.
int preload_shuffle_gen() {
  cudaFuncAttributes a;
  return cudaFuncGetAttributes(&a, (const void*)k_gg_draw_classify) == cudaSuccess ? 0 : -1;
}
}  // namespace sme
