// pcg64_host.cpp — host-side, bit-exact restatement of numpy's
// Generator(PCG64).permutation(n) (the permutation GENERATION step of
// random_permutation, permute.py:71-81, and of riffle_shuffle_permutation,
// permute.py:142-157).  SURVEY.md §8(f) row 2.
//
// Why on the host: Fisher–Yates is a chain of n-1 dependent swaps driven by one
// sequential random stream; its cost at 50M elements is the cache misses of the
// random swap partner (numpy: ~1.4 s per axis), not arithmetic.  The swap
// partners depend only on the random stream, never on the array, so they can be
// drawn ahead and their cache lines prefetched: the loop becomes bandwidth-bound
// instead of latency-bound.  The output is the int32 forward vector the GPU path
// uploads directly (half the bytes of numpy's int64 arange).
//
// Algorithm (numpy/random/_generator.pyx `shuffle` 1-D fast path + `_shuffle_raw`,
// numpy/random/src/distributions/distributions.c `random_interval`, pcg64.h):
//   a = arange(n); for i = n-1 .. 1: j = random_interval(i); swap(a[i], a[j])
//   random_interval(max): mask = all-ones up to max's top bit; draw
//     next_uint32() & mask until <= max (max < 2^32 here: n <= 2^31)
//   next_uint32: the low half of a fresh next_uint64, buffering the high half
//     for the following call (has_uint32 / uinteger)
//   next_uint64 (PCG XSL-RR 128/64): state = state * M + inc (mod 2^128);
//     out = rotr64(hi(state) ^ lo(state), hi(state) >> 58)
// Pinned by tests/test_host.py against numpy itself (sizes 1..2^20, several
// seeds, and the two consecutive permutations of one riffle generator).
#include <stdint.h>
#include <stddef.h>

#include <sys/mman.h>

#include <algorithm>
#include <atomic>
#include <thread>
#include <vector>

#include "../../include/sme.h"

#define SME_API extern "C" __attribute__((visibility("default")))

namespace sme {
void set_error(const char* fmt, ...);
}

namespace {

typedef unsigned __int128 u128;

constexpr u128 kMult = ((u128)2549297995355413924ULL << 64) | (u128)4865540595714422341ULL;

struct Pcg64 {
  u128 state, inc;
  bool has32;
  uint32_t buf32;

  inline uint64_t next64() {
    state = state * kMult + inc;
    const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
    const unsigned rot = (unsigned)(hi >> 58);
    const uint64_t x = hi ^ lo;
    return (x >> rot) | (x << ((64u - rot) & 63u));
  }
  inline uint32_t next32() {
    if (has32) {
      has32 = false;
      return buf32;
    }
    const uint64_t v = next64();
    has32 = true;
    buf32 = (uint32_t)(v >> 32);
    return (uint32_t)v;
  }
  // random_interval(max) for 0 < max <= 0xFFFFFFFF
  inline uint32_t interval(uint32_t max) {
    uint32_t mask = max;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    uint32_t v;
    while ((v = (next32() & mask)) > max) {
    }
    return v;
  }
};

Pcg64 load_state(const uint64_t* st) {
  Pcg64 g;
  g.state = ((u128)st[0] << 64) | st[1];
  g.inc = ((u128)st[2] << 64) | st[3];
  g.has32 = st[4] != 0;
  g.buf32 = (uint32_t)st[5];
  return g;
}

void store_state(const Pcg64& g, uint64_t* st) {
  st[0] = (uint64_t)(g.state >> 64);
  st[1] = (uint64_t)g.state;
  st[2] = (uint64_t)(g.inc >> 64);
  st[3] = (uint64_t)g.inc;
  st[4] = g.has32 ? 1 : 0;
  st[5] = g.buf32;  // numpy keeps the stale half after consuming it
}

// state after `delta` more steps of the LCG (Brown's O(log delta) jump-ahead)
inline u128 advance(u128 state, u128 inc, uint64_t delta) {
  u128 acc_mult = 1, acc_plus = 0, cur_mult = kMult, cur_plus = inc;
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

inline uint64_t xsl_rr(u128 state) {
  const uint64_t hi = (uint64_t)(state >> 64), lo = (uint64_t)state;
  const unsigned rot = (unsigned)(hi >> 58);
  const uint64_t x = hi ^ lo;
  return (x >> rot) | (x << ((64u - rot) & 63u));
}

constexpr int kAhead = 32;           // swaps prefetched ahead
constexpr int64_t kBlock = 1 << 16;  // swap partners per producer block
constexpr int kRing = 8;             // producer blocks in flight

// swaps of steps i = hi, hi-1, ..., lo (j[k] is the partner of step hi - k)
inline void swap_run(int32_t* a, const uint32_t* j, int64_t hi, int64_t lo) {
  const int64_t m = hi - lo + 1;
  for (int64_t k = 0; k < m; ++k) {
    if (k + kAhead < m) __builtin_prefetch(a + j[k + kAhead], 1, 0);
    const int64_t i = hi - k;
    const int32_t t = a[i];
    a[i] = a[j[k]];
    a[j[k]] = t;
  }
}

}  // namespace

// st[6] = {state_hi, state_lo, inc_hi, inc_lo, has_uint32, uinteger} (numpy
// PCG64.state), updated in place to the state after the shuffle.
SME_API int sme_host_pcg64_permutation(uint64_t* st, int64_t n, int32_t* h_out) {
  if (!st || !h_out || n < 1 || n > INT32_MAX) {
    sme::set_error("sme_host_pcg64_permutation: bad arguments (n=%lld)", (long long)n);
    return SME_EINVAL;
  }
  Pcg64 g = load_state(st);
  // The swap partners are uniform over the whole array: with 4 KiB pages nearly
  // every one is also a TLB miss (which software prefetch does not hide).  Ask
  // for transparent huge pages on the (not yet touched) buffer before filling it.
  {
    const uintptr_t a = ((uintptr_t)h_out + (2u << 20) - 1) & ~(uintptr_t)((2u << 20) - 1);
    const uintptr_t b = ((uintptr_t)(h_out + n)) & ~(uintptr_t)((2u << 20) - 1);
    if (b > a) madvise((void*)a, b - a, MADV_HUGEPAGE);  // advisory; failure is harmless
  }
  for (int64_t i = 0; i < n; ++i) h_out[i] = (int32_t)i;
  const int64_t steps = n - 1;  // i = n-1 .. 1
  if (steps <= 4 * kBlock) {
    std::vector<uint32_t> j((size_t)steps);
    for (int64_t k = 0; k < steps; ++k) j[k] = g.interval((uint32_t)(n - 1 - k));
    if (steps > 0) swap_run(h_out, j.data(), n - 1, 1);
  } else {
    // Two-stage pipeline: a producer thread draws the swap partners (the PCG64
    // chain with its rejection loop, ~12 ns per step) block by block into a
    // ring; this thread applies the swaps of finished blocks with prefetching
    // (memory-bound).  The draw order — hence every bit of the output — is
    // numpy's; only the swaps wait for their block.
    const int64_t n_blocks = (steps + kBlock - 1) / kBlock;
    std::vector<uint32_t> ring((size_t)kRing * kBlock);
    std::atomic<int64_t> produced{0}, consumed{0};
    std::thread producer([&] {
      for (int64_t b = 0; b < n_blocks; ++b) {
        while (b - consumed.load(std::memory_order_acquire) >= kRing) std::this_thread::yield();
        uint32_t* j = ring.data() + (size_t)(b % kRing) * kBlock;
        const int64_t hi = n - 1 - b * kBlock, lo = std::max<int64_t>(1, hi - kBlock + 1);
        for (int64_t i = hi; i >= lo; --i) j[hi - i] = g.interval((uint32_t)i);
        produced.store(b + 1, std::memory_order_release);
      }
    });
    for (int64_t b = 0; b < n_blocks; ++b) {
      while (produced.load(std::memory_order_acquire) <= b) std::this_thread::yield();
      const int64_t hi = n - 1 - b * kBlock, lo = std::max<int64_t>(1, hi - kBlock + 1);
      swap_run(h_out, ring.data() + (size_t)(b % kRing) * kBlock, hi, lo);
      consumed.store(b + 1, std::memory_order_release);
    }
    producer.join();
  }
  store_state(g, st);
  return SME_OK;
}

// The swap partners of Generator(PCG64).permutation(n) without the swaps:
// h_j[i] = random_interval(i) for i = n-1 .. 1 in numpy's draw order (h_j[0] = 0),
// st updated exactly as the full shuffle leaves it.  The raw 64-bit outputs are
// produced in parallel, already split into numpy's uint32 order (low half, then
// the buffered high half), each thread jumping ahead to its share of a block with
// the LCG's O(log k) advance; one sequential pass then replays the masked
// rejection over that uint32 stream.  The swaps themselves run on the GPU
// (sme_fy_apply).
SME_API int sme_host_pcg64_swap_partners(uint64_t* st, int64_t n, uint32_t* h_j, int threads) {
  if (!st || !h_j || n < 1 || n > INT32_MAX) {
    sme::set_error("sme_host_pcg64_swap_partners: bad arguments (n=%lld)", (long long)n);
    return SME_EINVAL;
  }
  Pcg64 g = load_state(st);
  h_j[0] = 0;
  if (n == 1) return SME_OK;
  const int T = threads > 0 ? threads : (int)std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
  // 64-bit outputs per block (the draws consume about 1.3 n uint32, so small n get a small block)
  const int64_t kOut = std::min<int64_t>(1 << 20, std::max<int64_t>(1024, n));
  // two blocks: the workers fill the next while this thread replays the current one
  std::vector<uint32_t> ubuf[2] = {std::vector<uint32_t>((size_t)(2 * kOut + 1)),
                                   std::vector<uint32_t>((size_t)(2 * kOut + 1))};
  auto gen_block = [&](uint32_t* out, u128 b0, int64_t off) {
    auto body = [&, out, b0, off](int t) {
      const int64_t a0 = kOut * t / T, e0 = kOut * (t + 1) / T;
      u128 x = advance(b0, g.inc, (uint64_t)a0);
      for (int64_t k = a0; k < e0; ++k) {
        x = x * kMult + g.inc;
        const uint64_t v = xsl_rr(x);
        out[off + 2 * k] = (uint32_t)v;
        out[off + 2 * k + 1] = (uint32_t)(v >> 32);
      }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T; ++t) th.emplace_back(body, t);
    body(0);
    for (auto& x : th) x.join();
  };
  u128 next_base = g.state;              // state before the next block's first output
  int cur = 0;
  std::thread bg;                        // generates block `blocks` into ubuf[cur ^ 1]
  auto prefetch = [&]() {
    const u128 b0 = next_base;
    uint32_t* out = ubuf[cur ^ 1].data();
    bg = std::thread([&gen_block, out, b0] { gen_block(out, b0, 0); });
    next_base = advance(next_base, g.inc, (uint64_t)kOut);
  };
  // the first block, with a pending buffered half (numpy's has_uint32) in front
  const int64_t lead = g.has32 ? 1 : 0;
  if (lead) ubuf[0][0] = g.buf32;
  gen_block(ubuf[0].data(), next_base, lead);
  next_base = advance(next_base, g.inc, (uint64_t)kOut);
  int64_t blocks = 1;                    // blocks replayed so far (the current one included)
  const uint32_t* u = ubuf[0].data();
  int64_t d = 0, d_end = lead + 2 * kOut;  // read position / end in u
  prefetch();
  auto refill = [&]() {
    bg.join();
    cur ^= 1;
    u = ubuf[cur].data();
    d = 0;
    d_end = 2 * kOut;
    ++blocks;
    prefetch();
  };
  int64_t i = n - 1;
  while (i >= 1) {
    uint32_t mask = (uint32_t)i;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    const int64_t i_lo = (int64_t)(mask >> 1);  // the mask holds for i in (mask / 2, i]
    // branch-free rejection: every draw is written to h_j[i]; a rejected one is
    // overwritten by the next draw for the same i, an accepted one moves i on
    while (i > i_lo) {
      if (d_end - d >= 8 && i - 8 > i_lo) {
        // 8 draws with no bounds checks: at most 8 acceptances keep i above i_lo
        // (the mask holds) and the block holds 8 more values
#pragma GCC unroll 8
        for (int k = 0; k < 8; ++k) {
          const uint32_t v = u[d + k] & mask;
          h_j[i] = v;
          i -= (int64_t)(v <= (uint32_t)i);
        }
        d += 8;
        continue;
      }
      if (d == d_end) refill();
      const uint32_t v = u[d++] & mask;
      h_j[i] = v;
      i -= (int64_t)(v <= (uint32_t)i);
    }
  }
  bg.join();  // the block prefetched last is not needed
  // uint32 values consumed in total (the pending half counts as one), and where they
  // leave numpy's buffer: an odd number of fresh halves means a high half is pending
  const int64_t total_fresh = (blocks - 1) * 2 * kOut + (d - (blocks == 1 ? lead : 0));
  const int64_t outputs = (total_fresh + 1) / 2;
  g.state = advance(g.state, g.inc, (uint64_t)outputs);
  if (total_fresh > 0) {
    g.has32 = (total_fresh & 1) != 0;
    g.buf32 = (uint32_t)(xsl_rr(g.state) >> 32);  // the high half of the last output drawn
  } else {
    g.has32 = false;  // only the pending half was used (or nothing)
  }
  store_state(g, st);
  return SME_OK;
}
