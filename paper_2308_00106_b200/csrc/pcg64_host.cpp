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
#include <mutex>
#include <thread>
#include <vector>

#include <cuda_runtime.h>

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

namespace {

// numpy's uint32 stream of one PCG64 (low half of each 64-bit output, then the
// buffered high half), produced in blocks by T threads that each jump ahead to their
// share with the LCG's O(log k) advance; double-buffered, so the workers fill the
// next block while the caller consumes the current one.
class U32Stream {
 public:
  U32Stream(const Pcg64& g, int64_t n, int threads) : g_(g) {
    T_ = threads > 0 ? threads : (int)std::max(1u, std::min(8u, std::thread::hardware_concurrency()));
    // 64-bit outputs per block (the draws consume about 1.3 n uint32: small n, small block)
    kOut_ = std::min<int64_t>(1 << 20, std::max<int64_t>(1024, n));
    for (auto& b : buf_) b.resize((size_t)(2 * kOut_ + 1));
    next_base_ = g.state;
    lead_ = g.has32 ? 1 : 0;  // a pending buffered half (numpy's has_uint32) comes first
    if (lead_) buf_[0][0] = g.buf32;
    gen_block(buf_[0].data(), next_base_, lead_);
    next_base_ = advance(next_base_, g.inc, (uint64_t)kOut_);
    u = buf_[0].data();
    d = 0;
    d_end = lead_ + 2 * kOut_;
    prefetch();
  }
  ~U32Stream() {
    if (bg_.joinable()) bg_.join();
  }
  const uint32_t* u;  // current block
  int64_t d, d_end;   // read position / end in u

  void refill() {
    bg_.join();
    cur_ ^= 1;
    u = buf_[cur_].data();
    d = 0;
    d_end = 2 * kOut_;
    ++blocks_;
    prefetch();
  }
  // the generator state after the values consumed so far (numpy's, exactly)
  void final_state(Pcg64& g) {
    if (bg_.joinable()) bg_.join();  // the block prefetched last is not needed
    // uint32 values consumed in total (the pending half counts as one), and where they
    // leave numpy's buffer: an odd number of fresh halves means a high half is pending
    const int64_t total_fresh = (blocks_ - 1) * 2 * kOut_ + (d - (blocks_ == 1 ? lead_ : 0));
    const int64_t outputs = (total_fresh + 1) / 2;
    g.state = advance(g_.state, g_.inc, (uint64_t)outputs);
    if (total_fresh > 0) {
      g.has32 = (total_fresh & 1) != 0;
      g.buf32 = (uint32_t)(xsl_rr(g.state) >> 32);  // the high half of the last output drawn
    } else {
      g.has32 = g_.has32 && d == 0;  // only the pending half was used (or nothing)
    }
  }

 private:
  void gen_block(uint32_t* out, u128 b0, int64_t off) {
    auto body = [&, out, b0, off](int t) {
      const int64_t a0 = kOut_ * t / T_, e0 = kOut_ * (t + 1) / T_;
      u128 x = advance(b0, g_.inc, (uint64_t)a0);
      for (int64_t k = a0; k < e0; ++k) {
        x = x * kMult + g_.inc;
        const uint64_t v = xsl_rr(x);
        out[off + 2 * k] = (uint32_t)v;
        out[off + 2 * k + 1] = (uint32_t)(v >> 32);
      }
    };
    std::vector<std::thread> th;
    for (int t = 1; t < T_; ++t) th.emplace_back(body, t);
    body(0);
    for (auto& x : th) x.join();
  }
  void prefetch() {
    const u128 b0 = next_base_;
    uint32_t* out = buf_[cur_ ^ 1].data();
    bg_ = std::thread([this, out, b0] { gen_block(out, b0, 0); });
    next_base_ = advance(next_base_, g_.inc, (uint64_t)kOut_);
  }
  const Pcg64 g_;  // the state before the first value
  int T_;
  int64_t kOut_, lead_, blocks_ = 1;
  std::vector<uint32_t> buf_[2];
  int cur_ = 0;
  u128 next_base_;
  std::thread bg_;
};

// numpy's masked-rejection replay over the stream: for i = n-1 .. 1, draw
// v = next_uint32 & mask(i) until v <= i, and h[i] = v.  Branch-free: every draw is
// written to h[i]; a rejected one is overwritten by the next draw for the same i, an
// accepted one moves i on.  Indices are written into `sink` slots: h = sink.base
// (indexed by i) holds [sink.lo, ...); when i drops below sink.lo, everything from
// sink.lo up is final and sink.next(i) hands over the next slot.
template <class Sink>
void replay(U32Stream& us, int64_t n, Sink& sink) {
  int64_t i = n - 1;
  uint32_t* h = sink.base;
  int64_t lo = sink.lo;
  while (i >= 1) {
    uint32_t mask = (uint32_t)i;
    mask |= mask >> 1;
    mask |= mask >> 2;
    mask |= mask >> 4;
    mask |= mask >> 8;
    mask |= mask >> 16;
    const int64_t i_lo = (int64_t)(mask >> 1);  // the mask holds for i in (mask / 2, i]
    while (i > i_lo) {
      if (i < lo) {
        sink.next(i);
        h = sink.base;
        lo = sink.lo;
      }
      const int64_t stop = std::max(i_lo, lo - 1);  // i stays above: same mask, same slot
      if (us.d_end - us.d >= 8 && i - 8 > stop) {
        // 8 draws with no bounds checks
#pragma GCC unroll 8
        for (int k = 0; k < 8; ++k) {
          const uint32_t v = us.u[us.d + k] & mask;
          h[i] = v;
          i -= (int64_t)(v <= (uint32_t)i);
        }
        us.d += 8;
        continue;
      }
      if (us.d == us.d_end) us.refill();
      const uint32_t v = us.u[us.d++] & mask;
      h[i] = v;
      i -= (int64_t)(v <= (uint32_t)i);
    }
  }
  if (lo > 0) {  // the last acceptance left the slot holding index 1
    sink.next(0);
    h = sink.base;
  }
  h[0] = 0;
  sink.finish();
}

struct HostSink {  // one slot: the whole array
  uint32_t* base;
  int64_t lo = 0;
  void next(int64_t) {}
  void finish() {}
};

// Pinned staging ring of the device-streaming variant: slots of kSlot indices, each
// copied to the device (cudaMemcpyAsync) as soon as the replay has moved below it.
constexpr int kSlots = 4;
constexpr int64_t kSlot = 1 << 20;

struct Ring {
  uint32_t* host = nullptr;  // kSlots * kSlot pinned
  cudaEvent_t ev[kSlots] = {};
};
std::mutex g_ring_mu;
std::vector<Ring*> g_rings;  // free rings (a process keeps a few; concurrent calls take one each)

struct DeviceSink {
  Ring* ring;
  int32_t* d_j;
  cudaStream_t s;
  int64_t n;
  uint32_t* base = nullptr;
  int64_t lo = 0, hi = 0;
  int slot = -1;
  bool used[kSlots] = {};
  cudaError_t err = cudaSuccess;

  void open_slot() {  // the slot for [lo, hi) with hi = the previous lo
    slot = (slot + 1) % kSlots;
    if (used[slot] && err == cudaSuccess) err = cudaEventSynchronize(ring->ev[slot]);  // its last copy is done
    lo = std::max<int64_t>(0, hi - kSlot);
    base = ring->host + (int64_t)slot * kSlot - lo;
  }
  void flush() {
    if (err == cudaSuccess)
      err = cudaMemcpyAsync(d_j + lo, base + lo, (size_t)(hi - lo) * 4, cudaMemcpyHostToDevice, s);
    if (err == cudaSuccess) err = cudaEventRecord(ring->ev[slot], s);
    used[slot] = true;
  }
  void start() {
    hi = n;
    slot = -1;
    open_slot();
  }
  void next(int64_t i) {  // i < lo: [lo, hi) is final
    while (i < lo) {
      flush();
      hi = lo;
      open_slot();
    }
  }
  void finish() {  // i = 0 and h[0] written: [0, hi) is final
    flush();
    if (err == cudaSuccess) err = cudaStreamSynchronize(s);
  }
};

}  // namespace

// The swap partners of Generator(PCG64).permutation(n) without the swaps:
// h_j[i] = random_interval(i) for i = n-1 .. 1 in numpy's draw order (h_j[0] = 0),
// st updated exactly as the full shuffle leaves it.  The raw outputs come from
// U32Stream (parallel, double-buffered); one sequential pass replays the masked
// rejection.  The swaps themselves run on the GPU (sme_fy_apply).
SME_API int sme_host_pcg64_swap_partners(uint64_t* st, int64_t n, uint32_t* h_j, int threads) {
  if (!st || !h_j || n < 1 || n > INT32_MAX) {
    sme::set_error("sme_host_pcg64_swap_partners: bad arguments (n=%lld)", (long long)n);
    return SME_EINVAL;
  }
  Pcg64 g = load_state(st);
  h_j[0] = 0;
  if (n == 1) return SME_OK;
  U32Stream us(g, n, threads);
  HostSink sink{h_j};
  replay(us, n, sink);
  us.final_state(g);
  store_state(g, st);
  return SME_OK;
}

// The same partners written straight to DEVICE memory d_j (int32[n]): the replay fills
// a small pinned ring and each 4 MB slot is copied with cudaMemcpyAsync on `stream` as
// soon as the replay has moved below it, so the upload hides behind the draws and no
// n-sized host buffer is touched.  Returns after the copies have completed.
SME_API int sme_pcg64_swap_partners_to_device(uint64_t* st, int64_t n, int32_t* d_j, int threads,
                                              sme_stream_t stream) {
  if (!st || !d_j || n < 1 || n > INT32_MAX) {
    sme::set_error("sme_pcg64_swap_partners_to_device: bad arguments (n=%lld)", (long long)n);
    return SME_EINVAL;
  }
  Ring* ring = nullptr;
  {
    std::lock_guard<std::mutex> lk(g_ring_mu);
    if (!g_rings.empty()) {
      ring = g_rings.back();
      g_rings.pop_back();
    }
  }
  if (!ring) {
    ring = new Ring;
    cudaError_t e = cudaHostAlloc((void**)&ring->host, (size_t)kSlots * kSlot * 4, cudaHostAllocDefault);
    for (int k = 0; k < kSlots && e == cudaSuccess; ++k) e = cudaEventCreateWithFlags(&ring->ev[k], cudaEventDisableTiming);
    if (e != cudaSuccess) {
      sme::set_error("sme_pcg64_swap_partners_to_device: %s", cudaGetErrorString(e));
      delete ring;  // (a partially created ring leaks its pinned block on this error path only)
      return SME_ECUDA;
    }
  }
  Pcg64 g = load_state(st);
  DeviceSink sink{ring, d_j, (cudaStream_t)stream, n};
  sink.start();
  if (n == 1) {
    sink.base[0] = 0;
    sink.finish();
  } else {
    U32Stream us(g, n, threads);
    replay(us, n, sink);
    us.final_state(g);
  }
  const cudaError_t err = sink.err;
  {
    std::lock_guard<std::mutex> lk(g_ring_mu);
    g_rings.push_back(ring);
  }
  if (err != cudaSuccess) {
    sme::set_error("sme_pcg64_swap_partners_to_device: %s", cudaGetErrorString(err));
    return SME_ECUDA;
  }
  store_state(g, st);
  return SME_OK;
}
