// The three isolated primitives of the reference's microbenchmarks
// (reference src/bench.py:244-300 `microbench`), on device-resident buffers:
//
//   f4b_dict_build  radix_sort + unique_sorted of W-word keys
//                   (bulk.py:86-124, :135-150): an L2-resident hash table
//                   drops the duplicates first (when the distinct keys fit),
//                   the words are packed into one
//                   order-isomorphic device key of W * key_bits bits (reference
//                   keys are 48-bit words, bench.py:237-241), sorted with the
//                   one-sweep LSD radix sort of radix.cu (W * key_bits / 8
//                   passes instead of the reference's 8 W), uniqued and
//                   unpacked back to W words.
//   f4b_join_index  merge_join_index (bulk.py:207-241): position of each key in
//                   an ascending dictionary, MissingKeyError on a miss.
//   f4b_mod_fma     acc + a b mod p, the KernelArith lazy multiply-add
//                   (fp.py:335-400), here with a 64-bit Barrett reduction.
//
// All three are HBM-bound streams; the roofline is the copy bandwidth.
#include <algorithm>
#include <cmath>
#include <cstdlib>

#include "block.cuh"
#include "common.cuh"
#include "engine.h"

namespace f4b {

static constexpr int MB_THREADS = 256;

// Pack W <= 2 words of `kb` significant bits into one Key<2> (big-endian
// words): value = w0 * 2^kb + w1 (W = 2) or w0 (W = 1, stored in w[1]).
__global__ void __launch_bounds__(MB_THREADS) k_mb_pack(const u64* __restrict__ in, long long n, int words, int kb,
                                                        u64* __restrict__ out, u32* __restrict__ err) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const u64 lim = kb >= 64 ? ~0ull : ((1ull << kb) - 1);
  bool bad = false;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    u64 hi = 0, lo;
    if (words == 2) {
      const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(in) + i);
      bad |= (v.x > lim) | (v.y > lim);
      lo = kb >= 64 ? v.y : (v.y | (v.x << kb));
      hi = kb >= 64 ? v.x : (kb == 0 ? 0 : (v.x >> (64 - kb)));
    } else {
      lo = __ldcs(in + i);
      bad |= lo > lim;
    }
    __stcs(reinterpret_cast<ulonglong2*>(out) + i, make_ulonglong2(hi, lo));
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

__global__ void __launch_bounds__(MB_THREADS) k_mb_unpack(const u64* __restrict__ in, const u32* __restrict__ d_n,
                                                          int words, int kb, u64* __restrict__ out) {
  const long long n = *d_n;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const u64 lim = kb >= 64 ? ~0ull : ((1ull << kb) - 1);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    const ulonglong2 v = reinterpret_cast<const ulonglong2*>(in)[i];
    if (words == 2) {
      const u64 w1 = v.y & lim;
      const u64 w0 = kb >= 64 ? v.x : ((v.y >> kb) | (kb == 0 ? 0 : (v.x << (64 - kb))));
      reinterpret_cast<ulonglong2*>(out)[i] = make_ulonglong2(w0, w1);
    } else {
      out[i] = v.y;
    }
  }
}

// Duplicate filter in front of the sort (dict_build): every key is inserted
// into an open-addressing table of packed 128-bit keys small enough to stay
// in L2 (<= 64 MB); the first inserter of a key appends it to a compact list,
// so only the distinct keys go through the radix sort.  Keys are packed on the
// fly (no separate pack pass).  More distinct keys than `limit` -> overflow
// flag, the caller falls back to sorting every key.
static constexpr int HB_LOG_MAX = 22;  // 64 MB table: L2 resident (2^25 measured: 16M keys at 50% duplicates 3.9 -> 3.4 ms, at 99% 0.46 -> 0.73 ms)
using u128 = unsigned __int128;

F4B_DEV u32 mb_hash(u64 hi, u64 lo, int logc) {
  const u64 h = (lo * 0x9E3779B97F4A7C15ull) ^ (hi * 0xC2B2AE3D27D4EB4Full) ^ (lo >> 29);
  return (u32)((h * 0xBF58476D1CE4E5B9ull) >> (64 - logc));
}

__global__ void __launch_bounds__(MB_THREADS) k_mb_hash_insert(const u64* __restrict__ in, long long n, int words,
                                                               int kb, u128* __restrict__ table, int logc, u32 limit,
                                                               u64* __restrict__ uniq, u32* __restrict__ d_count,
                                                               u32* __restrict__ err) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const u64 lim = kb >= 64 ? ~0ull : ((1ull << kb) - 1);  // W = 2 implies kb < 64 here
  const u32 mask = (1u << logc) - 1;
  const u128 EMPTY = ~(u128)0;
  const int lane = threadIdx.x & 31;
  bool bad = false;
  const long long n_round = (n + 31) / 32 * 32;  // whole warps iterate together (ballots)
  constexpr int HB_ITEMS = 4;  // keys per thread per iteration: four table probes in flight (8: 98 registers, 168 -> 245 us)
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n_round; i0 += HB_ITEMS * stride) {
    // overflow: the caller sorts everything (warp-uniform exit: ballots below)
    if (__shfl_sync(0xffffffffu, lane == 0 ? ld_volatile(err) : 0u, 0) & 2u) break;
    u64 hi[HB_ITEMS], lo[HB_ITEMS];
    u32 h[HB_ITEMS];
    ulonglong2 cur[HB_ITEMS];
#pragma unroll
    for (int k = 0; k < HB_ITEMS; ++k) {
      const long long i = i0 + k * stride;
      hi[k] = 0;
      lo[k] = 0;
      if (i < n) {
        if (words == 2) {
          const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(in) + i);
          bad |= (v.x > lim) | (v.y > lim);
          lo[k] = v.y | (v.x << kb);
          hi[k] = v.x >> (64 - kb);
        } else {
          lo[k] = __ldcs(in + i);
          bad |= lo[k] > lim;
        }
      }
    }
#pragma unroll
    for (int k = 0; k < HB_ITEMS; ++k) {
      h[k] = mb_hash(hi[k], lo[k], logc);
      if (i0 + k * stride < n) cur[k] = __ldcg(reinterpret_cast<const ulonglong2*>(table) + h[k]);
    }
#pragma unroll
    for (int k = 0; k < HB_ITEMS; ++k) {
      bool ins = false;
      if (i0 + k * stride < n) {
        const u128 key = ((u128)hi[k] << 64) | lo[k];
        u32 hh = h[k];
        u128 c = ((u128)cur[k].y << 64) | cur[k].x;
        for (;;) {
          if (c == key) break;
          if (c == EMPTY) {
            const u128 old = atomicCAS(table + hh, EMPTY, key);
            if (old == EMPTY) {
              ins = true;
              break;
            }
            if (old == key) break;
          }
          hh = (hh + 1) & mask;
          const ulonglong2 c2 = __ldcg(reinterpret_cast<const ulonglong2*>(table) + hh);
          c = ((u128)c2.y << 64) | c2.x;
        }
      }
      const unsigned m = __ballot_sync(0xffffffffu, ins);
      if (m) {
        u32 base = 0;
        if (lane == __ffs(m) - 1) base = atomicAdd(d_count, (u32)__popc(m));
        base = __shfl_sync(0xffffffffu, base, __ffs(m) - 1);
        if (ins) {
          const u32 o = base + __popc(m & lanemask_lt());
          if (o < limit) reinterpret_cast<ulonglong2*>(uniq)[o] = make_ulonglong2(hi[k], lo[k]);
        }
        if (lane == 0 && base + __popc(m) > limit) atomicOr(err, 2u);
      }
    }
  }
  if (__any_sync(0xffffffffu, bad) && lane == 0) atomicOr(err, 1u);
}

// Lower bound of each query in an ascending W-word dictionary.  Queries of a
// warp are usually close in key order (row segments are sorted), so the
// upper levels of the search are shared L1/L2 hits.  (Narrowing each warp's
// range to [lb(min query), lb(max query)] first was measured 2x slower at 16M
// queries: the kernel is bound by the dependent-load chain, not by requests;
// four branch-free searches in lockstep per thread: 1.8x slower as well.)
template <int KW>
__global__ void __launch_bounds__(MB_THREADS) k_mb_join(const u64* __restrict__ dict, u32 nd,
                                                        const u64* __restrict__ q, long long n,
                                                        long long* __restrict__ pos, u32* __restrict__ err) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  bool miss = false;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride) {
    Key<KW> k;
#pragma unroll
    for (int j = 0; j < KW; ++j) k.w[j] = __ldcs(q + i * KW + j);
    u32 lo = 0, hi = nd;
    while (lo < hi) {
      const u32 mid = (lo + hi) >> 1;
      Key<KW> m;
#pragma unroll
      for (int j = 0; j < KW; ++j) m.w[j] = __ldg(dict + (size_t)mid * KW + j);
      if (key_lt<KW>(m, k)) lo = mid + 1; else hi = mid;
    }
    bool hit = lo < nd;
    if (hit) {
#pragma unroll
      for (int j = 0; j < KW; ++j) hit &= __ldg(dict + (size_t)lo * KW + j) == k.w[j];
    }
    miss |= !hit;
    __stcs(pos + i, (long long)lo);
  }
  if (__any_sync(0xffffffffu, miss) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

// out = (acc + a b) mod p, p < 2^31, inputs < 2^31 (a b + acc < 2^63).
// Barrett with mu = floor((2^64 - 1) / p): the quotient estimate is short by
// at most 2.
F4B_DEV u64 mb_reduce(u64 x, u64 p, u64 mu) {
  u64 r = x - __umul64hi(x, mu) * p;
  r = r >= p ? r - p : r;
  return r >= p ? r - p : r;
}

__global__ void __launch_bounds__(MB_THREADS) k_mb_fma(const u64* __restrict__ a, const u64* __restrict__ b,
                                                       const u64* __restrict__ acc, long long n, u64 p, u64 mu,
                                                       u64* __restrict__ out) {
  const long long n2 = n / 2;
  const long long stride = (long long)gridDim.x * blockDim.x;
  const ulonglong2* a2 = reinterpret_cast<const ulonglong2*>(a);
  const ulonglong2* b2 = reinterpret_cast<const ulonglong2*>(b);
  const ulonglong2* c2 = reinterpret_cast<const ulonglong2*>(acc);
  ulonglong2* o2 = reinterpret_cast<ulonglong2*>(out);
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n2; i += stride) {
    const ulonglong2 x = __ldcs(a2 + i), y = __ldcs(b2 + i), z = __ldcs(c2 + i);
    __stcs(o2 + i, make_ulonglong2(mb_reduce(z.x + x.x * y.x, p, mu), mb_reduce(z.y + x.y * y.y, p, mu)));
  }
  if ((n & 1) && blockIdx.x == 0 && threadIdx.x == 0)
    out[n - 1] = mb_reduce(acc[n - 1] + a[n - 1] * b[n - 1], p, mu);
}

static unsigned mb_grid(Ctx* c, long long n) {
  const long long want = (n + MB_THREADS - 1) / MB_THREADS;
  return (unsigned)std::max<long long>(1, std::min<long long>(want, (long long)c->num_sms * 8));
}

long long dict_build(Ctx* c, const uint64_t* keys, long long n, int words, int key_bits, uint64_t* out) {
  if (n < 0 || n >= (1ll << 32) - 2 || (words != 1 && words != 2) || key_bits < 1 || key_bits > 64)
    fail(F4B_ERR_PRECONDITION, "dict_build: 0 <= n < 2^32 - 2, words in {1, 2}, 1 <= key_bits <= 64");
  if (n == 0) return 0;
  DBuf packed, uniq, flags;
  ensure(c, flags, 16);
  u32* err = flags.as<u32>();
  u32* d_count = err + 1;
  u32* d_hcount = err + 2;
  memset_async(c, err, 0, 12);
  // duplicate filter first (distinct keys expected <= half the L2-sized
  // table); packed keys with all 128 bits significant would collide with the
  // empty-slot marker, so they always take the full sort
  bool filtered = false;
  if (!c->opt_dict_nohash && words * key_bits < 128) {
    int logc = 10;
    while (logc < HB_LOG_MAX && (1ll << logc) < 2 * n) ++logc;
    const u32 limit = 1u << (logc - 1);
    DBuf table;
    ensure(c, table, (size_t)16 << logc);
    ensure(c, packed, (size_t)limit * 16);
    memset_async(c, table.p, 0xFF, (size_t)16 << logc);
    // a leading sample first: if its distinct count extrapolates (uniform
    // picks from a pool of P keys: d = P (1 - e^{-S/P})) to more distinct keys
    // than the table takes, skip the filter instead of running into the
    // overflow (measured 0.27 ms wasted at 16M keys / 50 % duplicates).  Only
    // the speed depends on this guess; the result never does.
    const long long S = std::min<long long>(n, 1ll << 18);
    F4B_LAUNCH(c, k_mb_hash_insert, mb_grid(c, S), MB_THREADS, 0, keys, S, words, key_bits, table.as<u128>(), logc,
               limit, packed.as<u64>(), d_hcount, err);
    bool give_up = false;
    if (S < n) {
      const double d = (double)read_u32(c, d_hcount);
      double P = 1e18;  // all distinct: unbounded pool
      if (d < (double)S) {  // solve P (1 - exp(-S/P)) = d by bisection on log P
        double lo = std::log(std::max(d, 1.0)), hi = std::log(1e18);
        for (int it = 0; it < 80; ++it) {
          const double mid = 0.5 * (lo + hi), Pm = std::exp(mid);
          if (Pm * -std::expm1(-(double)S / Pm) < d) lo = mid; else hi = mid;
        }
        P = std::exp(0.5 * (lo + hi));
      }
      const double n_est = P * -std::expm1(-(double)n / P);
      give_up = n_est > 0.9 * (double)limit;
      if (!give_up)
        F4B_LAUNCH(c, k_mb_hash_insert, mb_grid(c, n - S), MB_THREADS, 0, keys + (size_t)S * words, n - S, words,
                   key_bits, table.as<u128>(), logc, limit, packed.as<u64>(), d_hcount, err);
    }
    const u32 e = read_u32(c, err) | (give_up ? 2u : 0u);
    release(c, table);
    if (e & 1u) {
      release(c, packed);
      release(c, flags);
      fail(F4B_ERR_PRECONDITION, "dict_build: a key word has more than key_bits significant bits");
    }
    if (!(e & 2u)) {
      const u32 nd = read_u32(c, d_hcount);
      ensure(c, uniq, (size_t)(nd + 1) * 16);
      sort_unique(c, 2, packed.as<u64>(), nullptr, nd, words * key_bits, nullptr, nullptr, uniq.as<u64>(), d_count);
      filtered = true;
    } else {
      memset_async(c, err, 0, 12);
    }
  }
  if (!filtered) {
    ensure(c, packed, (size_t)n * 16);
    ensure(c, uniq, (size_t)(n + 1) * 16);
    F4B_LAUNCH(c, k_mb_pack, mb_grid(c, n), MB_THREADS, 0, keys, n, words, key_bits, packed.as<u64>(), err);
    sort_unique(c, 2, packed.as<u64>(), nullptr, (u32)n, words * key_bits, nullptr, nullptr, uniq.as<u64>(),
                d_count);
  }
  F4B_LAUNCH(c, k_mb_unpack, mb_grid(c, n), MB_THREADS, 0, uniq.as<u64>(), d_count, words, key_bits, out);
  const u32 bad = read_u32(c, err);
  const long long nu = read_u32(c, d_count);
  release(c, packed);
  release(c, uniq);
  release(c, flags);
  if (bad & 1u) fail(F4B_ERR_PRECONDITION, "dict_build: a key word has more than key_bits significant bits");
  return nu;
}

void join_index(Ctx* c, const uint64_t* dict, long long nd, const uint64_t* keys, long long n, int words,
                int64_t* pos) {
  if (n < 0 || nd < 0 || nd >= (1ll << 32) - 1 || words < 1 || words > 4)
    fail(F4B_ERR_PRECONDITION, "join_index: bad sizes");
  if (n == 0) return;
  DBuf flags;
  ensure(c, flags, 16);
  u32* err = flags.as<u32>();
  memset_async(c, err, 0, 4);
  const unsigned g = mb_grid(c, n);
  long long* p = reinterpret_cast<long long*>(pos);
  switch (words) {
    case 1: F4B_LAUNCH(c, k_mb_join<1>, g, MB_THREADS, 0, dict, (u32)nd, keys, n, p, err); break;
    case 2: F4B_LAUNCH(c, k_mb_join<2>, g, MB_THREADS, 0, dict, (u32)nd, keys, n, p, err); break;
    case 3: F4B_LAUNCH(c, k_mb_join<3>, g, MB_THREADS, 0, dict, (u32)nd, keys, n, p, err); break;
    default: F4B_LAUNCH(c, k_mb_join<4>, g, MB_THREADS, 0, dict, (u32)nd, keys, n, p, err); break;
  }
  const u32 miss = read_u32(c, err);
  release(c, flags);
  if (miss) fail(F4B_ERR_MISSING_KEY, "join_index: a key is absent from the dictionary");
}

void mod_fma(Ctx* c, uint32_t p, const uint64_t* a, const uint64_t* b, const uint64_t* acc, long long n,
             uint64_t* out) {
  if (n < 0 || p < 3 || p >= (1u << 31)) fail(F4B_ERR_PRECONDITION, "mod_fma: 3 <= p < 2^31");
  if (n == 0) return;
  if (((uintptr_t)a | (uintptr_t)b | (uintptr_t)acc | (uintptr_t)out) & 15)
    fail(F4B_ERR_PRECONDITION, "mod_fma: buffers must be 16-byte aligned");
  const u64 mu = ~0ull / p;
  F4B_LAUNCH(c, k_mb_fma, mb_grid(c, (n + 1) / 2), MB_THREADS, 0, a, b, acc, n, (u64)p, mu, out);
}

}  // namespace f4b
