// The three isolated primitives of the reference's microbenchmarks
// (reference src/bench.py:244-300 `microbench`), on device-resident buffers:
//
//   f4b_dict_build  radix_sort + unique_sorted of W-word keys
//                   (bulk.py:86-124, :135-150): the words are packed into
//                   one order-isomorphic 128-bit key (reference keys are
//                   48-bit words, bench.py:237-241); an MSD bucket pass
//                   (one global scatter by the top varying bits, then
//                   sub-buckets of ~1 key sorted and deduplicated in shared
//                   memory, written in order through a decoupled look-back)
//                   replaces the reference's 8 W LSD passes.  Skewed inputs
//                   that overflow a bucket take the one-sweep LSD radix sort
//                   of radix.cu (W * key_bits / 8 passes) + unique.
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

// MSD bucket path of dict_build (no hash table: the reference spec rejects
// atomic hash tables; the result is the sorted unique run
// whatever order keys land in a bucket):
//   k_msd_diff    OR of (key XOR key[0]) -> the highest bit where keys differ
//                 (`top`); bits above it are common and carry no order
//   k_msd_hist    bucket sizes of the D1-bit digit just below top
//                 (shared-memory histograms summed into global counts)
//   scan          -> bucket starts
//   k_msd_scatter packed 128-bit keys appended to their buckets (one global
//                 cursor per bucket)
//   k_msd_bucket  one CTA per bucket: keys to registers, scattered in shared
//                 memory by the next D2 bits into sub-buckets of ~1 key,
//                 first occurrences found and ranked inside their
//                 sub-bucket, written back sorted to the front of the
//                 bucket's range; distinct count per bucket
//   scan          -> output offsets (a decoupled look-back chaining the
//                 buckets was measured 30 % of the bucket kernel in barrier
//                 waits: a bucket's predecessor is still sorting)
//   k_msd_compact one warp per bucket: distinct keys unpacked to W words
// A bucket above MSD_CAP keys or a sub-bucket above MSD_SUBLEN keys sets err
// bit 2 and the caller sorts every key with the LSD path instead (skewed
// inputs: only the speed changes).
using u128 = unsigned __int128;
static constexpr int MSD_THREADS = 512;
static constexpr int MSD_BT = 256;       // k_msd_bucket: 4 CTAs per SM
static constexpr int MSD_CAP = 2048;     // keys per bucket in shared memory (~512 expected)
static constexpr int MSD_D2 = 11;        // sub-bucket digit bits (2048 sub-buckets)
static constexpr int MSD_SUBLEN = 1024;  // keys per sub-bucket (~1 expected)

F4B_DEV u128 msd_pack(const u64* __restrict__ in, long long i, int words, int kb, u64 lim, bool& bad) {
  if (words == 2) {
    const ulonglong2 v = __ldcs(reinterpret_cast<const ulonglong2*>(in) + i);
    bad |= (v.x > lim) | (v.y > lim);
    return ((u128)v.x << kb) | (u128)v.y;
  }
  const u64 w = __ldcs(in + i);
  bad |= w > lim;
  return (u128)w;
}

F4B_DEV int msd_top(const u64* diff) {  // bits below and including the highest differing bit
  return diff[0] ? 128 - __clzll((long long)diff[0]) : (diff[1] ? 64 - __clzll((long long)diff[1]) : 0);
}

__global__ void __launch_bounds__(MB_THREADS) k_msd_diff(const u64* __restrict__ in, long long n, int words, int kb,
                                                         u64* __restrict__ diff, u32* __restrict__ err) {
  const u64 lim = kb >= 64 ? ~0ull : ((1ull << kb) - 1);
  bool bad = false;
  const u128 k0 = msd_pack(in, 0, words, kb, lim, bad);
  u128 acc = 0;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    acc |= msd_pack(in, i, words, kb, lim, bad) ^ k0;
  u64 hi = (u64)(acc >> 64), lo = (u64)acc;
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    hi |= __shfl_xor_sync(0xffffffffu, hi, o);
    lo |= __shfl_xor_sync(0xffffffffu, lo, o);
  }
  if ((threadIdx.x & 31) == 0) {
    if (hi) atomicOr(reinterpret_cast<unsigned long long*>(diff), (unsigned long long)hi);
    if (lo) atomicOr(reinterpret_cast<unsigned long long*>(diff) + 1, (unsigned long long)lo);
  }
  if (__any_sync(0xffffffffu, bad) && (threadIdx.x & 31) == 0) atomicOr(err, 1u);
}

F4B_DEV u32 msd_digit(u128 v, int shift, int bits) { return (u32)(v >> shift) & ((1u << bits) - 1u); }

// bucket sizes: shared-memory histogram per CTA, summed into C[nb]
__global__ void __launch_bounds__(MSD_THREADS) k_msd_hist(const u64* __restrict__ in, long long n, int words, int kb,
                                                          int d1, const u64* __restrict__ diff, u32* __restrict__ C) {
  extern __shared__ u32 h[];
  const int nb = 1 << d1;
  for (int i = threadIdx.x; i < nb; i += blockDim.x) h[i] = 0;
  __syncthreads();
  const int s1 = max(msd_top(diff) - d1, 0);
  bool bad = false;
  const long long stride = (long long)gridDim.x * blockDim.x;
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += stride)
    atomicAdd(h + msd_digit(msd_pack(in, i, words, kb, ~0ull, bad), s1, d1), 1u);
  __syncthreads();
  for (int d = threadIdx.x; d < nb; d += blockDim.x)
    if (h[d]) atomicAdd(C + d, h[d]);
}

// keys appended to their bucket through one global cursor per bucket: all
// CTAs extend the same bucket tails at the same time, so the 16-byte stores
// fill whole sectors while they are L2-resident (per-CTA ranges were measured
// 2.7x DRAM read amplification from partial-sector write-backs)
__global__ void __launch_bounds__(MSD_THREADS) k_msd_scatter(const u64* __restrict__ in, long long n, int words,
                                                             int kb, int d1, const u64* __restrict__ diff,
                                                             u32* __restrict__ cur, u128* __restrict__ out) {
  const int s1 = max(msd_top(diff) - d1, 0);
  bool bad = false;
  const long long stride = (long long)gridDim.x * blockDim.x;
  // four keys per thread per iteration: loads and cursor atomics in flight
  for (long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x; i0 < n; i0 += 4 * stride) {
    u128 v[4];
    u32 o[4];
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i0 + k * stride < n) v[k] = msd_pack(in, i0 + k * stride, words, kb, ~0ull, bad);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i0 + k * stride < n) o[k] = atomicAdd(cur + msd_digit(v[k], s1, d1), 1u);
#pragma unroll
    for (int k = 0; k < 4; ++k)
      if (i0 + k * stride < n) out[o[k]] = v[k];
  }
}

// One bucket per CTA:
//   keys -> registers, sub-bucket histogram, scan, scatter into B (shared);
//   phase 1: a key is the first occurrence of its value when no earlier key
//            of its sub-bucket equals it (copies stop at the first compare);
//   phase 2: a first occurrence's rank = number of first occurrences of its
//            sub-bucket below it -> output slot.
// Work per sub-bucket is O(len * distinct); a sub-bucket above MSD_SUBLEN
// keys or a bucket above MSD_CAP keys flags the LSD fallback.
__global__ void __launch_bounds__(MSD_BT, 4) k_msd_bucket(u128* __restrict__ keys, const u32* __restrict__ O, int d1,
                                                          const u64* __restrict__ diff, u32* __restrict__ Dc,
                                                          u32* __restrict__ err) {
  extern __shared__ __align__(16) unsigned char smem[];
  constexpr int NS = 1 << MSD_D2, PER = NS / MSD_BT, KPT = MSD_CAP / MSD_BT;
  u128* B = reinterpret_cast<u128*>(smem);
  u32* C = reinterpret_cast<u32*>(B + MSD_CAP);  // [NS] counts -> cursors -> sub-bucket ends
  u32* D = C + NS;                               // [NS] distinct counts -> output offsets
  u32* F = D + NS;                               // [MSD_CAP / 32] first-occurrence bits
  __shared__ u32 ws[33];
  __shared__ u32 s_bad;
  if (threadIdx.x == 0) s_bad = 0;
  for (int j = threadIdx.x; j < NS; j += blockDim.x) C[j] = D[j] = 0;
  for (int j = threadIdx.x; j < MSD_CAP / 32; j += blockDim.x) F[j] = 0;
  __syncthreads();
  const u32 tile = blockIdx.x;
  const u32 base = O[tile], size = O[tile + 1] - base;
  const bool over = size > (u32)MSD_CAP;
  const int s1 = max(msd_top(diff) - d1, 0), s2 = max(s1 - MSD_D2, 0);
  u128 v[KPT];
  u32 dg[KPT], pos[KPT];
#pragma unroll
  for (int k = 0; k < KPT; ++k) {
    const u32 i = threadIdx.x + k * MSD_BT;
    dg[k] = NS;
    if (!over && i < size) {
      v[k] = keys[base + i];
      dg[k] = msd_digit(v[k], s2, MSD_D2);
    }
  }
#pragma unroll
  for (int k = 0; k < KPT; ++k)
    if (dg[k] < NS) atomicAdd(C + dg[k], 1u);
  __syncthreads();
  u32 loc[PER], sum = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    loc[q] = C[threadIdx.x * PER + q];
    sum += loc[q];
    if (loc[q] > (u32)MSD_SUBLEN) s_bad = 1;
  }
  u32 tot;
  u32 run = block_scan_excl(sum, ws, &tot);
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    C[threadIdx.x * PER + q] = run;
    run += loc[q];
  }
  __syncthreads();
  const bool bad = over || s_bad;
  if (!bad) {
#pragma unroll
    for (int k = 0; k < KPT; ++k)
      if (dg[k] < NS) {
        pos[k] = atomicAdd(C + dg[k], 1u);
        B[pos[k]] = v[k];
      }
  }
  __syncthreads();  // C[j] = end of sub-bucket j = start of j + 1
  u32 first = 0;
  if (!bad) {
#pragma unroll
    for (int k = 0; k < KPT; ++k)
      if (dg[k] < NS) {
        const u32 st = dg[k] ? C[dg[k] - 1] : 0u;
        const u128 x = B[pos[k]];  // keys are re-read from shared memory: registers stay < 64
        bool f = true;
        for (u32 u = st; u < pos[k]; ++u)
          if (B[u] == x) {
            f = false;
            break;
          }
        if (f) {
          first |= 1u << k;
          atomicAdd(D + dg[k], 1u);
          atomicOr(F + (pos[k] >> 5), 1u << (pos[k] & 31));
        }
      }
  }
  __syncthreads();
  sum = 0;
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    loc[q] = D[threadIdx.x * PER + q];
    sum += loc[q];
  }
  u32 dtot;
  run = block_scan_excl(sum, ws, &dtot);
#pragma unroll
  for (int q = 0; q < PER; ++q) {
    D[threadIdx.x * PER + q] = run;
    run += loc[q];
  }
  if (threadIdx.x == 0) {
    if (bad) atomicOr(err, 2u);
    Dc[tile] = bad ? 0u : dtot;
  }
  __syncthreads();
  if (bad) return;
  // first occurrences, ranked, overwrite the front of the bucket's own range
  // (the keys are all in shared memory by now)
  u128 ranked[KPT];
  u32 loff[KPT];
#pragma unroll
  for (int k = 0; k < KPT; ++k)
    if (first & (1u << k)) {
      const u32 st = dg[k] ? C[dg[k] - 1] : 0u, en = C[dg[k]];
      const u128 x = B[pos[k]];
      u32 rank = 0;
      for (u32 u = st; u < en; ++u) rank += ((F[u >> 5] >> (u & 31)) & 1u) && B[u] < x;
      loff[k] = D[dg[k]] + rank;
      ranked[k] = x;
    }
  __syncthreads();  // every key of the bucket read (registers / shared) before the overwrite
#pragma unroll
  for (int k = 0; k < KPT; ++k)
    if (first & (1u << k)) keys[base + loff[k]] = ranked[k];
}

// distinct keys of bucket b (front of its range) -> out[Doff[b] ...],
// unpacked to W words; one warp per bucket
__global__ void __launch_bounds__(MB_THREADS) k_msd_compact(const u128* __restrict__ keys, const u32* __restrict__ O,
                                                            const u32* __restrict__ Dc, const u32* __restrict__ Doff,
                                                            int nb, int words, int kb, u64* __restrict__ out) {
  const int b = (int)(((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5), lane = threadIdx.x & 31;
  if (b >= nb) return;
  const u32 base = O[b], cnt = Dc[b], o = Doff[b];
  const u64 lim = kb >= 64 ? ~0ull : ((1ull << kb) - 1);
  for (u32 i = lane; i < cnt; i += 32) {
    const u128 x = keys[base + i];
    if (words == 2)
      reinterpret_cast<ulonglong2*>(out)[o + i] = make_ulonglong2((u64)(x >> kb), (u64)x & lim);
    else
      out[o + i] = (u64)x;
  }
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
  ensure(c, flags, 32);
  u32* err = flags.as<u32>();
  u32* d_count = err + 1;
  memset_async(c, err, 0, 32);
  // MSD bucket path (see above); D1 puts ~1K keys in a bucket
  bool done = false;
  if (!c->opt_dict_lsd && n <= (1ll << 24) + (1ll << 22)) {
    int d1 = 0;  // ~512 keys per bucket: 100 copies of ~5 distinct keys still fit MSD_CAP
    while (d1 < 15 && ((long long)512 << d1) < n) ++d1;
    const int nb = 1 << d1;
    const int G = std::max(1, std::min(c->num_sms * 2, (int)((n + 4095) / 4096)));
    DBuf H, O, st;
    ensure(c, H, (size_t)nb * 4 + 4);
    ensure(c, O, (size_t)(nb + 1) * 4);
    ensure(c, st, (size_t)nb * 4 + 8);
    ensure(c, packed, (size_t)n * 16);
    u64* diff = reinterpret_cast<u64*>(err + 4);  // 16-byte aligned: err + 4 .. + 7
    memset_async(c, st.p, 0, (size_t)nb * 4 + 8);
    memset_async(c, H.p, 0, (size_t)nb * 4 + 4);
    F4B_LAUNCH(c, k_msd_diff, mb_grid(c, n), MB_THREADS, 0, keys, n, words, key_bits, diff, err);
    const size_t hs = (size_t)nb * 4;
    check_cuda(cudaFuncSetAttribute(k_msd_hist, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)hs), "smem");
    F4B_LAUNCH(c, k_msd_hist, G, MSD_THREADS, hs, keys, n, words, key_bits, d1, diff, H.as<u32>());
    exclusive_scan_u32(c, H.as<u32>(), O.as<u32>(), (long long)nb);
    check_cuda(cudaMemcpyAsync(H.p, O.p, (size_t)nb * 4, cudaMemcpyDeviceToDevice, c->stream), "d2d");
    F4B_LAUNCH(c, k_msd_scatter, mb_grid(c, n), MB_THREADS, 0, keys, n, words, key_bits, d1, diff, H.as<u32>(),
               packed.as<u128>());
    const size_t bs = (size_t)MSD_CAP * 16 + (size_t)(2 << MSD_D2) * 4 + MSD_CAP / 8;
    check_cuda(cudaFuncSetAttribute(k_msd_bucket, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)bs), "smem");
    u32* Dc = st.as<u32>();  // [nb + 1] distinct per bucket -> (H) offsets
    F4B_LAUNCH(c, k_msd_bucket, nb, MSD_BT, bs, packed.as<u128>(), O.as<u32>(), d1, diff, Dc, err);
    exclusive_scan_u32(c, Dc, H.as<u32>(), (long long)nb);
    F4B_LAUNCH(c, k_msd_compact, (unsigned)((nb * 32ll + MB_THREADS - 1) / MB_THREADS), MB_THREADS, 0,
               packed.as<u128>(), O.as<u32>(), Dc, H.as<u32>(), nb, words, key_bits, out);
    check_cuda(cudaMemcpyAsync(d_count, H.as<u32>() + nb, 4, cudaMemcpyDeviceToDevice, c->stream), "d2d");
    const u32 e = read_u32(c, err);
    release(c, H);
    release(c, O);
    release(c, st);
    if (e & 1u) {
      release(c, packed);
      release(c, flags);
      fail(F4B_ERR_PRECONDITION, "dict_build: a key word has more than key_bits significant bits");
    }
    done = !(e & 2u);
    if (!done) memset_async(c, err, 0, 8);
  }
  if (done) {
    const long long nu = read_u32(c, d_count);
    release(c, packed);
    release(c, flags);
    return nu;
  }
  {
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
