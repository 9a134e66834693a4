// Dictionary sort + unique (reference bulk.py:86-124 `radix_sort`,
// :135-150 `unique_sorted`, :153-166 `stream_compact`, :169-184 `lower_bound`).
//
// sort_unique(): keys -> ascending unique keys, optionally dropping keys that
// are already in a sorted dictionary (the closure's "new monomials" filter,
// symbolic.py:281-290).  Two regimes:
//   * n <= small_cap: ONE kernel — the whole input sorted in shared memory
//     (block_sort_keys), unique, absent-filter, compact;
//   * otherwise a one-sweep LSD radix sort: one histogram kernel for all
//     digit passes, then ONE kernel per 8-bit pass (tiles claimed by ticket,
//     per-digit decoupled look-back for the global offsets, stable ranks via
//     __match_any_sync), then one fused unique/absent/compact kernel with
//     look-back.  Only the `bits` low bits of the compact device key are
//     sorted (cyclic-8: 4 passes instead of the reference's 24).
// The element count may live in device memory (d_n) so no host round trip is
// needed between the producer kernel and the sort.
#include "block.cuh"
#include "common.cuh"
#include "engine.h"

namespace f4b {

static constexpr int OS_THREADS = 256;
static constexpr int OS_WARPS = OS_THREADS / 32;
static constexpr int OS_LB = 4;  // look-back window (status loads per round trip)
static constexpr int OS_MAX_PASSES = 16;  // 128-bit keys; tickets[32]: one per pass + the unique kernel's

template <int KW>
struct OsItems {
  static constexpr int value = KW >= 4 ? 4 : (KW == 2 ? 8 : 16);
};

// tiles of at most 32 KB of keys are reordered in shared memory before the
// scatter (static shared memory stays under 48 KB)
template <int KW>
constexpr bool OS_STAGED = (size_t)KW * 8 * OS_THREADS * OsItems<KW>::value <= 32768;

template <int KW>
struct SmallCfg {  // single-CTA sort: 512 threads
  static constexpr int MAXIT = KW >= 4 ? 4 / (KW / 4) : (KW == 2 ? 8 : 16);
  static constexpr int CAP = 16 * 32 * MAXIT;
};

F4B_DEV u32 dev_n(const u32* d_n, u32 n) { return d_n ? *d_n : n; }

// Adaptive launches (n only known on the device): the single-CTA kernel runs
// when n <= small_cap, the one-sweep kernels when n > small_cap.
F4B_DEV bool skip_large(u32 n, u32 small_cap) { return small_cap && n <= small_cap; }

template <int KW>
__global__ void __launch_bounds__(OS_THREADS) k_os_hist(const u64* __restrict__ in, const u32* d_n, u32 n_host,
                                                        int npass, u32* __restrict__ hist, u32 small_cap) {
  __shared__ u32 h[OS_MAX_PASSES][256];
  const u32 n = dev_n(d_n, n_host);
  if (skip_large(n, small_cap)) return;
  for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) (&h[0][0])[i] = 0;
  __syncthreads();
  for (long long base = (long long)blockIdx.x * blockDim.x; base < n; base += (long long)gridDim.x * blockDim.x) {
    const long long i = base + threadIdx.x;
    const bool valid = i < n;
    Key<KW> k;
    if (valid) k = key_load<KW>(in, i);
    // plain shared atomics: a warp-aggregated count (__match_any_sync per
    // digit) was measured 3x slower on uniform keys (12 passes, 16M keys)
    if (valid)
      for (int p = 0; p < npass; ++p) atomicAdd(&h[p][key_digit<KW>(k, 8 * p)], 1u);
  }
  __syncthreads();
  for (int i = threadIdx.x; i < npass * 256; i += blockDim.x) {
    u32 v = (&h[0][0])[i];
    if (v) atomicAdd(hist + i, v);
  }
}

template <int KW>
__global__ void __launch_bounds__(OS_THREADS, KW == 1 ? 3 : (OS_STAGED<KW> ? 4 : 1)) k_os_pass(const u64* __restrict__ in, u64* __restrict__ out,
                                                        const u32* d_n, u32 n_host, int bit,
                                                        const u32* __restrict__ hist, u32* status, u32* ticket,
                                                        u32 small_cap) {
  constexpr int ITEMS = OsItems<KW>::value;
  constexpr int TILE = OS_THREADS * ITEMS;
  __shared__ u32 wh[OS_WARPS][256];
  __shared__ u32 gbase[256];
  __shared__ u32 s_toff[OS_STAGED<KW> ? 256 : 1];
  __shared__ Key<KW> s_keys[OS_STAGED<KW> ? TILE : 1];
  __shared__ u32 ws[33];
  __shared__ u32 s_tile;
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u32 n = dev_n(d_n, n_host);
  if (skip_large(n, small_cap)) return;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  for (int i = threadIdx.x; i < OS_WARPS * 256; i += OS_THREADS) (&wh[0][0])[i] = 0;
  __syncthreads();
  const u32 tile = s_tile;
  if ((long long)tile * TILE >= n) return;
  // digit bases of this pass (every CTA scans the 256-bin histogram)
  {
    u32 tot;
    u32 b = block_scan_excl(hist[threadIdx.x], ws, &tot);
    gbase[threadIdx.x] = b;
  }
  const long long wbase = (long long)tile * TILE + (long long)warp * 32 * ITEMS;
  Key<KW> k[ITEMS];
  u32 rank[ITEMS], dig[ITEMS];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    const long long idx = wbase + it * 32 + lane;
    const bool valid = idx < n;
    u32 d = 256u + lane;
    if (valid) {
      k[it] = key_load<KW>(in, idx);
      d = key_digit<KW>(k[it], bit);
    }
    dig[it] = d;
    const unsigned peers = __match_any_sync(0xffffffffu, d);
    const u32 before = __popc(peers & lanemask_lt());
    const u32 cnt = valid ? wh[warp][d] : 0u;
    rank[it] = cnt + before;
    __syncwarp();
    if (valid && before == 0) wh[warp][d] = cnt + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  // tile count per digit -> publish + look-back (one thread per digit)
  {
    const int d = threadIdx.x;
    u32 run = 0;
#pragma unroll
    for (int w = 0; w < OS_WARPS; ++w) {
      const u32 t = wh[w][d];
      wh[w][d] = run;
      run += t;
    }
    u32* st = status + d;  // status[tile * 256 + d]
    u32 excl = 0;
    if (tile == 0) {
      atomicExch(st, LB_PRE | run);
    } else {
      atomicExch(st + (size_t)tile * 256, LB_AGG | run);
      // look back OS_LB predecessors per round trip (independent loads in
      // flight); a not-yet-published one is polled again
      long long j = (long long)tile - 1;
      bool done = false;
      while (!done) {
        u32 sv[OS_LB];
#pragma unroll
        for (int q = 0; q < OS_LB; ++q) sv[q] = j - q >= 0 ? ld_volatile(st + (size_t)(j - q) * 256) : LB_PRE;
        int q = 0;
#pragma unroll
        for (int t = 0; t < OS_LB; ++t) {
          if (done || q < t) continue;
          const u32 flag = sv[t] & ~LB_VAL;
          if (flag == 0) continue;  // not published: poll again from j - t
          excl += sv[t] & LB_VAL;
          q = t + 1;
          done = flag == LB_PRE;
        }
        j -= q;
      }
      __threadfence();
      atomicExch(st + (size_t)tile * 256, LB_PRE | (excl + run));
    }
    gbase[d] += excl;
    if constexpr (OS_STAGED<KW>) {
      // tile-local digit offsets: the tile is reordered by digit in shared
      // memory, then written out in consecutive runs per digit (coalesced
      // stores instead of one 8/16-byte scatter per key)
      u32 tot;
      const u32 toff = block_scan_excl(run, ws, &tot);
      s_toff[d] = toff;
      gbase[d] -= toff;  // global position = gbase[d] + tile-local position
    }
  }
  __syncthreads();
  if constexpr (OS_STAGED<KW>) {
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      const long long idx = wbase + it * 32 + lane;
      if (idx < n) s_keys[s_toff[dig[it]] + wh[warp][dig[it]] + rank[it]] = k[it];
    }
    __syncthreads();
    const u32 tile_n = (u32)min((long long)TILE, (long long)n - (long long)tile * TILE);
    for (u32 i = threadIdx.x; i < tile_n; i += OS_THREADS) {
      const Key<KW> kk = s_keys[i];
      key_store<KW>(out, (long long)gbase[key_digit<KW>(kk, bit)] + i, kk);
    }
  } else {
#pragma unroll
    for (int it = 0; it < ITEMS; ++it) {
      const long long idx = wbase + it * 32 + lane;
      if (idx < n) key_store<KW>(out, (long long)gbase[dig[it]] + wh[warp][dig[it]] + rank[it], k[it]);
    }
  }
}

// Fused unique + absent-from-dictionary filter + compaction with look-back.
template <int KW>
__global__ void __launch_bounds__(OS_THREADS) k_unique_absent(const u64* __restrict__ sorted, const u32* d_n,
                                                              u32 n_host, const u64* __restrict__ dict,
                                                              const u32* d_ndict, u64* __restrict__ out,
                                                              u32* status, u32* ticket, u32* d_count,
                                                              u32 small_cap) {
  constexpr int ITEMS = 8;
  constexpr int TILE = OS_THREADS * ITEMS;
  __shared__ u32 ws[33];
  __shared__ u32 s_tile, s_base;
  const u32 n = dev_n(d_n, n_host);
  if (skip_large(n, small_cap)) return;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const u32 tile = s_tile;
  const u32 ntiles = (n + TILE - 1) / TILE;
  if (tile >= ntiles) return;
  const u32 nd = dict ? *d_ndict : 0u;
  const long long base = (long long)tile * TILE + (long long)threadIdx.x * ITEMS;
  u32 keep = 0;
  unsigned mask = 0;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i) {
    const long long idx = base + i;
    if (idx >= n) break;
    const Key<KW> k = key_load<KW>(sorted, idx);
    bool f = idx == 0 || !key_eq<KW>(k, key_load<KW>(sorted, idx - 1));
    if (f && nd) {
      const u32 pos = key_lower_bound<KW>(dict, nd, k);
      f = !(pos < nd && key_eq<KW>(key_load<KW>(dict, pos), k));
    }
    if (f) {
      mask |= 1u << i;
      ++keep;
    }
  }
  u32 tot;
  u32 pre = block_scan_excl(keep, ws, &tot);
  if (threadIdx.x == 0) s_base = lookback_prefix(status, tile, tot);
  __syncthreads();
  u32 o = s_base + pre;
#pragma unroll
  for (int i = 0; i < ITEMS; ++i)
    if (mask & (1u << i)) key_store<KW>(out, o++, key_load<KW>(sorted, base + i));
  if (tile == ntiles - 1 && threadIdx.x == 0) *d_count = s_base + tot;
}

// Whole input in one CTA: sort + unique + absent + compact.
template <int KW>
__global__ void __launch_bounds__(512) k_small_sort_unique(const u64* __restrict__ in, const u32* d_n, u32 n_host,
                                                           int bits, const u64* __restrict__ dict,
                                                           const u32* d_ndict, u64* __restrict__ out,
                                                           u32* d_count) {
  if (dev_n(d_n, n_host) > (u32)SmallCfg<KW>::CAP) return;  // the one-sweep path handles it
  constexpr int MAXIT = SmallCfg<KW>::MAXIT;
  extern __shared__ __align__(16) unsigned char smraw[];
  Key<KW>* a = reinterpret_cast<Key<KW>*>(smraw);
  Key<KW>* b = a + SmallCfg<KW>::CAP;
  u32* wh = reinterpret_cast<u32*>(b + SmallCfg<KW>::CAP);
  __shared__ u32 ws[33];
  const u32 n = dev_n(d_n, n_host);
  for (u32 i = threadIdx.x; i < n; i += blockDim.x) a[i] = key_load<KW>(in, i);
  __syncthreads();
  block_sort_keys<KW, MAXIT>(a, b, (int)n, bits, wh, ws);
  const u32 nd = dict ? *d_ndict : 0u;
  // unique + absent, chunked block scan
  u32 o = 0;
  for (u32 c0 = 0; c0 < n; c0 += blockDim.x) {
    const u32 i = c0 + threadIdx.x;
    bool f = false;
    if (i < n) {
      f = i == 0 || !key_eq<KW>(a[i], a[i - 1]);
      if (f && nd) {
        const u32 pos = key_lower_bound<KW>(dict, nd, a[i]);
        f = !(pos < nd && key_eq<KW>(key_load<KW>(dict, pos), a[i]));
      }
    }
    u32 tot;
    const u32 pre = block_scan_excl(f ? 1u : 0u, ws, &tot);
    if (f) key_store<KW>(out, o + pre, a[i]);
    o += tot;
  }
  if (threadIdx.x == 0) *d_count = o;
}

template <int KW>
static void sort_unique_t(Ctx* c, const u64* in, const u32* d_n, u32 n_max, int bits, const u64* dict,
                          const u32* d_ndict, u64* out, u32* d_count) {
  if (n_max == 0) {
    check_cuda(cudaMemsetAsync(d_count, 0, 4, c->stream), "memset");
    return;
  }
  const size_t smem = (size_t)2 * SmallCfg<KW>::CAP * KW * 8 + 16 * 256 * 4;
  static bool attr = false;
  if (!attr) {
    check_cuda(cudaFuncSetAttribute(k_small_sort_unique<KW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)smem),
               "attr");
    attr = true;
  }
  // n known on the host: pick one path.  n on the device (d_n): launch both,
  // each kernel checks n against the small-input capacity.
  const bool small_possible = d_n ? true : n_max <= (u32)SmallCfg<KW>::CAP;
  if (small_possible)
    F4B_LAUNCH(c, k_small_sort_unique<KW>, 1, 512, smem, in, d_n, n_max, bits, dict, d_ndict, out, d_count);
  if (n_max <= (u32)SmallCfg<KW>::CAP) return;
  const u32 small_cap = d_n ? (u32)SmallCfg<KW>::CAP : 0u;
  constexpr int TILE = OS_THREADS * OsItems<KW>::value;
  const int npass = (bits + 7) / 8;
  if (npass > OS_MAX_PASSES || bits > 64 * KW) fail(F4B_ERR_PRECONDITION, "sort_unique: too many key bits");
  const u32 tiles = (n_max + TILE - 1) / TILE;
  const u32 utiles = (n_max + OS_THREADS * 8 - 1) / (OS_THREADS * 8);
  // scratch: hist[npass*256] | tickets[32] | status[npass*tiles*256] | ustatus[utiles]
  const size_t words = (size_t)npass * 256 + 32 + (size_t)npass * tiles * 256 + utiles + 16;
  ensure(c, c->sort_hist, words * 4);
  u32* hist = c->sort_hist.as<u32>();
  u32* tickets = hist + npass * 256;
  u32* status = tickets + 32;
  u32* ustatus = status + (size_t)npass * tiles * 256;
  check_cuda(cudaMemsetAsync(hist, 0, words * 4, c->stream), "memset sort scratch");
  ensure(c, c->sort_a, (size_t)(n_max + 1) * KW * 8);
  ensure(c, c->sort_b, (size_t)(n_max + 1) * KW * 8);
  u64* bufs[2] = {c->sort_a.as<u64>(), c->sort_b.as<u64>()};
  const int hblocks = (int)std::min<long long>((n_max + OS_THREADS - 1) / OS_THREADS, (long long)c->num_sms * 4);
  F4B_LAUNCH(c, k_os_hist<KW>, hblocks, OS_THREADS, 0, in, d_n, n_max, npass, hist, small_cap);
  const u64* src = in;
  for (int p = 0; p < npass; ++p) {
    u64* dst = bufs[p & 1];
    F4B_LAUNCH(c, k_os_pass<KW>, tiles, OS_THREADS, 0, src, dst, d_n, n_max, 8 * p, hist + p * 256,
               status + (size_t)p * tiles * 256, tickets + p, small_cap);
    src = dst;
  }
  F4B_LAUNCH(c, k_unique_absent<KW>, utiles, OS_THREADS, 0, src, d_n, n_max, dict, d_ndict, out, ustatus,
             tickets + 31, d_count, small_cap);
}

void sort_unique(Ctx* c, int KW, const uint64_t* in, const uint32_t* d_n, uint32_t n_max, int bits,
                 const uint64_t* dict, const uint32_t* d_ndict, uint64_t* out, uint32_t* d_count) {
  switch (KW) {
    case 1: sort_unique_t<1>(c, in, d_n, n_max, bits, dict, d_ndict, out, d_count); break;
    case 2: sort_unique_t<2>(c, in, d_n, n_max, bits, dict, d_ndict, out, d_count); break;
    case 4: sort_unique_t<4>(c, in, d_n, n_max, bits, dict, d_ndict, out, d_count); break;
    case 8: sort_unique_t<8>(c, in, d_n, n_max, bits, dict, d_ndict, out, d_count); break;
    default: fail(F4B_ERR_PRECONDITION, "unsupported key width");
  }
}

}  // namespace f4b
