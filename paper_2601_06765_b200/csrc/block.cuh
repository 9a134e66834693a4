// CTA-level building blocks for the single-pass FBSP kernels:
//   * block_scan_excl  — exclusive scan of one u32 per thread
//   * lookback_prefix  — decoupled look-back over tile aggregates (tiles are
//                        claimed through an atomic ticket, so every earlier
//                        tile is resident and the spin always terminates)
//   * block_sort_keys  — stable LSD radix sort of up to TILE keys held in
//                        shared memory (warp-contiguous segments, ranking
//                        with __match_any_sync, per-warp running counts)
//   * block_unique     — unique of a sorted shared-memory key run
#pragma once
#include "common.cuh"

namespace f4b {

// status word of the look-back: 2 flag bits + 30-bit value
static constexpr u32 LB_AGG = 1u << 30;
static constexpr u32 LB_PRE = 2u << 30;
static constexpr u32 LB_VAL = (1u << 30) - 1u;

// Exclusive scan of v across the CTA (blockDim.x multiple of 32, <= 1024).
// `ws` must hold 33 u32.  Returns the prefix; *total = block sum.
F4B_DEV u32 block_scan_excl(u32 v, u32* ws, u32* total) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  u32 x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) ws[warp] = x;
  __syncthreads();
  if (warp == 0) {
    u32 s = lane < nw ? ws[lane] : 0u;
    u32 t = s;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      u32 y = __shfl_up_sync(0xffffffffu, t, o);
      if (lane >= o) t += y;
    }
    if (lane < nw) ws[lane] = t - s;
    if (lane == 31) ws[32] = t;
  }
  __syncthreads();
  u32 res = ws[warp] + x - v;
  *total = ws[32];
  __syncthreads();
  return res;
}

F4B_DEV u32 ld_volatile(const u32* p) {
  u32 v;
  asm volatile("ld.volatile.global.u32 %0, [%1];" : "=r"(v) : "l"(p));
  return v;
}

// Decoupled look-back for one counter per tile.  Called by ONE thread.
// status[] zero-initialised; returns the exclusive prefix of `count`.
// lb_publish (the tile's aggregate) and lb_resolve (the wait for the
// predecessors) may be split so the caller works in between.
F4B_DEV void lb_publish(u32* status, u32 tile, u32 count) {
  atomicExch(status + tile, (tile == 0 ? LB_PRE : LB_AGG) | count);
}

F4B_DEV u32 lb_resolve(u32* status, u32 tile, u32 count) {
  if (tile == 0) return 0;
  // 4 predecessors per round trip (independent loads in flight); one not
  // yet published is polled again
  u32 excl = 0;
  long long j = (long long)tile - 1;
  bool done = false;
  while (!done) {
    u32 sv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) sv[q] = j - q >= 0 ? ld_volatile(status + (j - q)) : LB_PRE;
    int q = 0;
#pragma unroll
    for (int t = 0; t < 4; ++t) {
      if (done || q < t) continue;
      const u32 flag = sv[t] & ~LB_VAL;
      if (flag == 0) continue;
      excl += sv[t] & LB_VAL;
      q = t + 1;
      done = flag == LB_PRE;
    }
    j -= q;
  }
  __threadfence();
  atomicExch(status + tile, LB_PRE | (excl + count));
  return excl;
}

F4B_DEV u32 lookback_prefix(u32* status, u32 tile, u32 count) {
  lb_publish(status, tile, count);
  return lb_resolve(status, tile, count);
}

// Stable LSD radix sort of n (<= cap) keys in shared memory, low `bits` bits.
// `a` holds the keys on entry and on exit; `b` is scratch of the same size.
// wh: [nwarps][256] u32 shared scratch; ws: 33 u32.  Requires blockDim >= 256.
template <int KW, int MAXIT>
F4B_DEV void block_sort_keys(Key<KW>* a, Key<KW>* b, int n, int bits, u32* wh, u32* ws) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5, nw = blockDim.x >> 5;
  const int seg = ((n + nw - 1) / nw + 31) & ~31;  // keys per warp, multiple of 32
  const int lo = warp * seg, hi = min(n, lo + seg);
  Key<KW>* src = a;
  Key<KW>* dst = b;
  for (int bit = 0; bit < bits; bit += 8) {
    for (int i = threadIdx.x; i < nw * 256; i += blockDim.x) wh[i] = 0;
    __syncthreads();
    u32 pos[MAXIT];
#pragma unroll
    for (int it = 0; it < MAXIT; ++it) {
      const int idx = lo + it * 32 + lane;
      const bool valid = idx < hi;
      u32 d = 256u + lane;
      if (valid) d = key_digit<KW>(src[idx], bit);
      const unsigned peers = __match_any_sync(0xffffffffu, d);
      const u32 before = __popc(peers & lanemask_lt());
      const u32 cnt = valid ? wh[warp * 256 + d] : 0u;
      pos[it] = cnt + before;
      __syncwarp();
      if (valid && before == 0) wh[warp * 256 + d] = cnt + __popc(peers);
      __syncwarp();
    }
    __syncthreads();
    // digit-major exclusive offsets: digit base + prefix over warps
    u32 tot = 0;
    if (threadIdx.x < 256)
      for (int w = 0; w < nw; ++w) tot += wh[w * 256 + threadIdx.x];
    u32 total;
    u32 base = block_scan_excl(threadIdx.x < 256 ? tot : 0u, ws, &total);
    if (threadIdx.x < 256) {
      u32 run = base;
      for (int w = 0; w < nw; ++w) {
        u32 t = wh[w * 256 + threadIdx.x];
        wh[w * 256 + threadIdx.x] = run;
        run += t;
      }
    }
    __syncthreads();
#pragma unroll
    for (int it = 0; it < MAXIT; ++it) {
      const int idx = lo + it * 32 + lane;
      if (idx < hi) {
        const Key<KW> k = src[idx];
        dst[wh[warp * 256 + key_digit<KW>(k, bit)] + pos[it]] = k;
      }
    }
    __syncthreads();
    Key<KW>* t = src;
    src = dst;
    dst = t;
  }
  if (src != a) {
    for (int i = threadIdx.x; i < n; i += blockDim.x) a[i] = src[i];
    __syncthreads();
  }
}

}  // namespace f4b
