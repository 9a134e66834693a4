// Stable LSD radix sort of multiword keys + unique (reference bulk.py:86-124
// `radix_sort`, :135-150 `unique_sorted`, :153-166 `stream_compact`).
//
// The reference always runs 8*W byte passes.  Here only the bits that can
// differ are sorted: the device key format packs a batch's monomials into
// `bits` = lane_bits * n_lanes low bits, so cyclic-8 needs 4 passes instead
// of 24.  Output order is identical (a sorted set is unique).
//
// Each pass is count -> scan -> scatter over 4096-key tiles (8 warps x 32
// lanes x ITEMS).  Ranking inside a tile is stable: warps own contiguous
// sub-tiles, keys are visited in order, equal digits inside a warp step are
// ranked with __match_any_sync, and per-warp running counts in shared memory
// carry across steps; a per-digit prefix over warps plus the scanned global
// (digit-major, tile-minor) histogram gives each key its final slot.
#include "common.cuh"
#include "engine.h"

namespace f4b {

static constexpr int RS_THREADS = 256;
static constexpr int RS_WARPS = RS_THREADS / 32;

template <int KW>
struct RsItems {
  static constexpr int value = KW >= 4 ? 4 : (KW == 2 ? 8 : 16);
};

template <int KW>
__global__ void __launch_bounds__(RS_THREADS) k_radix_count(const u64* __restrict__ in, long long n, int bit,
                                                            u32* __restrict__ hist, int tiles) {
  constexpr int ITEMS = RsItems<KW>::value;
  __shared__ u32 h[256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  h[threadIdx.x] = 0;
  __syncthreads();
  long long wbase = (long long)blockIdx.x * (RS_THREADS * ITEMS) + (long long)warp * 32 * ITEMS;
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    long long idx = wbase + it * 32 + lane;
    bool valid = idx < n;
    u32 d = 256u + lane;
    if (valid) d = key_digit<KW>(key_load<KW>(in, idx), bit);
    unsigned peers = __match_any_sync(0xffffffffu, d);
    if (valid && (peers & lanemask_lt()) == 0) atomicAdd(&h[d], (u32)__popc(peers));
  }
  __syncthreads();
  hist[(long long)threadIdx.x * tiles + blockIdx.x] = h[threadIdx.x];
}

template <int KW>
__global__ void __launch_bounds__(RS_THREADS) k_radix_scatter(const u64* __restrict__ in, u64* __restrict__ out,
                                                              long long n, int bit, const u32* __restrict__ offs,
                                                              int tiles) {
  constexpr int ITEMS = RsItems<KW>::value;
  __shared__ u32 wh[RS_WARPS][256];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int i = threadIdx.x; i < RS_WARPS * 256; i += RS_THREADS) (&wh[0][0])[i] = 0;
  __syncthreads();
  long long wbase = (long long)blockIdx.x * (RS_THREADS * ITEMS) + (long long)warp * 32 * ITEMS;
  Key<KW> k[ITEMS];
  u32 rank[ITEMS];
  u32 dig[ITEMS];
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    long long idx = wbase + it * 32 + lane;
    bool valid = idx < n;
    u32 d = 256u + lane;
    if (valid) {
      k[it] = key_load<KW>(in, idx);
      d = key_digit<KW>(k[it], bit);
    }
    dig[it] = d;
    unsigned peers = __match_any_sync(0xffffffffu, d);
    u32 before = __popc(peers & lanemask_lt());
    u32 cnt = valid ? wh[warp][d] : 0u;
    rank[it] = cnt + before;
    __syncwarp();
    if (valid && before == 0) wh[warp][d] = cnt + __popc(peers);
    __syncwarp();
  }
  __syncthreads();
  {
    const int d = threadIdx.x;
    u32 run = offs[(long long)d * tiles + blockIdx.x];
#pragma unroll
    for (int w = 0; w < RS_WARPS; ++w) {
      u32 t = wh[w][d];
      wh[w][d] = run;
      run += t;
    }
  }
  __syncthreads();
#pragma unroll
  for (int it = 0; it < ITEMS; ++it) {
    long long idx = wbase + it * 32 + lane;
    if (idx < n) key_store<KW>(out, (long long)wh[warp][dig[it]] + rank[it], k[it]);
  }
}

template <int KW>
static void radix_sort_t(Ctx* c, const u64* in, long long n, int bits, u64** result) {
  constexpr int ITEMS = RsItems<KW>::value;
  ensure(c, c->sort_a, (size_t)(n + 1) * KW * sizeof(u64));
  ensure(c, c->sort_b, (size_t)(n + 1) * KW * sizeof(u64));
  u64* bufs[2] = {c->sort_a.as<u64>(), c->sort_b.as<u64>()};
  if (n <= 1 || bits <= 0) {
    if (n > 0)
      check_cuda(cudaMemcpyAsync(bufs[0], in, (size_t)n * KW * sizeof(u64), cudaMemcpyDeviceToDevice, c->stream),
                 "sort copy");
    *result = bufs[0];
    return;
  }
  const int tile = RS_THREADS * ITEMS;
  const int tiles = (int)((n + tile - 1) / tile);
  ensure(c, c->sort_hist, ((size_t)256 * tiles + 1) * 2 * sizeof(u32));
  u32* hist = c->sort_hist.as<u32>();
  u32* offs = hist + (size_t)256 * tiles + 1;
  const u64* src = in;
  int which = 0;
  for (int b = 0; b < bits; b += 8) {
    F4B_LAUNCH(c, k_radix_count<KW>, tiles, RS_THREADS, 0, src, n, b, hist, tiles);
    check_cuda(cudaGetLastError(), "k_radix_count");
    exclusive_scan_u32(c, hist, offs, (long long)256 * tiles);
    F4B_LAUNCH(c, k_radix_scatter<KW>, tiles, RS_THREADS, 0, src, bufs[which], n, b, offs, tiles);
    check_cuda(cudaGetLastError(), "k_radix_scatter");
    src = bufs[which];
    which ^= 1;
  }
  *result = const_cast<u64*>(src);
}

void radix_sort_keys(Ctx* c, int KW, const uint64_t* in, long long n, int bits, uint64_t** result) {
  switch (KW) {
    case 1: radix_sort_t<1>(c, in, n, bits, result); break;
    case 2: radix_sort_t<2>(c, in, n, bits, result); break;
    case 4: radix_sort_t<4>(c, in, n, bits, result); break;
    case 8: radix_sort_t<8>(c, in, n, bits, result); break;
    default: fail(F4B_ERR_PRECONDITION, "unsupported key width");
  }
}

// ---------------------------------------------------------------------------
// unique: head flags -> scan -> compact
// ---------------------------------------------------------------------------
template <int KW>
__global__ void k_head_flags(const u64* __restrict__ keys, long long n, uint8_t* __restrict__ flags) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  uint8_t f = 1;
  if (i > 0) f = key_eq<KW>(key_load<KW>(keys, i), key_load<KW>(keys, i - 1)) ? 0 : 1;
  flags[i] = f;
}

template <int KW>
__global__ void k_compact_keys(const u64* __restrict__ keys, long long n, const uint8_t* __restrict__ flags,
                               const u32* __restrict__ pos, u64* __restrict__ out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n || !flags[i]) return;
  key_store<KW>(out, pos[i], key_load<KW>(keys, i));
}

template <int KW>
static long long unique_t(Ctx* c, const u64* sorted, long long n, u64* out) {
  if (n == 0) return 0;
  ensure(c, c->flags, (size_t)n + 16);
  ensure(c, c->tmp_u32a, ((size_t)n + 1) * sizeof(u32));
  uint8_t* flags = c->flags.as<uint8_t>();
  u32* pos = c->tmp_u32a.as<u32>();
  const int T = 256;
  unsigned blocks = (unsigned)((n + T - 1) / T);
  F4B_LAUNCH(c, k_head_flags<KW>, blocks, T, 0, sorted, n, flags);
  check_cuda(cudaGetLastError(), "k_head_flags");
  exclusive_scan_flags(c, flags, pos, n);
  F4B_LAUNCH(c, k_compact_keys<KW>, blocks, T, 0, sorted, n, flags, pos, out);
  check_cuda(cudaGetLastError(), "k_compact_keys");
  return (long long)read_u32(c, pos + n);
}

long long unique_keys(Ctx* c, int KW, const uint64_t* sorted, long long n, uint64_t* out) {
  switch (KW) {
    case 1: return unique_t<1>(c, sorted, n, out);
    case 2: return unique_t<2>(c, sorted, n, out);
    case 4: return unique_t<4>(c, sorted, n, out);
    case 8: return unique_t<8>(c, sorted, n, out);
    default: fail(F4B_ERR_PRECONDITION, "unsupported key width");
  }
}

}  // namespace f4b
