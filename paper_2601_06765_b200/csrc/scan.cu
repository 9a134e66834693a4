// Device-wide exclusive scan (reference bulk.py:65-79 `exclusive_scan`):
// reduce-then-scan over 4096-element tiles (256 threads x 16 items), warp
// shuffles inside a block, recursion over the tile sums.  out has n+1
// entries, out[n] = total.
#include "common.cuh"
#include "engine.h"

namespace f4b {

static constexpr int SCAN_THREADS = 256;
static constexpr int SCAN_ITEMS = 16;
static constexpr int SCAN_TILE = SCAN_THREADS * SCAN_ITEMS;

// Block-wide exclusive scan of one value per thread; returns the prefix and
// writes the block total to *total.
F4B_DEV u32 block_exclusive_scan(u32 v, u32* total) {
  __shared__ u32 warp_sums[SCAN_THREADS / 32];
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  u32 x = v;
#pragma unroll
  for (int o = 1; o < 32; o <<= 1) {
    u32 y = __shfl_up_sync(0xffffffffu, x, o);
    if (lane >= o) x += y;
  }
  if (lane == 31) warp_sums[warp] = x;
  __syncthreads();
  if (warp == 0) {
    u32 s = lane < SCAN_THREADS / 32 ? warp_sums[lane] : 0;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      u32 y = __shfl_up_sync(0xffffffffu, s, o);
      if (lane >= o) s += y;
    }
    if (lane < SCAN_THREADS / 32) warp_sums[lane] = s;
  }
  __syncthreads();
  u32 base = warp ? warp_sums[warp - 1] : 0;
  *total = warp_sums[SCAN_THREADS / 32 - 1];
  __syncthreads();
  return base + x - v;
}

struct LoadU32 {
  const u32* p;
  F4B_DEV u32 operator()(long long i) const { return p[i]; }
};
struct LoadFlag {
  const uint8_t* p;
  F4B_DEV u32 operator()(long long i) const { return p[i] ? 1u : 0u; }
};

template <class Load>
__global__ void __launch_bounds__(SCAN_THREADS) k_tile_sums(Load ld, long long n, u32* sums) {
  long long base = (long long)blockIdx.x * SCAN_TILE + (long long)threadIdx.x * SCAN_ITEMS;
  u32 s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i)
    if (base + i < n) s += ld(base + i);
  u32 total;
  block_exclusive_scan(s, &total);
  if (threadIdx.x == 0) sums[blockIdx.x] = total;
}

template <class Load>
__global__ void __launch_bounds__(SCAN_THREADS) k_tile_scan(Load ld, long long n, const u32* tile_prefix, u32* out) {
  long long base = (long long)blockIdx.x * SCAN_TILE + (long long)threadIdx.x * SCAN_ITEMS;
  u32 v[SCAN_ITEMS];
  u32 s = 0;
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    v[i] = (base + i < n) ? ld(base + i) : 0u;
    s += v[i];
  }
  u32 total;
  u32 run = block_exclusive_scan(s, &total) + (tile_prefix ? tile_prefix[blockIdx.x] : 0u);
#pragma unroll
  for (int i = 0; i < SCAN_ITEMS; ++i) {
    if (base + i < n) out[base + i] = run;
    run += v[i];
  }
  if (base < n && base + SCAN_ITEMS >= n) out[n] = run;  // the thread owning the last element
}

// Recursive worker with an explicit scratch cursor.
template <class Load>
static void scan_level(Ctx* c, Load ld, u32* out, long long n, u32* scratch) {
  long long tiles = (n + SCAN_TILE - 1) / SCAN_TILE;
  if (tiles <= 1) {
    F4B_LAUNCH(c, k_tile_scan<Load>, 1, SCAN_THREADS, 0, ld, n, nullptr, out);
    check_cuda(cudaGetLastError(), "k_tile_scan");
    return;
  }
  u32* sums = scratch;
  u32* prefix = scratch + tiles + 1;
  F4B_LAUNCH(c, k_tile_sums<Load>, (unsigned)tiles, SCAN_THREADS, 0, ld, n, sums);
  check_cuda(cudaGetLastError(), "k_tile_sums");
  scan_level<LoadU32>(c, LoadU32{sums}, prefix, tiles, prefix + tiles + 1);
  F4B_LAUNCH(c, k_tile_scan<Load>, (unsigned)tiles, SCAN_THREADS, 0, ld, n, prefix, out);
  check_cuda(cudaGetLastError(), "k_tile_scan");
}

static size_t scan_scratch_words(long long n) {
  size_t need = 0;
  for (long long t = (n + SCAN_TILE - 1) / SCAN_TILE; t > 1; t = (t + SCAN_TILE - 1) / SCAN_TILE)
    need += 2 * (size_t)(t + 1);
  return need + 64;
}

void exclusive_scan_u32(Ctx* c, const uint32_t* in, uint32_t* out, long long n) {
  if (n <= 0) {
    check_cuda(cudaMemsetAsync(out, 0, sizeof(u32), c->stream), "scan memset");
    return;
  }
  ensure(c, c->scan_tmp, scan_scratch_words(n) * sizeof(u32));
  scan_level<LoadU32>(c, LoadU32{in}, out, n, c->scan_tmp.as<u32>());
}

void exclusive_scan_flags(Ctx* c, const uint8_t* flags, uint32_t* out, long long n) {
  if (n <= 0) {
    check_cuda(cudaMemsetAsync(out, 0, sizeof(u32), c->stream), "scan memset");
    return;
  }
  ensure(c, c->scan_tmp, scan_scratch_words(n) * sizeof(u32));
  scan_level<LoadFlag>(c, LoadFlag{flags}, out, n, c->scan_tmp.as<u32>());
}

}  // namespace f4b
