// F_p elimination to the fully reduced row echelon form on the device.
//
// Replaces reference `psge_reduce` (pkg/src/fpgb/sparselin.py:281-369).  The
// reduced echelon form of a matrix is unique, so any pivot schedule yields
// the reference's bytes; this one is the Faugère–Lachartre split validated in
// SURVEY.md §7.3(3):
//
//   E1  pivot per distinct leading column: fewest nonzeros, then lowest row
//       index — the reference rule (sparselin.py:316), via a 64-bit atomicMin
//       over (len << 32 | row).  A = pivot rows, C = the other nonzero rows.
//   E2  every C row is swept left to right over the A columns with a dense
//       F_p accumulator in shared memory (one CTA per row, warp-0 ballot scan
//       for the next nonzero A column, block-parallel sparse AXPY with the
//       normalized A row; Montgomery products in registers).  What remains
//       lives on the non-A columns: the dense block D' (|C| x K).
//   E3  D' forward elimination in one cooperative kernel (one grid barrier
//       per pivot: next pivot = min (leading column, row) over live rows;
//       pivot rows frozen once chosen), then a row-parallel
//       back-substitution to RREF(D').
//       RREF(D') rows are the rows with NEW leading columns — the
//       `nonpivot_rows` the F4 driver harvests (groebner.py:285-287).
//   E4  (full RREF only) every A row is swept over the A columns right of its
//       lead, then reduced in one shot by RREF(D') and made monic — the
//       reference's back-reduction (sparselin.py:337-349) done row-parallel.
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <climits>
#include <cstdlib>
#include <cstring>
#include <type_traits>
#include <vector>

#include "block.cuh"
#include "common.cuh"
#include "engine.h"

namespace cg = cooperative_groups;

struct f4b_echelon {
  f4b::Ctx* ctx = nullptr;
  long long M = 0;
  long long n_rows = 0, n_cols = 0, nA = 0, nC = 0, K = 0, rankD = 0, zero_rows = 0;
  bool full = false;
  bool partial = false;  // only the pivot rows of chosen lead columns were back-reduced (echelon_complete_rows)
  int64_t numeric_ns = 0, backsub_ns = 0;
  // input CSR (owned if uploaded from host)
  f4b::DBuf own_rp, own_col, own_val;
  const uint32_t *rp = nullptr, *col = nullptr, *val = nullptr;
  // structure
  f4b::DBuf prow;      // u32 [N] pivot row of each column or NONE
  f4b::DBuf invl;      // u32 [N] inverse of the pivot row's lead coefficient
  f4b::DBuf desc;      // uint4 [N] (tail start, tail end, inverse lead, pivot row)
  f4b::DBuf abits;     // u32 [(N+31)/32] A-column bitmap
  f4b::DBuf acols;     // u32 [nA] A columns ascending
  f4b::DBuf apos;      // u32 [N] index of each A column in acols
  f4b::DBuf nonA;      // u32 [K] non-A columns ascending
  f4b::DBuf Rd;        // u32 [rankD * K] RREF(D') rows (dense, non-A coordinates)
  f4b::DBuf dpiv;      // u32 [rankD] D' pivot positions (non-A coordinates)
  // outputs: pool + per-row slots
  f4b::DBuf pool_col, pool_val;  // u32
  f4b::DBuf a_off, a_len;        // u32 [nA] (pivot rows, ascending lead)
  f4b::DBuf d_off, d_len;        // u32 [rankD] (nonpivot rows, ascending lead)
  f4b::DBuf cursor;              // u64
  f4b::DBuf stats;               // u64 [2] sweep work counters
  f4b::DBuf rdev;                // u32 rank(D') written by k_dense_post
  unsigned long long sweep_pivots = 0, sweep_tail_nnz = 0;
  size_t pool_cap = 0;
  long long pivot_nnz = 0, nonpivot_nnz = 0;
};

namespace f4b {

static constexpr u32 NONE = 0xFFFFFFFFu;
static constexpr int SW_THREADS = 256;

static inline unsigned nb(long long n, int t) { return (unsigned)std::max<long long>(1, (n + t - 1) / t); }

// ---------------------------------------------------------------------------
// E1 fused (one cooperative launch): pivot selection, column structure, the
// A-column bitmap, A / non-A column lists (ascending), A-column positions and
// the C-row list, with 4 grid barriers and one host read of (nA, nC).
// ---------------------------------------------------------------------------
struct PrepOut {
  u32 nA, nC;
};
__global__ void __launch_bounds__(256) k_psge_prep(Fp fp, const u32* __restrict__ rp, const u32* __restrict__ col,
                                                   const u32* __restrict__ val, u32 r, u32 N,
                                                   unsigned long long* __restrict__ pk, u32* __restrict__ prow,
                                                   u32* __restrict__ invl, uint4* __restrict__ desc,
                                                   u32* __restrict__ abits, u32* __restrict__ acols,
                                                   u32* __restrict__ apos, u32* __restrict__ nonA,
                                                   u32* __restrict__ crows, u32* __restrict__ cnt, PrepOut* out) {
  cg::grid_group grid = cg::this_grid();
  __shared__ u32 ws[33];
  const int tid = threadIdx.x, lane = tid & 31;
  const u32 G = gridDim.x;
  const long long gt = (long long)blockIdx.x * blockDim.x + tid, GT = (long long)G * blockDim.x;
  // contiguous, 32-aligned column chunks and row chunks per CTA
  const u32 cw = (((N + G - 1) / G) + 31) & ~31u;
  const u32 c_lo = min(N, blockIdx.x * cw), c_hi = min(N, c_lo + cw);
  const u32 rw = (r + G - 1) / G;
  const u32 r_lo = min(r, blockIdx.x * rw), r_hi = min(r, r_lo + rw);
  auto bsum = [&](u32 v) -> u32 {
    u32 t;
    block_scan_excl(v, ws, &t);
    return t;
  };
  for (long long c = gt; c < N; c += GT) pk[c] = ~0ull;
  grid.sync();
  // P1: pivot per distinct lead: fewest nonzeros, then lowest row (sparselin.py:316)
  for (long long i = gt; i < r; i += GT) {
    const u32 s = rp[i], e = rp[i + 1];
    if (e > s) atomicMin(pk + col[s], ((unsigned long long)(e - s) << 32) | (unsigned long long)i);
  }
  grid.sync();
  // P2: column structure over this CTA's chunk; A-column bitmap by warp ballot
  {
    u32 na = 0;
    for (u32 c0 = c_lo; c0 < c_hi; c0 += blockDim.x) {
      const u32 c = c0 + tid;
      bool a = false;
      if (c < c_hi) {
        const unsigned long long k = __ldcg(pk + c);
        a = k != ~0ull;
        const u32 row = a ? (u32)(k & 0xFFFFFFFFull) : NONE;
        const u32 inv = a ? fp.inv(val[rp[row]]) : 0u;
        prow[c] = row;
        invl[c] = inv;
        desc[c] = a ? make_uint4(rp[row] + 1, rp[row + 1], inv, row) : make_uint4(0, 0, 0, NONE);
      }
      const unsigned bm = __ballot_sync(0xffffffffu, a);
      if (lane == 0 && c < c_hi) abits[c >> 5] = bm;
      na += a;
    }
    na = bsum(na);
    if (tid == 0) cnt[blockIdx.x] = na;
  }
  grid.sync();
  // P3: column positions; C-row flags counted per row chunk
  u32 baseA = 0, nA = 0;
  {
    u32 sb = 0, st = 0;
    for (u32 b = tid; b < G; b += blockDim.x) {
      const u32 v = __ldcg(cnt + b);
      st += v;
      if (b < blockIdx.x) sb += v;
    }
    baseA = bsum(sb);
    nA = bsum(st);
  }
  for (u32 c0 = c_lo; c0 < c_hi; c0 += blockDim.x) {
    const u32 c = c0 + tid;
    const bool a = c < c_hi && __ldcg(prow + c) != NONE;
    u32 tt;
    const u32 pre = block_scan_excl(a ? 1u : 0u, ws, &tt);
    if (c < c_hi) {
      const u32 pa = baseA + pre;  // A columns before c
      if (a) {
        acols[pa] = c;
        apos[c] = pa;
      } else {
        nonA[c - pa] = c;
      }
    }
    baseA += tt;
  }
  u32 nc = 0;
  for (u32 i = r_lo + tid; i < r_hi; i += blockDim.x) {
    const u32 s = rp[i], e = rp[i + 1];
    nc += (e > s && __ldcg(prow + col[s]) != i);
  }
  nc = bsum(nc);
  grid.sync();  // everyone has read cnt[] (column counts) before it is reused
  if (tid == 0) cnt[blockIdx.x] = nc;
  grid.sync();
  // P4: C rows, ascending
  u32 baseC = 0, nC = 0;
  {
    u32 sb = 0, st = 0;
    for (u32 b = tid; b < G; b += blockDim.x) {
      const u32 v = __ldcg(cnt + b);
      st += v;
      if (b < blockIdx.x) sb += v;
    }
    baseC = bsum(sb);
    nC = bsum(st);
  }
  for (u32 i0 = r_lo; i0 < r_hi; i0 += blockDim.x) {
    const u32 i = i0 + tid;
    bool isc = false;
    if (i < r_hi) {
      const u32 s = rp[i], e = rp[i + 1];
      isc = e > s && __ldcg(prow + col[s]) != i;
    }
    u32 tt;
    const u32 pre = block_scan_excl(isc ? 1u : 0u, ws, &tt);
    if (isc) crows[baseC + pre] = i;
    baseC += tt;
  }
  if (blockIdx.x == 0 && tid == 0) {
    out->nA = nA;
    out->nC = nC;
  }
}

// ---------------------------------------------------------------------------
// Block helpers
// ---------------------------------------------------------------------------
F4B_DEV u32 block_sum(u32 v, u32* red) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
#pragma unroll
  for (int o = 16; o; o >>= 1) v += __shfl_xor_sync(0xffffffffu, v, o);
  if (lane == 0) red[warp] = v;
  __syncthreads();
  u32 t = 0;
  if (threadIdx.x < 32) {
    t = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0;
#pragma unroll
    for (int o = 16; o; o >>= 1) t += __shfl_xor_sync(0xffffffffu, t, o);
    if (threadIdx.x == 0) red[32] = t;
  }
  __syncthreads();
  t = red[32];
  __syncthreads();
  return t;
}

// exclusive block scan of a 0/1 flag; returns prefix, total in *tot
F4B_DEV u32 block_scan_flag(u32 f, u32* red, u32* tot) {
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  unsigned b = __ballot_sync(0xffffffffu, f);
  u32 pre = __popc(b & lanemask_lt());
  if (lane == 0) red[warp] = __popc(b);
  __syncthreads();
  if (threadIdx.x < 32) {
    u32 x = threadIdx.x < (blockDim.x >> 5) ? red[threadIdx.x] : 0;
    u32 y = x;
#pragma unroll
    for (int o = 1; o < 32; o <<= 1) {
      u32 z = __shfl_up_sync(0xffffffffu, y, o);
      if (threadIdx.x >= o) y += z;
    }
    red[threadIdx.x] = y - x;
    if (threadIdx.x == 31) red[32] = y;
  }
  __syncthreads();
  u32 res = red[warp] + pre;
  *tot = red[32];
  __syncthreads();
  return res;
}

// Write the nonzeros of acc[lo, hi) (ascending) to the output pool.
template <typename T>
F4B_DEV void emit_row(const T* acc, u32 lo, u32 hi, const u32* __restrict__ colmap, u32* __restrict__ pcol,
                      u32* __restrict__ pval, size_t cap, unsigned long long* cursor, u32* slot_off, u32* slot_len,
                      u32* err, u32* red, u32* sh) {
  u32 cnt = 0;
  for (u32 c = lo + threadIdx.x; c < hi; c += blockDim.x) cnt += acc[c] != 0;
  cnt = block_sum(cnt, red);
  if (threadIdx.x == 0) {
    unsigned long long base = atomicAdd(cursor, (unsigned long long)cnt);
    if (base + cnt > cap) {
      atomicOr(err, (u32)DEVERR_CAPACITY);
      sh[0] = NONE;
    } else {
      sh[0] = (u32)base;
    }
    *slot_off = (u32)base;
    *slot_len = cnt;
  }
  __syncthreads();
  u32 base = sh[0];
  __syncthreads();
  if (base == NONE) return;
  for (u32 c0 = lo; c0 < hi; c0 += blockDim.x) {
    u32 c = c0 + threadIdx.x;
    u32 v = c < hi ? acc[c] : 0u;
    u32 tot;
    u32 p = block_scan_flag(v != 0, red, &tot);
    if (v) {
      pcol[base + p] = colmap ? colmap[c] : c;
      pval[base + p] = v;
    }
    base += tot;
  }
}

// ---------------------------------------------------------------------------
// E2 / E4: sparse sweep of a row over the A columns with a dense accumulator
// ---------------------------------------------------------------------------
// MODE 0: C rows  -> write the non-A part densely into Dp[slot][K]
// MODE 1: A rows  -> sweep right of the lead, reduce by RREF(D'), make monic, emit
// T: accumulator lane type (u16 when p < 2^16: half the shared memory, so
// more rows in flight and more L1 left for descriptor / pivot-row hits).
//
// One barrier per pivot: every warp scans for the next pivot itself (same
// data -> same answer) and takes the multiplier from its own ballot.  The
// scan reads columns >= cur only, while the update of pivot c writes
// columns > c only, so a warp still scanning can never see a different
// pivot; acc[c] is zeroed after the barrier, when no scan reads it.
template <int MODE, typename T>
__global__ void __launch_bounds__(SW_THREADS) k_sweep(
    Fp fp, const u32* __restrict__ rp, const u32* __restrict__ col, const u32* __restrict__ val, u32 N,
    const u32* __restrict__ rows, u32 nrows, const uint4* __restrict__ desc, const u32* __restrict__ invl,
    const u32* __restrict__ abits_g, T* __restrict__ gacc, u32* __restrict__ Dp, u32 K,
    const u32* __restrict__ nonA, const u32* __restrict__ Rd, u32 rankD, const u32* __restrict__ dpiv,
    u32* __restrict__ pcol, u32* __restrict__ pval, size_t cap, unsigned long long* cursor,
    u32* __restrict__ s_off, u32* __restrict__ s_len, u32* __restrict__ err, unsigned long long* __restrict__ stats) {
  extern __shared__ u32 smem[];
  const u32 nwords = (N + 31) / 32;
  u32* abits = smem;
  unsigned long long n_piv = 0, n_tail = 0;  // work counters (thread 0)
  T* acc = gacc ? gacc + (size_t)blockIdx.x * N : reinterpret_cast<T*>(smem + nwords);
  __shared__ u32 red[33];
  __shared__ u32 sh[4];
  __shared__ u32 coef_n;
  __shared__ u32 coef_k[256];
  __shared__ u32 coef_v[256];
  const int tid = threadIdx.x, lane = tid & 31;
  for (u32 w = tid; w < nwords; w += blockDim.x) abits[w] = abits_g[w];
  __syncthreads();
  for (u32 rr = blockIdx.x; rr < nrows; rr += gridDim.x) {
    const u32 i = rows[rr];
    const u32 s = rp[i], e = rp[i + 1];
    const u32 lead = col[s];
    for (u32 c = lead + tid; c < N; c += blockDim.x) acc[c] = 0;
    __syncthreads();
    for (u32 k = s + tid; k < e; k += blockDim.x) acc[col[k]] = (T)val[k];
    __syncthreads();
    // per-warp scan: next pivot column >= from, and acc at it (warp-uniform)
    auto scan = [&](u32 from, u32& value) -> u32 {
      for (u32 c0 = from & ~31u; c0 < N; c0 += 32) {
        const u32 cc = c0 + lane;
        const u32 v = (cc >= from && cc < N) ? (u32)acc[cc] : 0u;
        const bool hit = v != 0 && ((abits[cc >> 5] >> (cc & 31)) & 1u);
        const unsigned b = __ballot_sync(0xffffffffu, hit);
        if (b) {
          const int src = __ffs(b) - 1;
          value = __shfl_sync(0xffffffffu, v, src);
          return c0 + src;
        }
      }
      return N;
    };
    u32 av = 0;
    u32 c = scan(MODE == 1 ? lead + 1 : lead, av);
    while (c < N) {
      const uint4 d = __ldg(desc + c);
      const u32 fm = fp.to_mont(fp.neg(fp.mul(av, d.z)));
      if (tid == 0) {
        ++n_piv;
        n_tail += d.y - d.x;
      }
      u32 k = d.x + tid;
      for (; k + blockDim.x < d.y; k += 2 * blockDim.x) {
        const u32 c0 = __ldg(col + k), c1 = __ldg(col + k + blockDim.x);
        const u32 v0 = __ldg(val + k), v1 = __ldg(val + k + blockDim.x);
        acc[c0] = (T)fp.add((u32)acc[c0], fp.mont_mul(fm, v0));
        acc[c1] = (T)fp.add((u32)acc[c1], fp.mont_mul(fm, v1));
      }
      if (k < d.y) {
        const u32 cc = __ldg(col + k);
        acc[cc] = (T)fp.add((u32)acc[cc], fp.mont_mul(fm, __ldg(val + k)));
      }
      __syncthreads();
      if (tid == 0) acc[c] = 0;
      c = scan(c + 1, av);
    }
    __syncthreads();
    if (MODE == 0) {
      u32* out = Dp + (size_t)rr * K;
      for (u32 q = tid; q < K; q += blockDim.x) {
        const u32 cc = nonA[q];
        out[q] = cc >= lead ? (u32)acc[cc] : 0u;
      }
      __syncthreads();
    } else {
      // one-shot reduction by RREF(D'): coefficients at D' pivot columns
      for (u32 k0 = 0; k0 < rankD; k0 += 256) {
        if (tid == 0) coef_n = 0;
        __syncthreads();
        for (u32 k = k0 + tid; k < min(rankD, k0 + 256); k += blockDim.x) {
          const u32 cc = nonA[dpiv[k]];
          const u32 v = cc > lead ? (u32)acc[cc] : 0u;
          if (v) {
            u32 slot = atomicAdd(&coef_n, 1u);
            coef_k[slot] = k;
            coef_v[slot] = fp.to_mont(fp.neg(v));
          }
        }
        __syncthreads();
        const u32 nco = coef_n;
        if (nco) {
          for (u32 q = tid; q < K; q += blockDim.x) {
            const u32 cc = nonA[q];
            if (cc <= lead) continue;
            u32 a = (u32)acc[cc];
            for (u32 t = 0; t < nco; ++t) a = fp.add(a, fp.mont_mul(coef_v[t], __ldg(Rd + (size_t)coef_k[t] * K + q)));
            acc[cc] = (T)a;
          }
        }
        __syncthreads();
      }
      // monic: the lead coefficient is untouched by the sweep
      const u32 inv = invl[lead];
      for (u32 c2 = lead + tid; c2 < N; c2 += blockDim.x) {
        const u32 v = (u32)acc[c2];
        if (v) acc[c2] = (T)fp.mul(v, inv);
      }
      __syncthreads();
      emit_row<T>(acc, lead, N, nullptr, pcol, pval, cap, cursor, s_off + rr, s_len + rr, err, red, sh + 1);
      __syncthreads();
    }
  }
  if (stats && tid == 0 && n_piv) {
    atomicAdd(stats, n_piv);
    atomicAdd(stats + 1, n_tail);
  }
}

// ---------------------------------------------------------------------------
// E2, blocked: one CTA per C row, pivots taken 32 A-columns at a time.
// The sequential dependency between pivots only runs through the A columns,
// so for a window of BW consecutive A columns (starting at the first nonzero
// one) the multipliers come from a BW x BW unit-triangular solve in one warp
// (the pivot rows' in-window entries staged densely in shared memory), and
// the rest of every active pivot tail is applied afterwards by the whole CTA
// at once (shared-memory atomicAdd into a lazily reduced u32 accumulator: each
// product is < p, a column receives at most nA of them, and p * nA < 2^32 is
// checked on the host).  Three CTA barriers per window instead of one per
// pivot application.  Same multipliers as the column-by-column sweep, so the
// D' row is bit-identical.
// ---------------------------------------------------------------------------
static constexpr int BW = 32;
__global__ void __launch_bounds__(256) k_sweep_blk(Fp fp, u32 mu, const u32* __restrict__ rp,
                                                   const u32* __restrict__ col, const u32* __restrict__ val, u32 N,
                                                   const u32* __restrict__ rows, u32 nrows,
                                                   const uint4* __restrict__ desc, const u32* __restrict__ abits_g,
                                                   const u32* __restrict__ acols, const u32* __restrict__ apos,
                                                   u32 nA, u32* __restrict__ Dp, u32 K, const u32* __restrict__ nonA,
                                                   unsigned long long* __restrict__ stats) {
  extern __shared__ __align__(16) u32 smem[];
  constexpr int NWARP = 8;
  constexpr u32 PENDING = 0xFFFFFFFFu;
  const u32 nwords = (N + 31) / 32;
  u32* abits = smem;
  u32* acc = smem + ((nwords + 3) & ~3u);
  __shared__ u32 s_cw[NWARP][BW];  // window columns (a per-warp copy)
  __shared__ uint4 s_dw[BW];       // window pivot descriptors
  __shared__ u32 s_X[BW];          // inverse leads times R^2 (Montgomery)
  __shared__ u32 s_P[BW][BW + 1];  // in-window entries of the window pivots
  __shared__ u32 s_m[BW];          // multipliers (Montgomery), PENDING until solved
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u32 p = fp.p;
  auto red = [&](u32 v) -> u32 {  // v mod p for v < 2^32 (Barrett, mu = floor(2^32 / p))
    const u32 r = v - __umulhi(v, mu) * p;
    return r >= p ? r - p : r;
  };
  volatile u32* vm = s_m;
  for (u32 w = tid; w < nwords; w += blockDim.x) abits[w] = abits_g[w];
  for (u32 q = tid; q < BW * (BW + 1); q += blockDim.x) (&s_P[0][0])[q] = 0;
  if (tid < BW) s_m[tid] = PENDING;
  __syncthreads();
  unsigned long long n_piv = 0, n_tail = 0;
  for (u32 rr = blockIdx.x; rr < nrows; rr += gridDim.x) {
    const u32 i = rows[rr];
    const u32 s = rp[i], e = rp[i + 1];
    const u32 lead = col[s];
    for (u32 c = lead + tid; c < N; c += blockDim.x) acc[c] = 0;
    __syncthreads();
    for (u32 k = s + tid; k < e; k += blockDim.x) acc[col[k]] = val[k];
    __syncthreads();
    u32 from = lead;
    while (true) {
      // (1) every warp: window start = first nonzero A column >= from, the
      // BW A columns from there (same data, same answer in every warp)
      u32 c = N;
      for (u32 c0 = from & ~31u; c0 < N; c0 += 32) {
        const u32 cc = c0 + lane;
        const bool hit = cc >= from && cc < N && ((abits[cc >> 5] >> (cc & 31)) & 1u) && red(acc[cc]) != 0;
        const unsigned b = __ballot_sync(0xffffffffu, hit);
        if (b) {
          c = c0 + __ffs(b) - 1;
          break;
        }
      }
      if (c >= N) break;
      const u32 a0 = __ldg(apos + c);
      const u32 nw = min((u32)BW, nA - a0);
      const u32 cw = (u32)lane < nw ? __ldg(acols + a0 + lane) : 0xFFFFFFFFu;
      s_cw[warp][lane] = cw;
      const u32 clast = __shfl_sync(0xffffffffu, cw, nw - 1);
      __syncwarp();
      // (2) stage the in-window entries P[t][u] of the window pivots (rows of
      // P were cleared by the same warp after their last use)
      for (u32 t = warp; t < nw; t += NWARP) {
        const uint4 d = __ldg(desc + s_cw[warp][t]);
        if (lane == 0) {
          s_dw[t] = d;
          s_X[t] = fp.to_mont(fp.to_mont(d.z));
        }
        for (u32 k0 = d.x; k0 < d.y; k0 += 32) {
          const u32 k = k0 + lane;
          const u32 cc = k < d.y ? __ldg(col + k) : 0xFFFFFFFFu;
          if (cc <= clast && ((abits[cc >> 5] >> (cc & 31)) & 1u)) {
            u32 lo = 0, hi = nw;  // position of cc among the window columns
            while (lo + 1 < hi) {
              const u32 mid = (lo + hi) >> 1;
              if (s_cw[warp][mid] <= cc) lo = mid; else hi = mid;
            }
            s_P[t][lo] = __ldg(val + k);
          }
          if (__shfl_sync(0xffffffffu, cc, 31) > clast) break;
        }
      }
      __syncthreads();
      if (warp == 0) {
        // (3) unit-triangular solve; lane u holds the value of column u; each
        // multiplier is published as soon as it is known
        u32 v = (u32)lane < nw ? red(acc[cw]) : 0u;
        for (u32 t = 0; t < nw; ++t) {
          const u32 vt = __shfl_sync(0xffffffffu, v, t);
          u32 m = 0;
          if (vt) {
            m = fp.mont_mul(p - vt, s_X[t]);  // -(v_t / lead_t), Montgomery form
            if ((u32)lane > t) v = fp.add(v, fp.mont_mul(m, s_P[t][lane]));
          }
          if (lane == 0) vm[t] = m;
        }
      } else {
        // (4) meanwhile: the rest of each published tail — columns right of
        // the window and the non-A columns inside it
        for (u32 t = warp - 1; t < nw; t += NWARP - 1) {
          u32 m;
          while ((m = vm[t]) == PENDING) {
          }
          if (!m) continue;
          const uint4 d = s_dw[t];
          ++n_piv;
          n_tail += d.y - d.x;
          for (u32 k0 = d.x; k0 < d.y; k0 += 32 * 4) {
            u32 cc[4], vv[4];
#pragma unroll
            for (int z = 0; z < 4; ++z) {
              const u32 k = k0 + z * 32 + lane;
              cc[z] = k < d.y ? __ldg(col + k) : N;
              vv[z] = k < d.y ? __ldg(val + k) : 0u;
            }
#pragma unroll
            for (int z = 0; z < 4; ++z) {
              const u32 cz = cc[z];
              if (cz < N && (cz > clast || !((abits[cz >> 5] >> (cz & 31)) & 1u)))
                atomicAdd(acc + cz, fp.mont_mul(m, vv[z]));
            }
          }
        }
      }
      __syncthreads();
      // clear the window state: P rows (by their staging warp), multipliers
      for (u32 t = warp; t < nw; t += NWARP) s_P[t][lane] = 0;
      if (tid < BW) s_m[tid] = PENDING;
      from = clast + 1;
    }
    u32* out = Dp + (size_t)rr * K;
    for (u32 q = tid; q < K; q += blockDim.x) {
      const u32 cc = nonA[q];
      out[q] = cc >= lead ? red(acc[cc]) : 0u;
    }
    __syncthreads();
  }
  if (stats && lane == 0 && n_piv) {
    atomicAdd(stats, n_piv);
    atomicAdd(stats + 1, n_tail);
  }
}

// ---------------------------------------------------------------------------
// E2, fixed windows with precomputed block inverses.
//
// The A columns are cut into FIXED windows of 32 consecutive A columns
// (acols[32j .. 32j+32)).  Inside window j the pivot rows form an upper
// triangular block T_j (diagonal = lead coefficients, above it the pivot
// rows' entries at the window's A columns).  Sweeping a row over window j
// with values v (the row's entries at the window columns) produces the
// multipliers m with  m T_j = -v,  i.e.  m = v W_j  with  W_j = -T_j^{-1}.
// T_j depends only on the pivot rows, so W_j is built ONCE per matrix
// (k_win_build, one warp per window) instead of being re-derived by a serial
// 32-step solve in every C row; a C row then gets all 32 multipliers from one
// 32x32 vector-matrix product (independent lanes, no serial chain, every warp
// computes them itself: no barrier between solve and apply), and the active
// pivots' tails are applied by the whole CTA as one flat list of 4-entry
// groups (all loads of a window in flight at once).  One CTA barrier per
// non-empty window.  The multipliers equal the column-by-column sweep's, so
// D' is bit-identical with k_sweep<0> / k_sweep_blk.
// ---------------------------------------------------------------------------
// k_tail_copy: one warp per A column (pivot a = 32 j + t of window j) walks
// its pivot row's tail once, coalesced: reserves ceil(len / 4) packed groups
// (winD[a]; any placement works, the sweep follows winD), copies the tail
// into them (PK: (col << 16 | val) in one u32 when N, p < 2^16, else
// (col, val) pairs; padding points at the dummy accumulator slot N with value
// 0), and scatters the tail's in-window entries (A columns of window j, a
// prefix of the tail) into the window's dense block T_j (Montgomery) and its
// row masks.  k_win_build then only solves: the in-window prefixes were a
// serial chain of dependent L2 loads per pivot there (~30 us per launch).
template <bool PK>
__global__ void __launch_bounds__(256) k_tail_copy(Fp fp, const u32* __restrict__ col, const u32* __restrict__ val,
                                                   u32 N, const uint4* __restrict__ desc,
                                                   const u32* __restrict__ abits, const u32* __restrict__ acols,
                                                   const u32* __restrict__ apos, const u32* __restrict__ pnA, u32 nA,
                                                   uint2* __restrict__ winD, u32* __restrict__ gcursor,
                                                   u32* __restrict__ winT, u32* __restrict__ winM,
                                                   typename std::conditional<PK, u32, uint2>::type* __restrict__ tails) {
  const int lane = threadIdx.x & 31;
  const u32 a = blockIdx.x * 8 + (threadIdx.x >> 5);
  if (pnA) nA = *pnA;  // enqueued before the host knows nA (grid sized by N)
  if (a >= nA) return;
  const u32 j = a >> 5, t = a & 31;
  const u32 cw = __ldg(acols + a);
  const u32 clast = __ldg(acols + min(32 * j + 31, nA - 1));
  const uint4 d = __ldg(desc + cw);
  const u32 len = d.y - d.x, ng = (len + 3) >> 2, n4 = 4 * ng;
  u32 g0 = 0;
  if (lane == 0) g0 = atomicAdd(gcursor, ng);
  g0 = __shfl_sync(0xffffffffu, g0, 0);
  if (lane == 0) winD[a] = make_uint2(g0, g0 + ng);
  u32 mask = 0;
  for (u32 k0 = 0; k0 < n4; k0 += 128) {
    u32 cc[4], vv[4];
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const u32 k = k0 + q * 32 + lane;
      cc[q] = k < len ? __ldg(col + d.x + k) : N;
      vv[q] = k < len ? __ldg(val + d.x + k) : 0u;
    }
#pragma unroll
    for (int q = 0; q < 4; ++q) {
      const u32 k = k0 + q * 32 + lane;
      if (k < n4) {
        if constexpr (PK) tails[(size_t)4 * g0 + k] = (cc[q] << 16) | vv[q];
        else tails[(size_t)4 * g0 + k] = make_uint2(cc[q], vv[q]);
      }
      if (cc[q] <= clast && ((__ldg(abits + (cc[q] >> 5)) >> (cc[q] & 31)) & 1u)) {
        const u32 u = __ldg(apos + cc[q]) - 32 * j;
        winT[(size_t)j * 1024 + t * 32 + u] = fp.to_mont(vv[q]);
        mask |= 1u << u;
      }
    }
  }
#pragma unroll
  for (int o = 16; o; o >>= 1) mask |= __shfl_xor_sync(0xffffffffu, mask, o);
  if (lane == 0) winM[a] = mask;
}

// Block inverses W_j = -T_j^{-1} (one warp per window, T_j from k_tail_copy):
// lane s solves x T = e_s right-looking (Montgomery domain), its vector in
// shared memory (sA[u][s], conflict free; a rolled loop keeps the code in the
// instruction cache): x_t = a_t / lead_t, then a_u -= x_t T[t][u].
static constexpr int WB_WARPS = 4;
__global__ void __launch_bounds__(32 * WB_WARPS) k_win_build(Fp fp, u32 N, const uint4* __restrict__ desc,
                                                             const u32* __restrict__ acols,
                                                             const u32* __restrict__ pnA, u32 nA,
                                                             const u32* __restrict__ winT,
                                                             const u32* __restrict__ winM, u32* __restrict__ winW,
                                                             u32* __restrict__ winC) {
  __shared__ u32 sT[WB_WARPS][32][33];  // T[r][t] (Montgomery): pivot r's entry at window column t (r < t)
  __shared__ u32 sA[WB_WARPS][32][33];  // sA[u][s]: lane s's working vector
  __shared__ u32 sM[WB_WARPS][32];      // nonzero pattern of T's row r
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  const u32 j = blockIdx.x * WB_WARPS + warp;
  if (pnA) nA = *pnA;
  const u32 nwin = (nA + 31) / 32;
  if (j >= nwin) return;
  const unsigned FULL = 0xffffffffu;
  const u32 base = j * 32;
  const u32 nw = min(32u, nA - base);
  const u32 cw = (u32)lane < nw ? __ldg(acols + base + lane) : N;
  const uint4 d = (u32)lane < nw ? __ldg(desc + cw) : make_uint4(0, 0, 1, NONE);
  winC[base + lane] = cw;
  sM[warp][lane] = (u32)lane < nw ? __ldg(winM + base + lane) : 0u;
#pragma unroll 8
  for (int r = 0; r < 32; ++r) sT[warp][r][lane] = __ldg(winT + (size_t)j * 1024 + r * 32 + lane);
  __syncwarp();
  const u32 ilm_l = fp.to_mont(d.z);
  const u32 one_m = fp.to_mont(1u);
  for (int u = 0; u < 32; ++u) sA[warp][u][lane] = lane == u ? one_m : 0u;
  __syncwarp();
  for (int t = 0; t < 32; ++t) {
    const u32 xt = fp.mont_mul(sA[warp][t][lane], __shfl_sync(FULL, ilm_l, t));
    sA[warp][t][lane] = xt;
    // the nonzeros of row t only, four independent updates in flight
    for (u32 mk = sM[warp][t]; mk;) {
      int u[4];
#pragma unroll
      for (int q = 0; q < 4; ++q) {
        u[q] = mk ? __ffs(mk) - 1 : -1;
        mk &= mk - 1;
      }
      u32 a4[4], t4[4];
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (u[q] >= 0) {
          a4[q] = sA[warp][u[q]][lane];
          t4[q] = sT[warp][t][u[q]];
        }
#pragma unroll
      for (int q = 0; q < 4; ++q)
        if (u[q] >= 0) sA[warp][u[q]][lane] = fp.sub(a4[q], fp.mont_mul(xt, t4[q]));
    }
  }
  __syncwarp();
  // W[s][t] = -x^{(s)}_t times R^2: mont_mul(v_s, W[s][t]) summed over s is
  // the multiplier m_t in Montgomery form
#pragma unroll 8
  for (u32 s = 0; s < 32; ++s) {
    const u32 xm = (s < nw && (u32)lane < nw) ? sA[warp][lane][s] : 0u;
    winW[(size_t)j * 1024 + s * 32 + lane] = fp.to_mont(fp.neg(xm));
  }
}

// MODE 0: C rows -> D' (dense rows over the non-A columns).  MODE 1 (full
// RREF only): the pivot rows themselves, each swept from just after its own
// lead (the window solve gives its own and earlier pivots zero multipliers),
// then reduced in one step by RREF(D') (one coefficient per D' pivot),
// made monic and emitted as sparse rows — the back-reduction of
// sparselin.py:337-349 with the same window machinery as the C rows.
struct SweepOut {
  const u32* invl;
  const u32* Rd;
  u32 rankD;
  const u32* dpiv;
  u32* pcol;
  u32* pval;
  size_t cap;
  unsigned long long* cursor;
  u32* s_off;
  u32* s_len;
  u32* err;
  unsigned long long* tr;  // trace (F4B_SWEEP_TRACE): rows, windows, misses, cycles find | mult | apply | out
};
template <bool PK, int MODE, bool TR = false>
__global__ void __launch_bounds__(256) k_sweep_win(Fp fp, u32 mu, const u32* __restrict__ rp,
                                                   const u32* __restrict__ col, const u32* __restrict__ val, u32 N,
                                                   const u32* __restrict__ rows, u32 nrows,
                                                   const u32* __restrict__ abits_g, const u32* __restrict__ winW,
                                                   const u32* __restrict__ winC, const uint2* __restrict__ winD,
                                                   u32 nwin, const uint4* __restrict__ tails,
                                                   u32* __restrict__ Dp, u32 K, const u32* __restrict__ nonA,
                                                   unsigned long long* __restrict__ stats, const SweepOut so) {
  extern __shared__ __align__(16) u32 smem[];
  constexpr int NWARP = 8;
  constexpr int H = 4;  // 32-group spans per warp in flight
  const u32 nwords = (N + 31) / 32;
  u32* abits = smem;
  u32* apre = smem + nwords;  // A columns before word w
  u32* acc = smem + ((2 * nwords + 3) & ~3u);  // N + 1 slots (slot N absorbs padding)
  __shared__ u32 s_act[NWARP][32];
  __shared__ u32 s_ms[32], s_msh[32], s_ng[32], s_g0[32];
  __shared__ u32 s_cn, s_ck[MODE == 1 ? 256 : 1], s_cv[MODE == 1 ? 256 : 1], s_red[33], s_sh[4];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u32 p = fp.p;
  auto red = [&](u32 v) -> u32 {  // v mod p for v < 2^32 (Barrett, mu = floor(2^32 / p))
    const u32 r = v - __umulhi(v, mu) * p;
    return r >= p ? r - p : r;
  };
  const unsigned long long pinv64 = ~0ull / p;  // Shoup constants below without a 64-bit division
  for (u32 w = tid; w < nwords; w += blockDim.x) abits[w] = abits_g[w];
  __syncthreads();
  if (warp == 0) {
    u32 run = 0;
    for (u32 w0 = 0; w0 < nwords; w0 += 32) {
      const u32 w = w0 + lane;
      const u32 c = w < nwords ? __popc(abits[w]) : 0u;
      u32 x = c;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      if (w < nwords) apre[w] = run + x - c;
      run += __shfl_sync(0xffffffffu, x, 31);
    }
  }
  __syncthreads();
  unsigned long long n_piv = 0, n_tail = 0;
  for (u32 rr = blockIdx.x; rr < nrows; rr += gridDim.x) {
    const u32 i = rows[rr];
    const u32 s = rp[i], e = rp[i + 1];
    const u32 lead = col[s];
    for (u32 c = lead + tid; c <= N; c += blockDim.x) acc[c] = 0;
    __syncthreads();
    for (u32 k = s + tid; k < e; k += blockDim.x) acc[col[k]] = val[k];
    __syncthreads();
    u32 from = MODE == 1 ? lead + 1 : lead;
    unsigned long long tq0 = 0, tw = 0, tmiss = 0, tcf = 0, tcm = 0, tca = 0, tcfind = 0, tcv = 0, tqf = 0;
    const bool trc = TR && so.tr && tid == 0;  // TR: trace build only (the counters cost registers)
    if (trc) tq0 = clock64();
    u32 pj = 0xFFFFFFFFu, pcw = 0;
    uint2 pdd = make_uint2(0, 0);
    uint4 pw4 = make_uint4(0, 0, 0, 0);
    while (true) {
      // next nonzero A column >= from (every warp, same answer)
      // (128 columns per step: four independent ballots, then the first hit)
      u32 c = N;
      for (u32 c0 = from & ~31u; c0 < N; c0 += 128) {
        unsigned b[4];
#pragma unroll
        for (int q = 0; q < 4; ++q) {
          const u32 cc = c0 + 32 * q + lane;
          const bool hit = cc >= from && cc < N && ((abits[cc >> 5] >> (cc & 31)) & 1u) && red(acc[cc]) != 0;
          b[q] = __ballot_sync(0xffffffffu, hit);
        }
        if (b[0] | b[1] | b[2] | b[3]) {
          const int q = b[0] ? 0 : b[1] ? 1 : b[2] ? 2 : 3;
          c = c0 + 32 * q + __ffs(q == 0 ? b[0] : q == 1 ? b[1] : q == 2 ? b[2] : b[3]) - 1;
          break;
        }
      }
      if (c >= N) break;
      const u32 j = (apre[c >> 5] + __popc(abits[c >> 5] & ((1u << (c & 31)) - 1u))) >> 5;
      if (trc) {
        ++tw;
        tmiss += j != pj;
        tqf = clock64();
        tcfind += tqf - tq0;
      }
      // this window's columns, tail groups and block-inverse slice: from the
      // registers if the previous window prefetched them (the usual case:
      // consecutive windows), then the next window's are prefetched so their
      // L2 latency hides behind this window's product and tail application
      u32 cw;
      uint2 dd;
      uint4 w4;
      if (j == pj) {
        cw = pcw;
        dd = pdd;
        w4 = pw4;
      } else {
        cw = __ldg(winC + j * 32 + lane);
        dd = __ldg(winD + j * 32 + lane);
        w4 = __ldg(reinterpret_cast<const uint4*>(winW + (size_t)j * 1024 + lane * 32) + warp);
      }
      if (j + 1 < nwin) {
        pj = j + 1;
        pcw = __ldg(winC + pj * 32 + lane);
        pdd = __ldg(winD + pj * 32 + lane);
        pw4 = __ldg(reinterpret_cast<const uint4*>(winW + (size_t)pj * 1024 + lane * 32) + warp);
      } else {
        pj = 0xFFFFFFFFu;
      }
      const u32 v = (cw < N && (MODE == 1 ? cw > lead : cw >= lead)) ? red(acc[cw]) : 0u;
      if (trc) {
        const u32 vv = v;
        asm volatile("" ::"r"(vv), "r"(w4.x), "r"(dd.x));  // v, window data ready
        tcv += clock64() - tqf;
      }
      // multipliers m = v W, split over the 8 warps: warp w owns pivots
      // t = 4w .. 4w+3 (lane s contributes v_s W[s][t], one 16-byte load),
      // warp sums, then Shoup constants and group counts into shared memory
      {
        u32 part[4] = {v ? fp.mont_mul(v, w4.x) : 0u, v ? fp.mont_mul(v, w4.y) : 0u, v ? fp.mont_mul(v, w4.z) : 0u,
                       v ? fp.mont_mul(v, w4.w) : 0u};
#pragma unroll
        for (int o = 16; o; o >>= 1)
#pragma unroll
          for (int i = 0; i < 4; ++i) part[i] = fp.add(part[i], __shfl_xor_sync(0xffffffffu, part[i], o));
        const u32 t = 4 * warp + (lane & 3);
        const uint2 dt = make_uint2(__shfl_sync(0xffffffffu, dd.x, t), __shfl_sync(0xffffffffu, dd.y, t));
        if (lane < 4) {
          const u32 mt = lane == 0 ? part[0] : lane == 1 ? part[1] : lane == 2 ? part[2] : part[3];
          // standard-domain multiplier and its Shoup constant floor(ms 2^32 / p):
          // ms * x mod p is then x*ms - umulhi(x, msh)*p, in [0, 2p)
          const u32 ms = fp.mont_mul(mt, 1u);
          s_ms[t] = ms;
          // floor(ms 2^32 / p) from the 64-bit reciprocal (no division):
          // the estimate is short by at most one
          u32 q = 0;
          if (ms) {
            const unsigned long long X = (unsigned long long)ms << 32;
            unsigned long long qe = __umul64hi(X, pinv64);
            if (X - qe * p >= p) ++qe;
            q = (u32)qe;
          }
          s_msh[t] = q;
          s_ng[t] = ms ? dt.y - dt.x : 0u;
          s_g0[t] = dt.x;
        }
      }
      unsigned long long tq1 = 0;
      if (trc) {
        tq1 = clock64();
        tcf += tq1 - tq0;  // find + window data + multipliers (this thread)
      }
      __syncthreads();
      if (trc) {
        const unsigned long long tq2 = clock64();
        tcm += tq2 - tq1;  // barrier after the multipliers
        tq0 = tq2;
      }
      const u32 ng = s_ng[lane], ms = s_ms[lane], msh = s_msh[lane];
      u32 x = ng;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, x, o);
        if (lane >= o) x += y;
      }
      const u32 tot = __shfl_sync(0xffffffffu, x, 31);
      const u32 off = x - ng;
      const unsigned act = __ballot_sync(0xffffffffu, ng != 0);
      if (ng) s_act[warp][__popc(act & lanemask_lt())] = lane;
      if (warp == 0 && lane == 0) {
        n_piv += __popc(act);
        n_tail += 4ull * tot;
      }
      const uint2 dd_g = make_uint2(s_g0[lane], 0u);
      __syncwarp();
      // apply: the active pivots' groups as one flat list [0, tot); warp w
      // takes spans of 32 consecutive groups, lane L group a0 + L; the pivot
      // owning a group from ballots over the pivots' offsets (no search)
      for (u32 b0 = 0; b0 < tot; b0 += 256 * H) {
        uint4 ev[H][PK ? 1 : 2];
        u32 mss[H], mhs[H];
#pragma unroll
        for (int h = 0; h < H; ++h) {
          const u32 a0 = b0 + 256 * h + 32 * warp;  // warp-uniform
          const u32 a = a0 + lane;
          mss[h] = 0;
          mhs[h] = 0;
          if (a0 < tot) {
            const int k0 = __popc(__ballot_sync(0xffffffffu, ng && off <= a0)) - 1;
            unsigned sm = __ballot_sync(0xffffffffu, ng && off > a0 && off < a0 + 32);
            int cnt = 0;
            while (sm) {
              const int t = __ffs(sm) - 1;
              sm &= sm - 1;
              cnt += a >= __shfl_sync(0xffffffffu, off, t);
            }
            const int t = s_act[warp][min(k0 + cnt, 31)];
            const u32 offt = __shfl_sync(0xffffffffu, off, t);
            const u32 g0 = __shfl_sync(0xffffffffu, dd_g.x, t);
            const u32 mt = __shfl_sync(0xffffffffu, ms, t), mh = __shfl_sync(0xffffffffu, msh, t);
            if (a < tot) {
              const size_t g = (size_t)g0 + (a - offt);
              if constexpr (PK) {
                ev[h][0] = __ldg(tails + g);
              } else {
                ev[h][0] = __ldg(tails + 2 * g);
                ev[h][1] = __ldg(tails + 2 * g + 1);
              }
              mss[h] = mt;
              mhs[h] = mh;
            }
          }
        }
#pragma unroll
        for (int h = 0; h < H; ++h) {
          if (!mss[h]) continue;
          u32 cc[4], vv[4];
          if constexpr (PK) {
            const u32 w4[4] = {ev[h][0].x, ev[h][0].y, ev[h][0].z, ev[h][0].w};
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              cc[q] = w4[q] >> 16;
              vv[q] = w4[q] & 0xFFFFu;
            }
          } else {
            cc[0] = ev[h][0].x; vv[0] = ev[h][0].y; cc[1] = ev[h][0].z; vv[1] = ev[h][0].w;
            cc[2] = ev[h][1].x; vv[2] = ev[h][1].y; cc[3] = ev[h][1].z; vv[3] = ev[h][1].w;
          }
#pragma unroll
          for (int q = 0; q < 4; ++q)
            atomicAdd(acc + cc[q], vv[q] * mss[h] - __umulhi(vv[q], mhs[h]) * p);
        }
      }
      __syncthreads();
      if (trc) {
        const unsigned long long tq3 = clock64();
        tca += tq3 - tq0;  // apply + barrier
        tq0 = tq3;
      }
      from = __reduce_max_sync(0xffffffffu, cw < N ? cw : 0u) + 1;
    }
    if (trc) {
      atomicAdd(so.tr + 0, 1ull);
      atomicAdd(so.tr + 1, tw);
      atomicAdd(so.tr + 2, tmiss);
      atomicAdd(so.tr + 3, tcf);
      atomicAdd(so.tr + 4, tcm);
      atomicAdd(so.tr + 5, tca);
      atomicAdd(so.tr + 6, clock64() - tq0);
      atomicAdd(so.tr + 7, tcfind);
      atomicAdd(so.tr + 8, tcv);
    }
    if (MODE == 0) {
      u32* out = Dp + (size_t)rr * K;
      for (u32 q = tid; q < K; q += blockDim.x) {
        const u32 cc = nonA[q];
        out[q] = cc >= lead ? red(acc[cc]) : 0u;
      }
      __syncthreads();
    } else {
      // reduce right of the lead (the lazy sums), then one step by RREF(D'):
      // x <- x - sum_k x[D' pivot k] R_k (R in reduced echelon form)
      // (the A columns right of the lead are eliminated: the window sweep
      // leaves stale partial sums there, which are cleared, not read)
      for (u32 c2 = lead + 1 + tid; c2 < N; c2 += blockDim.x)
        acc[c2] = ((abits[c2 >> 5] >> (c2 & 31)) & 1u) ? 0u : red(acc[c2]);
      __syncthreads();
      for (u32 k0 = 0; k0 < so.rankD; k0 += 256) {
        if (tid == 0) s_cn = 0;
        __syncthreads();
        for (u32 k = k0 + tid; k < min(so.rankD, k0 + 256); k += blockDim.x) {
          const u32 cc = nonA[so.dpiv[k]];
          const u32 v = cc > lead ? acc[cc] : 0u;
          if (v) {
            const u32 slot = atomicAdd(&s_cn, 1u);
            s_ck[slot] = k;
            s_cv[slot] = fp.to_mont(fp.neg(v));
          }
        }
        __syncthreads();
        const u32 nco = s_cn;
        if (nco)
          for (u32 q = tid; q < K; q += blockDim.x) {
            const u32 cc = nonA[q];
            if (cc <= lead) continue;
            u32 x = acc[cc];
            if (PK) {  // p < 2^16: raw Montgomery-coefficient products summed in 64 bits (< 256 p^2), one REDC
              unsigned long long a = 0;
              for (u32 t = 0; t < nco; ++t) a += (unsigned long long)s_cv[t] * __ldg(so.Rd + (size_t)s_ck[t] * K + q);
              const u32 m = (u32)a * fp.pprime;
              const unsigned long long u = (a + (unsigned long long)m * p) >> 32;
              x = fp.add(x, (u32)(u >= p ? u - p : u));
            } else {
              for (u32 t = 0; t < nco; ++t) x = fp.add(x, fp.mont_mul(s_cv[t], __ldg(so.Rd + (size_t)s_ck[t] * K + q)));
            }
            acc[cc] = x;
          }
        __syncthreads();
      }
      // monic (the lead is untouched by the sweep), then the sparse row
      const u32 inv = so.invl[lead];
      if (tid == 0) acc[lead] = fp.mul(red(acc[lead]), inv);
      for (u32 c2 = lead + 1 + tid; c2 < N; c2 += blockDim.x) {
        const u32 v = acc[c2];
        if (v) acc[c2] = fp.mul(v, inv);
      }
      __syncthreads();
      emit_row<u32>(acc, lead, N, nullptr, so.pcol, so.pval, so.cap, so.cursor, so.s_off + rr, so.s_len + rr, so.err,
                    s_red, s_sh + 1);
      __syncthreads();
    }
  }
  if (stats && tid == 0 && n_piv) {
    atomicAdd(stats, n_piv);
    atomicAdd(stats + 1, n_tail);
  }
}

// ---------------------------------------------------------------------------
// E3a: cooperative forward elimination of the dense block D' (R x K)
// ---------------------------------------------------------------------------
// One grid barrier per PIVOT (not per column): every CTA keeps the leading
// column of its live rows; the next pivot is the global minimum of
// (lead << 32 | row), published with one 64-bit atomicMin per CTA.  Pivot
// rows are frozen once chosen, so other CTAs read them without a second
// barrier.  Grid barriers = rank(D') + 1.
// row[q] += fm * prow[q] for q = q0, q0+32, ... < K — 8 independent L2 loads in
// flight per lane (the pivot row lives in L2; the un-pipelined loop was
// latency bound).
__device__ __forceinline__ void row_axpy8(const Fp& fp, u32* row, const u32* prow, u32 fm, u32 q0, u32 K) {
  for (u32 qb = q0; qb < K; qb += 32 * 8) {
    u32 pv[8], rv[8];
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const u32 q = qb + 32 * j;
      pv[j] = q < K ? __ldcg(prow + q) : 0u;
      rv[j] = q < K ? row[q] : 0u;
    }
#pragma unroll
    for (int j = 0; j < 8; ++j) {
      const u32 q = qb + 32 * j;
      if (q < K) row[q] = fp.add(rv[j], fp.mont_mul(fm, pv[j]));
    }
  }
}

__device__ __forceinline__ u32 first_nonzero_warp(const u32* row, u32 from, u32 K) {
  const int lane = threadIdx.x & 31;
  for (u32 b0 = from & ~31u; b0 < K; b0 += 32) {
    const u32 q = b0 + lane;
    const bool nz = q >= from && q < K && row[q] != 0;
    const unsigned m = __ballot_sync(0xffffffffu, nz);
    if (m) return b0 + __ffs(m) - 1;
  }
  return K;
}

__global__ void __launch_bounds__(256) k_dense_forward(Fp fp, u32* Dp, u32 R, u32 K, unsigned long long* cand,
                                                       u32* lead, uint8_t* used, u32* piv_of_col) {
  cg::grid_group grid = cg::this_grid();
  __shared__ unsigned long long bmin[8];
  __shared__ u32 s_inv;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const int nwarps = blockDim.x >> 5;
  const u32 G = gridDim.x;
  const u32 lo = (u32)(((unsigned long long)R * blockIdx.x) / G);
  const u32 hi = (u32)(((unsigned long long)R * (blockIdx.x + 1)) / G);
  for (u32 i = lo + warp; i < hi; i += nwarps) {
    const u32 l = first_nonzero_warp(Dp + (size_t)i * K, 0, K);
    if (lane == 0) lead[i] = l;
  }
  __syncthreads();
  for (u32 step = 0;; ++step) {
    unsigned long long m = ~0ull;
    for (u32 i = lo + tid; i < hi; i += blockDim.x)
      if (!used[i] && lead[i] < K) m = min(m, ((unsigned long long)lead[i] << 32) | i);
#pragma unroll
    for (int o = 16; o; o >>= 1) m = min(m, __shfl_xor_sync(0xffffffffu, m, o));
    if (lane == 0) bmin[warp] = m;
    __syncthreads();
    if (tid == 0) {
      unsigned long long mm = ~0ull;
      for (int w = 0; w < nwarps; ++w) mm = min(mm, bmin[w]);
      if (mm != ~0ull) atomicMin(cand + step, mm);
    }
    grid.sync();
    const unsigned long long win = __ldcg(cand + step);
    if (win == ~0ull) break;
    const u32 c = (u32)(win >> 32), pr = (u32)(win & 0xFFFFFFFFull);
    const u32* prow_p = Dp + (size_t)pr * K;
    if (tid == 0) {
      s_inv = fp.inv(__ldcg(prow_p + c));
      if (pr >= lo && pr < hi) {
        used[pr] = 1;
        piv_of_col[c] = pr;
      }
    }
    __syncthreads();
    const u32 inv = s_inv;
    // rows leading at c: eliminate, then find their new lead
    for (u32 i = lo + warp; i < hi; i += nwarps) {
      if (used[i] || lead[i] != c) continue;
      u32* row = Dp + (size_t)i * K;
      const u32 fm = fp.to_mont(fp.neg(fp.mul(row[c], inv)));
      row_axpy8(fp, row, prow_p, fm, c + lane, K);
      __syncwarp();
      const u32 l = first_nonzero_warp(row, c + 1, K);
      if (lane == 0) lead[i] = l;
    }
    __syncthreads();
  }
}


// E3b: back-substitution -> RREF(D') rows (dense), one CTA per pivot.
__global__ void __launch_bounds__(SW_THREADS) k_dense_back(Fp fp, const u32* __restrict__ Dp, u32 K,
                                                            const u32* __restrict__ dpiv, const u32* __restrict__ dprow,
                                                            const u32* __restrict__ rankD_p, const u32* __restrict__ pbits_g,
                                                            const u32* __restrict__ pinv, const u32* __restrict__ prow_of,
                                                            u32* __restrict__ Rd, u32* __restrict__ gacc) {
  extern __shared__ u32 smem[];
  const u32 rankD = *rankD_p;
  const u32 nwords = (K + 31) / 32;
  u32* pbits = smem;
  u32* acc = gacc ? gacc + (size_t)blockIdx.x * K : smem + nwords;
  __shared__ u32 sh[2];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  for (u32 w = tid; w < nwords; w += blockDim.x) pbits[w] = pbits_g[w];
  for (u32 k = blockIdx.x; k < rankD; k += gridDim.x) {
    const u32 c0p = dpiv[k];
    const u32* src = Dp + (size_t)dprow[k] * K;
    for (u32 q = tid; q < K; q += blockDim.x) acc[q] = q >= c0p ? src[q] : 0u;
    __syncthreads();
    u32 cur = c0p + 1;
    while (true) {
      if (warp == 0) {
        u32 found = K;
        for (u32 b0 = cur & ~31u; b0 < K; b0 += 32) {
          u32 q = b0 + lane;
          bool hit = q >= cur && q < K && acc[q] != 0 && ((pbits[q >> 5] >> (q & 31)) & 1u);
          unsigned b = __ballot_sync(0xffffffffu, hit);
          if (b) {
            found = b0 + __ffs(b) - 1;
            break;
          }
        }
        if (lane == 0) sh[0] = found;
      }
      __syncthreads();
      const u32 q0 = sh[0];
      if (q0 >= K) break;
      const u32* prow_p = Dp + (size_t)prow_of[q0] * K;
      const u32 fm = fp.to_mont(fp.neg(fp.mul(acc[q0], pinv[q0])));
      for (u32 q = q0 + 1 + tid; q < K; q += blockDim.x) acc[q] = fp.add(acc[q], fp.mont_mul(fm, __ldg(prow_p + q)));
      if (tid == 0) acc[q0] = 0;
      __syncthreads();
      cur = q0 + 1;
    }
    const u32 inv = fp.inv(acc[c0p]);
    u32* out = Rd + (size_t)k * K;
    for (u32 q = tid; q < K; q += blockDim.x) out[q] = acc[q] ? fp.mul(acc[q], inv) : 0u;
    __syncthreads();
  }
}


// ---------------------------------------------------------------------------
// E3 (default): RREF(D') in pivot BLOCKS.
//
// Invariant: every live D' row is reduced by the basis B (kept in RREF), i.e.
// it is zero at every pivot column of B.  One iteration:
//   1 (all CTAs)  every live row offers itself (one atomicAdd); the first NP
//                 offers form the candidate block P.
//   2 (CTA 0)     Gaussian elimination of P restricted to a window of DB_W
//                 columns from its smallest lead (shared memory, one warp per
//                 row, one CTA barrier per pivot) finds the pivot columns L
//                 and the subset S of P's rows they come from; T = P[S, L] is
//                 invertible, T^-1 by a Gauss-Jordan sweep in shared memory,
//                 and T^-1·P[S] = RREF(span P[S]).  grid barrier.
//   3 (all CTAs)  with m = x[L]·T^-1 every live row and every old basis row
//                 is reduced in ONE product x <- x - m·P[S] (no pivot chain),
//                 the new basis rows T^-1·P[S] are written, new leads found
//                 in the same pass.  S's rows are consumed.
// D' has few distinct leading columns, but its live rows are nearly
// independent modulo B, so a block yields ~NP pivots: two grid barriers per
// block instead of one per pivot (k_dense_fwd_smem), no back-substitution
// (k_dense_back: B is reduced all along), and the full-width work is spread
// over the grid.  The RREF is unique, so the rows equal the reference's
// (sparselin.py:337-349).
// ---------------------------------------------------------------------------
struct DblkState {
  u32 cnt, np, rho, rho_old, iters, t2_us, t3_us, t3a_us;  // t*_us: CTA 0 phase times (trace)
  u32 t2a_us, t2b_us, t2c_us, pad;                         // phase 2 split: window load | forward | back + inverse
  u32 offers, distinct;                                    // trace: offers and distinct offered leads, summed over blocks
  u32 fc1, fc2, fc3, fcn;  // trace: forward loop kilocycles (min + barrier | update | barrier), iterations
  u32 q1, q2, q3;          // trace (CTA 1, us): phase-3 setup + coefficients | apply | offers
};
F4B_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %%globaltimer;" : "=l"(t));
  return t;
}
static constexpr int DB_THREADS = 512;
static constexpr int DB_NP = 32;  // max rows per block (one per lane of the selection warp)
static constexpr int DB_W = 128;  // window of the pivot search
static constexpr int DB_G = 8;    // rows per apply group
// SR: this CTA's D' rows live in shared memory for the whole kernel (phase 3
// reads and writes them there); a row goes back to Dp only when it is one of
// the block's first DB_NP offers — CTA 0's window and the pivot rows are read
// from Dp, and only candidates are ever read there.
template <bool SMALLP, bool SR>
__global__ void __launch_bounds__(DB_THREADS) k_dense_blk(Fp fp, u32* __restrict__ Dp, u32 R, u32 K, u32 rpc, u32 maxt,
                                                          u32* __restrict__ lead, u32* __restrict__ cand,
                                                          u32* __restrict__ Bm, u32* __restrict__ colpiv,
                                                          u32* __restrict__ gwin, u32* __restrict__ gT,
                                                          DblkState* __restrict__ st, u32* __restrict__ Rd,
                                                          u32* __restrict__ dpiv, u32* __restrict__ rank_out,
                                                          u32* __restrict__ order, u32* __restrict__ dflag) {
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) u32 smem[];
  constexpr int NW = DB_THREADS / 32;
  const unsigned FULL = 0xffffffffu;
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  const u32 G = gridDim.x, bid = blockIdx.x;
  const u32 p = fp.p;
  const bool tiny = p < 32768u;                          // 2 p^2 < 2^31
  const u32 mu32 = (u32)(0x100000000ull / p);            // Barrett constant
  __shared__ u32 s_T[DB_NP][DB_NP + 1];  // CTA 0: Y (-> T^-1); all: T^-1 of the block
  __shared__ u32 s_U[DB_NP][DB_NP + 33];  // CTA 0: pivot rows at L | Z
  __shared__ u32 s_crow[DB_NP], s_rl[DB_NP];
  __shared__ u32 s_wrow[DB_NP], s_wcol[DB_NP];
  __shared__ u32 s_red[33];
  __shared__ u32 s_nt, s_na, s_np, s_c0;
  // CTA 0 phase 2: the block's window | Z, aliasing the phase-3 arrays
  u32(*s_X)[DB_W + 32] = reinterpret_cast<u32(*)[DB_W + 32]>(smem);
  u32* s_c = smem;                    // [maxt][DB_NP] coefficients
  u32* s_task = smem + maxt * DB_NP;  // [maxt] kind<<30 | index
  u32* s_act = s_task + maxt;         // [maxt] active task list
  u32* s_lead = s_act + maxt;         // [rpc] leads of this CTA's rows
  const u32 lo = bid * rpc;
  const u32 nr = lo < R ? min(rpc, R - lo) : 0u;
  // coefficients are held in Montgomery form c' = c R.  SMALLP (p < 2^16):
  // raw products c' v summed in 64 bits (< 32 p^2 < p 2^32) and one REDC
  // give sum c v mod p; otherwise Montgomery products and one modulo.
  auto prod = [&](u32 c, u32 v) -> u64 { return SMALLP ? (u64)c * v : (u64)fp.mont_mul(c, v); };
  auto red64 = [&](u64 a) -> u32 {
    if (SMALLP) {
      const u32 m = (u32)a * fp.pprime;
      const u64 u = (a + (u64)m * p) >> 32;
      return (u32)(u >= p ? u - p : u);
    }
    return (u32)(a % p);
  };
  u32 it_no = 1;  // block number (trace: distinct offered leads per block)
  auto offer = [&](u32 row, u32 l) -> bool {
    const u32 s = atomicAdd(&st->cnt, 1u);
    if (s < (u32)DB_NP) cand[s] = row;
    if (dflag) {
      atomicAdd(&st->offers, 1u);
      if (atomicMax(dflag + l, it_no) < it_no) atomicAdd(&st->distinct, 1u);
    }
    return s < (u32)DB_NP;
  };
  u32* s_f = s_lead + rpc;  // [maxt] first nonzero column of each task
  // SR: [rpc][K] this CTA's rows, after the window / task area
  u32* s_rows = smem + max((u32)(DB_NP * (DB_W + 32)), maxt * (DB_NP + 3) + rpc);
  __shared__ u32 s_wbn, s_wb[DB_NP];  // SR: rows to write back (offered into the candidate slots)
  u32 ro = 0;
  auto task_row = [&](u32 td) -> u32* {
    const u32 kind = td >> 30, idx = td & 0x3FFFFFFFu;
    if (SR && kind == 0) return s_rows + (size_t)idx * K;
    return kind == 0 ? Dp + (size_t)(lo + idx) * K : Bm + (size_t)(kind == 1 ? idx : ro + idx) * K;
  };
  // prologue: leads of this CTA's rows (contiguous in D'), first offers
  for (u32 r = tid; r < nr; r += DB_THREADS) s_lead[r] = K;
  __syncthreads();
  {
    const u32* x0 = Dp + (size_t)lo * K;
    const u32 tot = nr * K;  // host: rpc * K < 2^32
    for (u32 e0 = tid; e0 < tot; e0 += 8 * DB_THREADS) {
      u32 v[8];
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const u32 e = e0 + h * DB_THREADS;
        v[h] = e < tot ? __ldcg(x0 + e) : 0u;
      }
#pragma unroll
      for (int h = 0; h < 8; ++h) {
        const u32 e = e0 + h * DB_THREADS;
        if (SR && e < tot) s_rows[e] = v[h];
        if (v[h]) {
          const u32 r = e / K, q = e - r * K;
          if (q < s_lead[r]) atomicMin(&s_lead[r], q);
        }
      }
    }
  }
  __syncthreads();
  for (u32 r = tid; r < nr; r += DB_THREADS) {
    lead[lo + r] = s_lead[r];
    if (s_lead[r] < K) offer(lo + r, s_lead[r]);  // Dp still holds the rows here
  }
  unsigned long long t2 = 0, t3 = 0, t3a = 0, tm = 0, t2a = 0, t2b = 0, t2c = 0;
  while (true) {
    grid.sync();  // offers complete, every row of this iteration final
    if (bid == 0 && tid == 0) tm = gtimer();
    if (bid == 0) {
      // 2a: the candidates' window [c0, c0 + DB_W) in shared memory, each
      // row augmented with its coefficient vector over the candidates (Z)
      const u32 nc = min(__ldcg(&st->cnt), (u32)DB_NP);
      const u32 rho = st->rho;
      if (warp == 0) {
        u32 row = 0, l = K;
        if ((u32)lane < nc) {
          row = __ldcg(cand + lane);
          l = __ldcg(lead + row);
        }
        s_crow[lane] = row;
        const u32 c0 = __reduce_min_sync(FULL, l);
        if (lane == 0) {
          s_c0 = c0;
          s_np = 0;
        }
      }
      __syncthreads();
      const u32 c0 = s_c0;
      for (u32 w = warp; w < nc; w += NW) {
        const u32* src = Dp + (size_t)s_crow[w] * K + c0;
        u32 v[DB_W / 32];
#pragma unroll
        for (int h = 0; h < DB_W / 32; ++h) {
          const u32 q = lane + 32 * h;
          v[h] = c0 + q < K ? __ldcg(src + q) : 0u;
        }
        u32 l = DB_W;
#pragma unroll
        for (int h = DB_W / 32 - 1; h >= 0; --h) {
          s_X[w][lane + 32 * h] = v[h];
          const unsigned bm = __ballot_sync(FULL, v[h] != 0);
          if (bm) l = 32 * h + __ffs(bm) - 1;
        }
        s_X[w][DB_W + lane] = (u32)lane == w ? 1u : 0u;
        if (lane == 0) s_rl[w] = l;
      }
      __syncthreads();
      unsigned long long tb0 = 0;
      if (tid == 0) {
        tb0 = gtimer();
        t2a += tb0 - tm;
      }
      // 2b: forward elimination inside the window (row scaling, no inverses);
      // the pivot is the lowest candidate of the smallest lead (one 32-bit
      // warp min), each warp updates its two rows interleaved
      __shared__ unsigned long long s_upd;
      unsigned long long fa = 0, fb = 0, fc = 0, fn = 0, ft0 = 0;
      while (true) {
        if (dflag && tid == 0) {
          ft0 = clock64();
          s_upd = 0;
        }
        const u32 key = ((u32)lane < nc && s_rl[lane] < (u32)DB_W) ? (s_rl[lane] << 5) | (u32)lane : 0xFFFFFFFFu;
        const u32 m = __reduce_min_sync(FULL, key);
        if (m == 0xFFFFFFFFu) break;
        const u32 pw = m & 31u, c = m >> 5;
        __syncthreads();  // every warp has read s_rl
        unsigned long long ft1 = 0;
        if (dflag && tid == 0) ft1 = clock64();
        if (tid == 0) {
          s_wrow[s_np] = pw;  // candidate slot for now
          s_wcol[s_np] = c;   // window column for now
          s_np = s_np + 1;
          s_rl[pw] = DB_W + 1;  // used
        }
        const u32* prw = s_X[pw];
        static_assert(DB_NP == 2 * NW, "two candidate rows per warp");
        const u32 wa = warp, wb = warp + NW;
        const bool ua = wa < nc && wa != pw && s_rl[wa] == c;  // rows leading right of c are zero at c
        const bool ub = wb < nc && wb != pw && s_rl[wb] == c;
        if (ua || ub) {
          u32* xa = s_X[wa];
          u32* xb = s_X[wb];
          // x <- a x - x[c] prow: p < 2^15 sums both raw products in 32 bits
          // and reduces once (Barrett); otherwise Montgomery products
          const u32 a = tiny ? prw[c] : fp.to_mont(prw[c]);
          const u32 ba = ua ? (tiny ? p - xa[c] : fp.to_mont(fp.neg(xa[c]))) : 0u;
          const u32 bb = ub ? (tiny ? p - xb[c] : fp.to_mont(fp.neg(xb[c]))) : 0u;
          auto comb = [&](u32 m1, u32 x1, u32 m2, u32 x2) -> u32 {
            if (tiny) {
              const u32 t = m1 * x1 + m2 * x2;  // < 2 p^2 < 2^31
              const u32 r = t - __umulhi(t, mu32) * p;
              return r >= p ? r - p : r;
            }
            return fp.add(fp.mont_mul(m1, x1), fp.mont_mul(m2, x2));
          };
          u32 la = DB_W, lb = DB_W;
#pragma unroll
          for (int h = DB_W / 32; h >= 0; --h) {  // h = DB_W/32: the coefficients
            if (h < DB_W / 32 && 32 * h + 31 < (int)c) continue;  // left of c: zero in both rows
            const u32 q = lane + 32 * h;
            const u32 pq = prw[q];
            u32 va = 0, vb = 0;
            if (q > c) {
              if (ua) {
                va = comb(a, xa[q], ba, pq);
                xa[q] = va;
              }
              if (ub) {
                vb = comb(a, xb[q], bb, pq);
                xb[q] = vb;
              }
            } else if (q == c) {
              if (ua) xa[q] = 0;
              if (ub) xb[q] = 0;
            }
            if (h < DB_W / 32) {
              const unsigned b1 = __ballot_sync(FULL, va != 0), b2 = __ballot_sync(FULL, vb != 0);
              if (b1) la = 32 * h + __ffs(b1) - 1;
              if (b2) lb = 32 * h + __ffs(b2) - 1;
            }
          }
          if (lane == 0) {
            if (ua) s_rl[wa] = la;
            if (ub) s_rl[wb] = lb;
          }
        }
        if (dflag && lane == 0) atomicMax(&s_upd, (unsigned long long)clock64());
        __syncthreads();
        if (dflag && tid == 0) {
          const unsigned long long ft3 = clock64(), fu = max(s_upd, ft1);
          fa += ft1 - ft0;
          fb += fu - ft1;
          fc += ft3 - fu;
          fn += 1;
        }
      }
      if (dflag && tid == 0) {
        st->fc1 += (u32)(fa / 1000);
        st->fc2 += (u32)(fb / 1000);
        st->fc3 += (u32)(fc / 1000);
        st->fcn += (u32)fn;
      }
      if (tid == 0) {
        const unsigned long long tc0 = gtimer();
        t2b += tc0 - tb0;
        tb0 = tc0;
      }
      // 2c: Y = U_L^-1 Z by back-substitution on the coefficient vectors (U_L
      // = the pivot rows at the pivot columns, upper triangular; Z their
      // expressions over the candidate slots): one warp, lane = slot, no CTA
      // barrier per pivot.  Y's rows have the identity at L: T^-1 = Y[:, S].
      const u32 np = s_np;
      for (u32 e = tid; e < np * (DB_NP + 32); e += DB_THREADS) {
        const u32 i = e / (DB_NP + 32), k = e % (DB_NP + 32);
        const u32* x = s_X[s_wrow[i]];
        s_U[i][k] = k < DB_NP ? (k < np ? fp.to_mont(x[s_wcol[k]]) : 0u) : x[DB_W + (k - DB_NP)];
      }
      __syncthreads();
      if (SMALLP && warp == 0) {
        // p < 2^16: left-looking, y_i = d_i (z_i - sum_{j>i} U_ij y_j) with
        // the raw products summed in 64 bits (< 32 p^2 < p 2^32), one REDC
        // per row; the loads of a row's dot product are independent
        const u32 dl = (u32)lane < np ? fp.to_mont(fp.inv(fp.mont_mul(s_U[lane][lane], 1u))) : 0u;
        for (int i = (int)np - 1; i >= 0; --i) {
          u64 acc0 = 0, acc1 = 0;
          int j = i + 1;
          for (; j + 2 <= (int)np; j += 2) {
            acc0 += (u64)s_U[i][j] * s_U[j][DB_NP + lane];
            acc1 += (u64)s_U[i][j + 1] * s_U[j + 1][DB_NP + lane];
          }
          if (j < (int)np) acc0 += (u64)s_U[i][j] * s_U[j][DB_NP + lane];
          s_U[i][DB_NP + lane] =
              fp.mont_mul(__shfl_sync(FULL, dl, i), fp.sub(s_U[i][DB_NP + lane], red64(acc0 + acc1)));
          __syncwarp();
        }
      } else if (warp == 0) {
        const u32 dl = (u32)lane < np ? fp.to_mont(fp.inv(fp.mont_mul(s_U[lane][lane], 1u))) : 0u;
        for (int i = (int)np - 1; i >= 0; --i) {
          const u32 y = fp.mont_mul(__shfl_sync(FULL, dl, i), s_U[i][DB_NP + lane]);
          s_U[i][DB_NP + lane] = y;
          int r = 0;
          for (; r + 4 <= i; r += 4) {  // four independent updates in flight
            u32 z[4], u[4];
#pragma unroll
            for (int q = 0; q < 4; ++q) {
              z[q] = s_U[r + q][DB_NP + lane];
              u[q] = s_U[r + q][i];
            }
#pragma unroll
            for (int q = 0; q < 4; ++q) s_U[r + q][DB_NP + lane] = fp.sub(z[q], fp.mont_mul(u[q], y));
          }
          for (; r < i; ++r) s_U[r][DB_NP + lane] = fp.sub(s_U[r][DB_NP + lane], fp.mont_mul(s_U[r][i], y));
        }
      }
      __syncthreads();
      if (tid == 0) t2c += gtimer() - tb0;
      // T^-1[i][j] = Y_i[slot of S_j]
      for (u32 e = tid; e < np * np; e += DB_THREADS) {
        const u32 i = e / np, j = e % np;
        gT[i * DB_NP + j] = fp.to_mont(s_U[i][DB_NP + s_wrow[j]]);
      }
      if (tid < (int)np) {
        const u32 row = s_crow[s_wrow[tid]], col = c0 + s_wcol[tid];
        gwin[tid] = row;
        gwin[DB_NP + tid] = col;
        colpiv[col] = rho + tid;
        lead[row] = K + 1;  // consumed: spans new basis rows
      }
      if (tid == 0) {
        st->np = np;
        st->rho_old = rho;
        st->rho = rho + np;
        st->cnt = 0;
        st->iters += 1;
      }
    }
    if (bid == 0 && tid == 0) {
      const unsigned long long t = gtimer();
      t2 += t - tm;
      tm = t;
    }
    grid.sync();
    const unsigned long long qa = dflag && bid == 1 && tid == 0 ? gtimer() : 0ull;
    const u32 np = __ldcg(&st->np);
    ro = __ldcg(&st->rho_old);
    if (np == 0) break;
    // 3: tasks of this CTA
    for (u32 e = tid; e < np * np; e += DB_THREADS) {
      const u32 k = e / np, j = e % np;
      s_T[k][j] = __ldcg(gT + k * DB_NP + j);
    }
    if (tid < (int)np) {
      s_wrow[tid] = __ldcg(gwin + tid);
      s_wcol[tid] = __ldcg(gwin + DB_NP + tid);
    }
    for (u32 r = tid; r < nr; r += DB_THREADS) s_lead[r] = __ldcg(lead + lo + r);
    __syncthreads();
    if (tid == 0) {
      u32 nt = 0;
      for (u32 r = 0; r < nr; ++r)
        if (s_lead[r] < K) s_task[nt++] = r;  // kind 0: live D' row
      for (u32 i = bid; i < ro; i += G) s_task[nt++] = (1u << 30) | i;  // kind 1: old basis row
      for (u32 k = (bid + G - ro % G) % G; k < np; k += G) s_task[nt++] = (2u << 30) | k;  // kind 2: new basis row
      s_nt = nt;
      s_na = 0;
    }
    __syncthreads();
    const u32 nt = s_nt;
    // coefficients, one warp per task: m = x[L]·T^-1 (kind 2: row k of T^-1)
    for (u32 t = warp; t < nt; t += NW) {
      const u32 td = s_task[t], kind = td >> 30, idx = td & 0x3FFFFFFFu;
      u32 m = 0;
      if (kind == 2) {
        m = (u32)lane < np ? s_T[idx][lane] : 0u;
      } else {
        const u32* x = task_row(td);
        const u32 xl = (u32)lane < np ? (SR && kind == 0 ? x[s_wcol[lane]] : __ldcg(x + s_wcol[lane])) : 0u;
        u64 acc = 0;
        for (u32 k = 0; k < np; ++k) {
          const u32 xk = __shfl_sync(FULL, xl, k);
          if (xk && (u32)lane < np) acc += prod(s_T[k][lane], xk);
        }
        m = red64(acc);
        if (m) m = fp.to_mont(m);
      }
      s_c[t * DB_NP + lane] = m;
      if (__ballot_sync(FULL, m != 0) && lane == 0) s_act[atomicAdd(&s_na, 1u)] = t;
    }
    __syncthreads();
    const u32 na = s_na;
    if (bid == 0 && tid == 0) t3a += gtimer() - tm;
    const unsigned long long qb = dflag && bid == 1 && tid == 0 ? gtimer() : 0ull;
    // one pass over the columns: the block's np rows are loaded once per
    // column (one L2 round trip) and applied to every active task
    for (u32 t = tid; t < nt; t += DB_THREADS) s_f[t] = K;
    __syncthreads();
    for (u32 q = tid; q < K; q += DB_THREADS) {
      u32 pv[DB_NP];
#pragma unroll
      for (int j = 0; j < DB_NP; ++j) pv[j] = (u32)j < np ? __ldcg(Dp + (size_t)s_wrow[j] * K + q) : 0u;
      for (u32 g0 = 0; g0 < na; g0 += DB_G) {
        const u32 ng = min((u32)DB_G, na - g0);
        u32 xb[DB_G];
        u64 acc[DB_G];
#pragma unroll
        for (int r = 0; r < DB_G; ++r) {
          acc[r] = 0;
          xb[r] = 0;
          if ((u32)r < ng) {
            const u32 td = s_task[s_act[g0 + r]];
            if ((td >> 30) != 2) xb[r] = SR && (td >> 30) == 0 ? task_row(td)[q] : __ldcg(task_row(td) + q);
          }
        }
#pragma unroll
        for (int r = 0; r < DB_G; ++r) {
          if ((u32)r < ng) {
            // coefficients past np are zero (lanes >= np wrote 0): the
            // groups of 4 beyond np are skipped (warp-uniform exit)
            const uint4* cr = reinterpret_cast<const uint4*>(s_c + s_act[g0 + r] * DB_NP);
            u64 a = 0;
#pragma unroll
            for (int j4 = 0; j4 < DB_NP / 4; ++j4) {
              if (4 * j4 >= (int)np) break;
              const uint4 cv = cr[j4];
              if (SMALLP && tiny)  // p < 2^15: four products < 4 p^2 < 2^32 summed in 32 bits
                a += (u64)(cv.x * pv[4 * j4] + cv.y * pv[4 * j4 + 1] + cv.z * pv[4 * j4 + 2] + cv.w * pv[4 * j4 + 3]);
              else
                a += prod(cv.x, pv[4 * j4]) + prod(cv.y, pv[4 * j4 + 1]) + prod(cv.z, pv[4 * j4 + 2]) +
                     prod(cv.w, pv[4 * j4 + 3]);
            }
            acc[r] = a;
          }
        }
#pragma unroll
        for (int r = 0; r < DB_G; ++r) {
          if ((u32)r < ng) {
            const u32 t = s_act[g0 + r], td = s_task[t];
            const u32 sres = red64(acc[r]);
            const u32 v = (td >> 30) == 2 ? sres : fp.sub(xb[r], sres);
            task_row(td)[q] = v;
            if (v && q < s_f[t]) atomicMin(&s_f[t], q);
          }
        }
      }
    }
    __syncthreads();
    for (u32 a = tid; a < na; a += DB_THREADS) {
      const u32 t = s_act[a], td = s_task[t];
      if ((td >> 30) == 0) s_lead[td & 0x3FFFFFFFu] = s_f[t];
    }
    __syncthreads();
    if (bid == 0 && tid == 0) t3 += gtimer() - tm;
    const unsigned long long qc = dflag && bid == 1 && tid == 0 ? gtimer() : 0ull;
    // 1 (next iteration): offers of the live rows
    ++it_no;
    if (SR) {
      if (tid == 0) s_wbn = 0;
      __syncthreads();
    }
    for (u32 r = tid; r < nr; r += DB_THREADS) {
      const u32 l = s_lead[r];
      if (l <= K) {  // K + 1 = consumed
        lead[lo + r] = l;
        if (l < K && offer(lo + r, l) && SR) s_wb[atomicAdd(&s_wbn, 1u)] = r;
      }
    }
    if (SR) {  // candidates are read from Dp (CTA 0's window, the pivot rows)
      __syncthreads();
      const u32 nwb = s_wbn;
      for (u32 e = tid; e < nwb * K; e += DB_THREADS) {
        const u32 i = e / K, q = e - i * K, r = s_wb[i];
        Dp[(size_t)(lo + r) * K + q] = s_rows[(size_t)r * K + q];
      }
    }
    if (dflag && bid == 1) {
      __syncthreads();
      if (tid == 0) {
        const unsigned long long qd = gtimer();
        atomicAdd(&st->q1, (u32)((qb - qa) / 1000));
        atomicAdd(&st->q2, (u32)((qc - qb) / 1000));
        atomicAdd(&st->q3, (u32)((qd - qc) / 1000));
      }
    }
  }
  // emit: basis rows in ascending pivot order
  const u32 rho = __ldcg(&st->rho);
  if (bid == 0) {
    if (tid == 0) {
      st->t2_us = (u32)(t2 / 1000);
      st->t2a_us = (u32)(t2a / 1000);
      st->t2b_us = (u32)(t2b / 1000);
      st->t2c_us = (u32)(t2c / 1000);
      st->t3_us = (u32)(t3 / 1000);
      st->t3a_us = (u32)(t3a / 1000);
    }
    u32 base = 0;
    for (u32 q0 = 0; q0 < K; q0 += DB_THREADS) {
      const u32 q = q0 + tid;
      const u32 j = q < K ? __ldcg(colpiv + q) : NONE;
      u32 tot;
      const u32 pre = block_scan_flag(j != NONE ? 1u : 0u, s_red, &tot);
      if (j != NONE) {
        dpiv[base + pre] = q;
        order[base + pre] = j;
      }
      base += tot;
    }
    if (tid == 0) *rank_out = rho;
  }
  grid.sync();
  for (u32 k = bid; k < rho; k += G) {
    const u32* src = Bm + (size_t)__ldcg(order + k) * K;
    u32* dst = Rd + (size_t)k * K;
    for (u32 q = tid; q < K; q += DB_THREADS) dst[q] = __ldcg(src + q);
  }
}

// E3b: pivots of D' in one CTA: pivot flags, their exclusive scan, the pivot
// lists (column, row), the inverse leads, the pivot bitmap and rank(D') —
// all on the device, no host read before the back-substitution.
__global__ void __launch_bounds__(1024) k_dense_post(Fp fp, const u32* __restrict__ Dp, u32 K,
                                                     const u32* __restrict__ pofc, u32* __restrict__ pinv,
                                                     u32* __restrict__ dpiv, u32* __restrict__ dprow,
                                                     u32* __restrict__ pbits, u32* __restrict__ rankD_out) {
  __shared__ u32 red[33];
  u32 base = 0;
  for (u32 q0 = 0; q0 < K; q0 += blockDim.x) {
    const u32 q = q0 + threadIdx.x;
    const u32 pr = q < K ? pofc[q] : NONE;
    const bool f = pr != NONE;
    if (q < K) pinv[q] = f ? fp.inv(Dp[(size_t)pr * K + q]) : 0u;
    const unsigned bm = __ballot_sync(0xffffffffu, f);
    if ((threadIdx.x & 31) == 0 && q < K) pbits[q >> 5] = bm;
    u32 tot;
    const u32 pre = block_scan_flag(f ? 1u : 0u, red, &tot);
    if (f) {
      dpiv[base + pre] = q;
      dprow[base + pre] = pr;
    }
    base += tot;
  }
  if (threadIdx.x == 0) *rankD_out = base;
}

// E3c: emit RREF(D') rows as sparse rows over the global columns
__global__ void __launch_bounds__(SW_THREADS) k_emit_dense(const u32* __restrict__ Rd, u32 K,
                                                            const u32* __restrict__ rankD_p,
                                                            const u32* __restrict__ dpiv, const u32* __restrict__ nonA,
                                                            u32* __restrict__ pcol, u32* __restrict__ pval, size_t cap,
                                                            unsigned long long* cursor, u32* s_off, u32* s_len,
                                                            u32* err) {
  __shared__ u32 red[33];
  __shared__ u32 sh[2];
  const u32 rankD = *rankD_p;
  for (u32 k = blockIdx.x; k < rankD; k += gridDim.x) {
    emit_row(Rd + (size_t)k * K, dpiv[k], K, nonA, pcol, pval, cap, cursor, s_off + k, s_len + k, err, red, sh);
    __syncthreads();
  }
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------
static Fp make_fp(Ctx* c) {
  Fp fp;
  fp.p = c->p;
  fp.pprime = c->pprime;
  fp.r2 = c->r2;
  return fp;
}

Fp make_fp_pub(Ctx* c) { return make_fp(c); }

static int sweep_grid(Ctx* c, size_t smem, long long rows) {
  int per_sm = (int)std::max<size_t>(1, std::min<size_t>(8, (220 * 1024) / std::max<size_t>(smem + 3072, 1)));
  return (int)std::max<long long>(1, std::min<long long>(rows, (long long)c->num_sms * per_sm));
}

// k_sweep<MODE, T>: u16 accumulators when p < 2^16 and the row fits shared
// memory, u32 in shared memory otherwise, u32 in HBM for very wide matrices.
// Window tables of k_sweep_win (k_tail_copy + k_win_build), enqueued either
// with the host's nA or, right behind k_psge_prep, with nA read on the device
// and the grids sized by N (the host then learns (nA, nC) while these run).
struct WinPrep {
  bool ok = false, pk = false;
  DBuf wW, wC, wD, wT, gcur, wTm, wM;
};
static bool win_eligible(Ctx* c, u32 N, long long nA_bound) {
  const size_t nwords = (N + 31) / 32;
  const size_t smem = (size_t)((2 * nwords + 3) & ~(size_t)3) * 4 + (size_t)(N + 1) * 4;
  // lazily reduced u32 accumulator: initial value + one product in [0, 2p)
  // per applied pivot
  return c->opt_sweep == 0 && nA_bound > 0 &&
         (unsigned long long)c->p * (2ull * (unsigned long long)nA_bound + 2) < (1ull << 32) && smem <= 180 * 1024;
}
static void win_prepare(Ctx* c, const Fp& fp, f4b_echelon* E, const u32* d_nA, u32 nA_bound, WinPrep& w) {
  const u32 N = (u32)E->n_cols;
  w.pk = N < 65535u && c->p < 65536u;
  const u32 nwin = (nA_bound + 31) / 32;
  const size_t groups = (size_t)(E->M + 4 * (long long)nA_bound) / 4 + 8;
  ensure(c, w.wW, (size_t)nwin * 1024 * sizeof(u32));
  ensure(c, w.wC, (size_t)nwin * 32 * sizeof(u32));
  ensure(c, w.wD, (size_t)nwin * 32 * sizeof(uint2));
  ensure(c, w.wT, groups * (w.pk ? 16 : 32));
  ensure(c, w.wTm, (size_t)nwin * 1024 * sizeof(u32));
  ensure(c, w.wM, (size_t)nwin * 32 * sizeof(u32));
  ensure(c, w.gcur, 16);
  check_cuda(cudaMemsetAsync(w.gcur.p, 0, 4, c->stream), "memset");
  check_cuda(cudaMemsetAsync(w.wTm.p, 0, (size_t)nwin * 1024 * sizeof(u32), c->stream), "memset");
  if (w.pk)
    F4B_LAUNCH(c, k_tail_copy<true>, nb(nA_bound, 8), 256, 0, fp, E->col, E->val, N, E->desc.as<uint4>(),
               E->abits.as<u32>(), E->acols.as<u32>(), E->apos.as<u32>(), d_nA, nA_bound, w.wD.as<uint2>(),
               w.gcur.as<u32>(), w.wTm.as<u32>(), w.wM.as<u32>(), w.wT.as<u32>());
  else
    F4B_LAUNCH(c, k_tail_copy<false>, nb(nA_bound, 8), 256, 0, fp, E->col, E->val, N, E->desc.as<uint4>(),
               E->abits.as<u32>(), E->acols.as<u32>(), E->apos.as<u32>(), d_nA, nA_bound, w.wD.as<uint2>(),
               w.gcur.as<u32>(), w.wTm.as<u32>(), w.wM.as<u32>(), w.wT.as<uint2>());
  F4B_LAUNCH(c, k_win_build, nb(nwin, WB_WARPS), 32 * WB_WARPS, 0, fp, N, E->desc.as<uint4>(), E->acols.as<u32>(),
             d_nA, nA_bound, w.wTm.as<u32>(), w.wM.as<u32>(), w.wW.as<u32>(), w.wC.as<u32>());
  w.ok = true;
}
static void win_release(Ctx* c, WinPrep& w) {
  for (DBuf* b : {&w.wW, &w.wC, &w.wD, &w.wT, &w.gcur, &w.wTm, &w.wM}) release(c, *b);
  w.ok = false;
}

// k_sweep<MODE, T>: u16 accumulators when p < 2^16 and the row fits shared
// memory, u32 in shared memory otherwise, u32 in HBM for very wide matrices.
template <int MODE>
static void launch_sweep(Ctx* c, const Fp& fp, f4b_echelon* E, const u32* rows, u32 nrows, u32* Dp, u32 K,
                         const u32* Rd, u32 rankD, const u32* dpiv, u32* pcol, u32* pval, size_t cap,
                         unsigned long long* cursor, u32* s_off, u32* s_len, u32* err,
                         unsigned long long* stats = nullptr, WinPrep* pre = nullptr) {
  const u32 N = (u32)E->n_cols;
  // c->opt_sweep (f4b_ctx_set_option "sweep"): 0 = automatic (windows, then
  // the blocked sweep, then k_sweep), 1 = start at the blocked sweep,
  // 2 = k_sweep only — the fallbacks are forced by the parity tests
  if (win_eligible(c, N, E->nA)) {
    // fixed windows with precomputed block inverses (k_win_build + k_sweep_win)
    const size_t nwords = (N + 31) / 32;
    const size_t smem = (size_t)((2 * nwords + 3) & ~(size_t)3) * 4 + (size_t)(N + 1) * 4;
    WinPrep local;
    WinPrep& w = pre && pre->ok ? *pre : local;
    if (!w.ok) win_prepare(c, fp, E, nullptr, (u32)E->nA, w);
    const bool pk = w.pk;
    const void* kf = pk ? (const void*)k_sweep_win<true, MODE> : (const void*)k_sweep_win<false, MODE>;
    static int per_sm_c[2] = {-1, -1};
    static size_t smem_c[2] = {0, 0};
    if (per_sm_c[pk] < 0 || smem_c[pk] != smem) {  // occupancy query once per (kernel, N)
      check_cuda(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024), "attr");
      check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&per_sm_c[pk], kf, 256, smem), "occupancy");
      smem_c[pk] = smem;
    }
    const int per_sm = std::max(1, per_sm_c[pk]);
    const int grid = (int)std::max<long long>(1, std::min<long long>(nrows, (long long)c->num_sms * per_sm));
    const u32 mu = (u32)((1ull << 32) / c->p);
    const u32 nwin = (u32)((E->nA + 31) / 32);
    static const bool strace = getenv("F4B_SWEEP_TRACE") != nullptr;
    DBuf trb;
    if (strace) {
      ensure(c, trb, 128);
      check_cuda(cudaMemsetAsync(trb.p, 0, 128, c->stream), "memset");
    }
    SweepOut so{E->invl.as<u32>(), Rd, rankD, dpiv, pcol, pval, cap, cursor, s_off, s_len, err,
                strace ? trb.as<unsigned long long>() : nullptr};
    {
      ProfScope ps(c, pk ? (MODE ? "k_sweep_win<true,1>" : "k_sweep_win<true>")
                         : (MODE ? "k_sweep_win<false,1>" : "k_sweep_win<false>"));
      if (pk && strace && MODE == 0)
        k_sweep_win<true, MODE, true><<<grid, 256, smem, c->stream>>>(fp, mu, E->rp, E->col, E->val, N, rows, nrows,
                 E->abits.as<u32>(), w.wW.as<u32>(), w.wC.as<u32>(), w.wD.as<uint2>(), nwin, w.wT.as<uint4>(), Dp, K,
                 E->nonA.as<u32>(), stats, so);
      else if (pk)
        k_sweep_win<true, MODE><<<grid, 256, smem, c->stream>>>(fp, mu, E->rp, E->col, E->val, N, rows, nrows,
                 E->abits.as<u32>(), w.wW.as<u32>(), w.wC.as<u32>(), w.wD.as<uint2>(), nwin, w.wT.as<uint4>(), Dp, K,
                 E->nonA.as<u32>(), stats, so);
      else
        k_sweep_win<false, MODE><<<grid, 256, smem, c->stream>>>(fp, mu, E->rp, E->col, E->val, N, rows, nrows,
                 E->abits.as<u32>(), w.wW.as<u32>(), w.wC.as<u32>(), w.wD.as<uint2>(), nwin, w.wT.as<uint4>(), Dp, K,
                 E->nonA.as<u32>(), stats, so);
      check_cuda(cudaGetLastError(), "k_sweep_win");
    }
    if (strace) {
      unsigned long long h[16];
      check_cuda(cudaMemcpyAsync(h, trb.p, 128, cudaMemcpyDeviceToHost, c->stream), "d2h");
      check_cuda(cudaStreamSynchronize(c->stream), "sync");
      const double rows = (double)std::max(1ull, h[0]), wins = (double)std::max(1ull, h[1]);
      fprintf(stderr, "[sweep%d] rows=%llu N=%u nA=%lld grid=%d windows/row=%.1f miss=%.2f cyc/window: find+mult %.0f (find %.0f v %.0f) bar %.0f apply+bar %.0f | tail/row %.0f\n",
              MODE, h[0], N, (long long)E->nA, grid, wins / rows, h[2] / wins, h[3] / wins, h[7] / wins, h[8] / wins,
              h[4] / wins, h[5] / wins, h[6] / rows);
      release(c, trb);
    }
    win_release(c, w);
    return;
  }
  if (pre && pre->ok) win_release(c, *pre);
  if (MODE == 0 && c->opt_sweep <= 1) {
    // blocked sweep: lazily reduced u32 accumulator needs p * (nA + 1) < 2^32
    const size_t bitmap = (size_t)((((N + 31) / 32) + 3) & ~3u) * 4;
    const size_t smem = bitmap + (size_t)N * 4;
    if ((unsigned long long)c->p * (unsigned long long)(E->nA + 1) < (1ull << 32) && smem <= 180 * 1024) {
      static bool battr = false;
      if (!battr) {
        check_cuda(cudaFuncSetAttribute(k_sweep_blk, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024),
                   "attr");
        battr = true;
      }
      const int per_sm = (int)std::max<size_t>(1, std::min<size_t>(8, (220 * 1024) / (smem + 8 * 1024)));
      const int grid = (int)std::max<long long>(1, std::min<long long>(nrows, (long long)c->num_sms * per_sm));
      const u32 mu = (u32)((1ull << 32) / c->p);
      F4B_LAUNCH(c, k_sweep_blk, grid, 256, smem, fp, mu, E->rp, E->col, E->val, N, rows, nrows, E->desc.as<uint4>(),
                 E->abits.as<u32>(), E->acols.as<u32>(), E->apos.as<u32>(), (u32)E->nA, Dp, K, E->nonA.as<u32>(),
                 stats);
      return;
    }
  }
  const size_t bitmap = (size_t)((N + 31) / 32) * 4;
  const bool small_p = c->p < 65536u;
  const size_t acc_b = (((size_t)N * (small_p ? 2 : 4)) + 15) & ~(size_t)15;
  const bool gl = bitmap + acc_b > 200 * 1024;
  const size_t smem = gl ? bitmap : bitmap + acc_b;
  const int grid = sweep_grid(c, smem, nrows);
  static bool attr = false;
  if (!attr) {
    check_cuda(cudaFuncSetAttribute(k_sweep<MODE, u32>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 4096),
               "attr");
    check_cuda(cudaFuncSetAttribute(k_sweep<MODE, uint16_t>, cudaFuncAttributeMaxDynamicSharedMemorySize,
                                    200 * 1024 + 4096), "attr");
    attr = true;
  }
  // profiled as k_sweep<MODE> (the tests check which sweep ran)
  ProfScope ps(c, MODE ? "k_sweep<1>" : "k_sweep<0>");
  if (gl) {
    DBuf gacc;
    ensure(c, gacc, (size_t)grid * N * sizeof(u32));
    k_sweep<MODE, u32><<<grid, SW_THREADS, smem, c->stream>>>(fp, E->rp, E->col, E->val, N, rows, nrows,
               E->desc.as<uint4>(), E->invl.as<u32>(), E->abits.as<u32>(), gacc.as<u32>(), Dp, K, E->nonA.as<u32>(),
               Rd, rankD, dpiv, pcol, pval, cap, cursor, s_off, s_len, err, stats);
    check_cuda(cudaGetLastError(), "k_sweep");
    release(c, gacc);
  } else if (small_p) {
    k_sweep<MODE, uint16_t><<<grid, SW_THREADS, smem, c->stream>>>(fp, E->rp, E->col, E->val, N, rows, nrows,
               E->desc.as<uint4>(), E->invl.as<u32>(), E->abits.as<u32>(), (uint16_t*)nullptr, Dp, K,
               E->nonA.as<u32>(), Rd, rankD, dpiv, pcol, pval, cap, cursor, s_off, s_len, err, stats);
    check_cuda(cudaGetLastError(), "k_sweep");
  } else {
    k_sweep<MODE, u32><<<grid, SW_THREADS, smem, c->stream>>>(fp, E->rp, E->col, E->val, N, rows, nrows,
               E->desc.as<uint4>(), E->invl.as<u32>(), E->abits.as<u32>(), (u32*)nullptr, Dp, K, E->nonA.as<u32>(),
               Rd, rankD, dpiv, pcol, pval, cap, cursor, s_off, s_len, err, stats);
    check_cuda(cudaGetLastError(), "k_sweep");
  }
}

static void run_a_sweep(Ctx* c, f4b_echelon* E, const std::vector<char>* want = nullptr);

// psge tail record (pool use, sweep counters, rank(D'), error flags) written
// by one thread into page-locked host memory (UVA)
__global__ void k_tail_gather(const unsigned long long* cursor, const unsigned long long* stats, const u32* rdev,
                              const u32* err, unsigned long long* out) {
  if (threadIdx.x != 0) return;
  volatile unsigned long long* o = out;
  o[0] = *cursor;
  o[1] = stats ? stats[0] : 0ull;
  o[2] = stats ? stats[1] : 0ull;
  o[3] = (unsigned long long)*rdev | ((unsigned long long)*err << 32);
  __threadfence_system();
}

static void psge_run(Ctx* c, f4b_echelon* E, int mode) {
  Fp fp = make_fp(c);
  static const bool etrace = getenv("F4B_ELIM_TRACE") != nullptr;
  const auto h0 = std::chrono::steady_clock::now();
  const long long a0 = c->raw_allocs, f0 = c->raw_frees;
  const double au0 = c->raw_alloc_us;
  std::vector<std::pair<const char*, double>> marks;
  // trace: host marks plus a device event per mark (device gaps = host work)
  static cudaEvent_t tev[12] = {};
  int ntev = 0;
  auto mark = [&](const char* w) {
    if (!etrace) return;
    marks.push_back({w, std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count()});
    if (ntev < 12) {
      if (!tev[ntev]) cudaEventCreate(&tev[ntev]);
      cudaEventRecord(tev[ntev++], c->stream);
    }
  };
  const long long r = E->n_rows, N = E->n_cols;
  cudaEvent_t ev0 = timing_event(c, 2), ev1 = timing_event(c, 3);
  check_cuda(cudaEventRecord(ev0, c->stream), "event");
  mark("start");
  ensure(c, c->errflag, 64);
  u32* err = c->errflag.as<u32>();
  check_cuda(cudaMemsetAsync(err, 0, 4, c->stream), "memset");
  const long long Nn = std::max<long long>(N, 1);
  WinPrep wpre;  // window tables queued behind k_psge_prep (see win_prepare)
  // E1: one cooperative launch (k_psge_prep) and one read of (nA, nC)
  DBuf pk, crows, pcnt;
  ensure(c, pk, Nn * sizeof(unsigned long long));
  ensure(c, E->prow, Nn * sizeof(u32));
  ensure(c, E->invl, Nn * sizeof(u32));
  ensure(c, E->desc, Nn * sizeof(uint4));
  ensure(c, E->abits, (size_t)((Nn + 31) / 32 + 1) * sizeof(u32));
  ensure(c, E->acols, (size_t)Nn * sizeof(u32));
  ensure(c, E->nonA, (size_t)Nn * sizeof(u32));
  ensure(c, E->apos, (size_t)Nn * sizeof(u32));
  ensure(c, crows, (size_t)std::max<long long>(r, 1) * sizeof(u32));
  {
    static int bpp = -1;
    if (bpp < 0) check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bpp, k_psge_prep, 256, 0), "occupancy");
    // every SM (a grid sized by the batch, ~2K rows per CTA, was measured
    // slower: 0.9 -> 1.2 ms of k_psge_prep per cyclic-8 step); F4B_PREP_G
    // overrides (experiments)
    static const int gp_env = getenv("F4B_PREP_G") ? atoi(getenv("F4B_PREP_G")) : 0;
    const int GP = gp_env > 0 ? std::min(gp_env, c->num_sms * std::max(1, std::min(bpp, 2)))
                              : c->num_sms * std::max(1, std::min(bpp, 2));
    ensure(c, pcnt, (size_t)GP * sizeof(u32) + sizeof(PrepOut) + 16);
    PrepOut* d_out = reinterpret_cast<PrepOut*>(pcnt.as<u32>() + GP);
    u32 ru = (u32)r, Nu = (u32)N;
    unsigned long long* pkp = pk.as<unsigned long long>();
    u32* prowp = E->prow.as<u32>();
    u32* invlp = E->invl.as<u32>();
    uint4* descp = E->desc.as<uint4>();
    u32* abitsp = E->abits.as<u32>();
    u32* acolsp = E->acols.as<u32>();
    u32* aposp = E->apos.as<u32>();
    u32* nonAp = E->nonA.as<u32>();
    u32* crowsp = crows.as<u32>();
    u32* cntp = pcnt.as<u32>();
    const u32* rpp = E->rp;
    const u32* colp = E->col;
    const u32* valp = E->val;
    void* args[] = {&fp, &rpp, &colp, &valp, &ru, &Nu, &pkp, &prowp, &invlp, &descp, &abitsp, &acolsp, &aposp,
                    &nonAp, &crowsp, &cntp, &d_out};
    {
      ProfScope ps(c, "k_psge_prep");
      check_cuda(cudaLaunchCooperativeKernel((void*)k_psge_prep, GP, 256, args, 0, c->stream), "k_psge_prep");
    }
    PrepOut ho;
    mark("prep launched");
    check_cuda(cudaMemcpyAsync(c->h_stat, d_out, sizeof(PrepOut), cudaMemcpyDeviceToHost, c->stream), "d2h");
    cudaEvent_t evp = timing_event(c, 0);
    check_cuda(cudaEventRecord(evp, c->stream), "event");
    // the window tables need only the device's nA: queued now, they run
    // while the host waits for (nA, nC)
    const long long nA_bound = std::min(r, N);
    if (win_eligible(c, (u32)N, nA_bound)) win_prepare(c, fp, E, &d_out->nA, (u32)nA_bound, wpre);
    check_cuda(cudaEventSynchronize(evp), "sync");
    mark("prep synced");
    memcpy(&ho, c->h_stat, sizeof(PrepOut));
    E->nA = ho.nA;
    E->K = N - E->nA;
    E->nC = ho.nC;
  }
  release(c, pk);
  release(c, pcnt);
  // E2: D' = C swept over the A columns
  const long long R = E->nC, K = E->K;
  DBuf Dp, cand, used, pofc, lead;
  E->rankD = 0;
  if (R > 0 && K > 0) {
    ensure(c, Dp, (size_t)R * K * sizeof(u32));
    ensure(c, E->stats, 16);
    check_cuda(cudaMemsetAsync(E->stats.p, 0, 16, c->stream), "memset");
    mark("sweep issue");
    launch_sweep<0>(c, fp, E, crows.as<u32>(), (u32)R, Dp.as<u32>(), (u32)K, nullptr, 0, nullptr, nullptr, nullptr, 0,
                    nullptr, nullptr, nullptr, err, E->stats.as<unsigned long long>(), &wpre);
    mark("sweep launched");
    // E3 default: RREF(D') in pivot blocks (k_dense_blk); c->opt_dense = 1
    // (f4b_ctx_set_option "dense") forces the general fallback below
    bool blk_done = false;
    if (c->opt_dense == 0 && R > 0 && K > 0 && R < (1ll << 30) && K < (1ll << 30)) {
      static int blk_occ = -1;
      static bool blk_attr = false;
      if (!blk_attr) {
        for (const void* kf : {(const void*)k_dense_blk<true, false>, (const void*)k_dense_blk<false, false>,
                               (const void*)k_dense_blk<true, true>, (const void*)k_dense_blk<false, true>})
          check_cuda(cudaFuncSetAttribute(kf, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024), "attr");
        blk_attr = true;
      }
      const long long rmaxb = std::max<long long>(1, std::min(R, K));
      long long rpc = std::max<long long>(2, (R + c->num_sms - 1) / c->num_sms);
      long long G = (R + rpc - 1) / rpc;
      const long long maxt = rpc + (rmaxb + G - 1) / G;
      const long long Kp = (K + 3) & ~3ll;
      const long long maxt3 = maxt + (DB_NP + G - 1) / G;
      size_t smem_b = (size_t)std::max<long long>(DB_NP * (DB_W + 32), maxt3 * (DB_NP + 3) + rpc) * 4;
      (void)Kp;
      // this CTA's rows resident in shared memory when they fit
      const bool sr = c->opt_dense_rows == 0 && smem_b + (size_t)rpc * K * 4 <= 196 * 1024;
      if (sr) smem_b += (size_t)rpc * K * 4;
      if (blk_occ < 0) {
        int o = 0;
        check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&o, k_dense_blk<false, true>, DB_THREADS, 196 * 1024),
                   "occupancy");
        blk_occ = o;
      }
      if (blk_occ >= 1 && G <= c->num_sms && smem_b <= 196 * 1024 && rpc * K < (1ll << 32)) {
        DBuf Bm, colp, lead_b, cand_b, gl, gT, stt, ordr;
        ensure(c, Bm, (size_t)rmaxb * K * sizeof(u32));
        ensure(c, colp, (size_t)K * sizeof(u32));
        ensure(c, lead_b, (size_t)R * sizeof(u32));
        ensure(c, cand_b, DB_NP * sizeof(u32));
        ensure(c, gl, 2 * DB_NP * sizeof(u32));
        ensure(c, gT, DB_NP * DB_NP * sizeof(u32));
        ensure(c, stt, sizeof(DblkState));
        ensure(c, ordr, (size_t)rmaxb * sizeof(u32));
        ensure(c, E->Rd, (size_t)rmaxb * K * sizeof(u32));
        ensure(c, E->dpiv, (size_t)rmaxb * sizeof(u32));
        ensure(c, E->rdev, 16);
        check_cuda(cudaMemsetAsync(colp.p, 0xFF, (size_t)K * sizeof(u32), c->stream), "memset");
        check_cuda(cudaMemsetAsync(stt.p, 0, sizeof(DblkState), c->stream), "memset");
        fp = make_fp(c);
        u32* dpp = Dp.as<u32>();
        u32 Ru = (u32)R, Ku = (u32)K, rpcu = (u32)rpc, maxtu = (u32)maxt3;
        u32 *leadp = lead_b.as<u32>(), *candp2 = cand_b.as<u32>(), *bmp = Bm.as<u32>(), *colpp = colp.as<u32>();
        u32 *glp = gl.as<u32>(), *gTp = gT.as<u32>(), *rdp = E->Rd.as<u32>(), *dpivp = E->dpiv.as<u32>();
        u32 *rkp = E->rdev.as<u32>(), *ordp = ordr.as<u32>();
        DblkState* sp = reinterpret_cast<DblkState*>(stt.p);
        static const bool btrace = getenv("F4B_BLK_TRACE") != nullptr;
        DBuf dfl;
        u32* dflp = nullptr;
        if (btrace) {
          ensure(c, dfl, (size_t)K * sizeof(u32));
          check_cuda(cudaMemsetAsync(dfl.p, 0, (size_t)K * sizeof(u32), c->stream), "memset");
          dflp = dfl.as<u32>();
        }
        void* argsb[] = {&fp, &dpp, &Ru, &Ku, &rpcu, &maxtu, &leadp, &candp2, &bmp, &colpp, &glp, &gTp, &sp, &rdp,
                         &dpivp, &rkp, &ordp, &dflp};
        {
          ProfScope ps(c, "k_dense_blk");
          const void* kf = c->p < 65536u ? (sr ? (const void*)k_dense_blk<true, true> : (const void*)k_dense_blk<true, false>)
                                          : (sr ? (const void*)k_dense_blk<false, true> : (const void*)k_dense_blk<false, false>);
          mark("dense issue");
          check_cuda(cudaLaunchCooperativeKernel(kf, (int)G, DB_THREADS, argsb, smem_b, c->stream), "k_dense_blk");
          mark("dense launched");
        }
        if (btrace) {
          release(c, dfl);
          DblkState hs;
          check_cuda(cudaMemcpyAsync(&hs, stt.p, sizeof(hs), cudaMemcpyDeviceToHost, c->stream), "d2h");
          check_cuda(cudaStreamSynchronize(c->stream), "sync");
          fprintf(stderr, "[blk] R=%lld K=%lld G=%lld rpc=%lld rank=%u iters=%u t2=%uus (load %u fwd %u back %u) t3=%uus (setup %uus) offers=%u distinct=%u fwd_kcyc(min+bar %u upd %u bar %u n %u) cta1(setup+coef %u apply %u offers %u us)\n",
                  (long long)R, (long long)K, (long long)G, (long long)rpc, hs.rho, hs.iters, hs.t2_us, hs.t2a_us,
                  hs.t2b_us, hs.t2c_us, hs.t3_us, hs.t3a_us, hs.offers, hs.distinct, hs.fc1, hs.fc2, hs.fc3, hs.fcn, hs.q1, hs.q2, hs.q3);
        }
        for (DBuf* b : {&Bm, &colp, &lead_b, &cand_b, &gl, &gT, &stt, &ordr}) release(c, *b);
        blk_done = true;
      }
    }
    if (blk_done) {
    } else {
    // E3a: cooperative forward elimination
    ensure(c, used, (size_t)R + 16);
    ensure(c, pofc, (size_t)K * sizeof(u32));
    ensure(c, cand, (size_t)(std::min(R, K) + 2) * sizeof(unsigned long long));
    ensure(c, lead, (size_t)R * sizeof(u32));
    check_cuda(cudaMemsetAsync(cand.p, 0xFF, (std::min(R, K) + 2) * sizeof(unsigned long long), c->stream), "memset");
    check_cuda(cudaMemsetAsync(used.p, 0, R, c->stream), "memset");
    check_cuda(cudaMemsetAsync(pofc.p, 0xFF, (size_t)K * sizeof(u32), c->stream), "memset");
    int bps = 0;
    check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_dense_forward, 256, 0), "occupancy");
    int G = (int)std::min<long long>((long long)c->num_sms * std::max(1, std::min(bps, 2)), std::max<long long>(R, 1));
    u32* dpp = Dp.as<u32>();
    u32 Ru = (u32)R, Ku = (u32)K;
    unsigned long long* candp = cand.as<unsigned long long>();
    u32* leadp = lead.as<u32>();
    uint8_t* usedp = used.as<uint8_t>();
    u32* pofcp = pofc.as<u32>();
    void* args[] = {&fp, &dpp, &Ru, &Ku, &candp, &leadp, &usedp, &pofcp};
    {
      ProfScope ps(c, "k_dense_forward");
      check_cuda(cudaLaunchCooperativeKernel((void*)k_dense_forward, G, 256, args, 0, c->stream), "k_dense_forward");
    }
    // pivots of D' (k_dense_post: one CTA, rank(D') stays on the device)
    const long long rmax = std::max<long long>(1, std::min(R, K));
    DBuf pinv, dprow, pbits;
    ensure(c, pinv, (size_t)K * sizeof(u32));
    ensure(c, E->dpiv, (size_t)rmax * sizeof(u32));
    ensure(c, dprow, (size_t)rmax * sizeof(u32));
    ensure(c, pbits, (size_t)((K + 31) / 32 + 1) * sizeof(u32));
    ensure(c, E->rdev, 16);
    F4B_LAUNCH(c, k_dense_post, 1, 1024, 0, fp, Dp.as<u32>(), (u32)K, pofc.as<u32>(), pinv.as<u32>(),
               E->dpiv.as<u32>(), dprow.as<u32>(), pbits.as<u32>(), E->rdev.as<u32>());
    ensure(c, E->Rd, (size_t)rmax * K * sizeof(u32));
    {
      size_t smem2 = (size_t)((K + 31) / 32) * 4 + (size_t)K * 4;
      DBuf gacc2;
      const bool gl2 = smem2 > 200 * 1024;  // accumulator in HBM for very wide blocks
      if (gl2) smem2 = (size_t)((K + 31) / 32) * 4;
      static bool attr1 = false;
      if (!attr1) {
        check_cuda(cudaFuncSetAttribute(k_dense_back, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 4096),
                   "attr");
        attr1 = true;
      }
      int g2 = sweep_grid(c, smem2, rmax);
      if (gl2) ensure(c, gacc2, (size_t)g2 * K * sizeof(u32));
      F4B_LAUNCH(c, k_dense_back, g2, SW_THREADS, smem2, fp, Dp.as<u32>(), (u32)K, E->dpiv.as<u32>(), dprow.as<u32>(),
                 E->rdev.as<u32>(), pbits.as<u32>(), pinv.as<u32>(), pofc.as<u32>(), E->Rd.as<u32>(),
                 gl2 ? gacc2.as<u32>() : nullptr);
      release(c, gacc2);
    }
    release(c, pinv);
    release(c, dprow);
    release(c, pbits);
    }
  } else {
    ensure(c, E->rdev, 16);
    check_cuda(cudaMemsetAsync(E->rdev.p, 0, 4, c->stream), "memset");
  }
  if (wpre.ok) win_release(c, wpre);  // no sweep (R = 0 or K = 0)
  release(c, Dp);
  release(c, cand);
  release(c, used);
  release(c, pofc);
  release(c, lead);
  release(c, crows);
  // E3c: emit the nonpivot rows (RREF(D')); sizes from rank(D') <= min(R, K)
  // so nothing waits for the host; one read-back of (rank, pool use, error
  // flag, sweep counters) at the end
  const long long rmax = (R > 0 && K > 0) ? std::max<long long>(1, std::min(R, K)) : 1;
  ensure(c, E->d_off, (size_t)rmax * sizeof(u32));
  ensure(c, E->d_len, (size_t)rmax * sizeof(u32));
  ensure(c, E->cursor, 16);
  if (E->pool_cap == 0) {
    E->pool_cap = (size_t)std::max<long long>(((R > 0 && K > 0) ? rmax * K : 0) + 2 * (long long)E->nA * 64 + 4096,
                                              1 << 20);
  }
  struct Tail {
    unsigned long long used_pool, st[2];
    u32 rankD, err;
  };
  Tail* ht = reinterpret_cast<Tail*>(c->h_stat);
  for (int attempt = 0; attempt < 8; ++attempt) {
    ensure(c, E->pool_col, E->pool_cap * sizeof(u32));
    ensure(c, E->pool_val, E->pool_cap * sizeof(u32));
    check_cuda(cudaMemsetAsync(E->cursor.p, 0, 8, c->stream), "memset");
    check_cuda(cudaMemsetAsync(err, 0, 4, c->stream), "memset");
    if (R > 0 && K > 0) {
      int g = (int)std::min<long long>(rmax, (long long)c->num_sms * 4);
      F4B_LAUNCH(c, k_emit_dense, g, SW_THREADS, 0, E->Rd.as<u32>(), (u32)K, E->rdev.as<u32>(), E->dpiv.as<u32>(),
                 E->nonA.as<u32>(), E->pool_col.as<u32>(), E->pool_val.as<u32>(), E->pool_cap,
                 E->cursor.as<unsigned long long>(), E->d_off.as<u32>(), E->d_len.as<u32>(), err);
      check_cuda(cudaGetLastError(), "k_emit_dense");
    }
    // one tiny kernel stores (pool use, sweep counters, rank, error) straight
    // into the page-locked host block (4 D2H copies before)
    F4B_LAUNCH(c, k_tail_gather, 1, 32, 0, E->cursor.as<unsigned long long>(),
               E->stats.p ? E->stats.as<unsigned long long>() : nullptr, E->rdev.as<u32>(), err,
               reinterpret_cast<unsigned long long*>(ht));
    check_cuda(cudaStreamSynchronize(c->stream), "sync");
    if (!(ht->err & DEVERR_CAPACITY)) break;
    if (attempt == 7) fail(F4B_ERR_OOM, "psge: nonpivot row pool still overflows after 8 resizes");
    // the cursor counts every requested slot, also past the capacity
    E->pool_cap = std::max<size_t>(2 * E->pool_cap, (size_t)ht->used_pool + 1024);
  }
  mark("tail synced");
  E->rankD = ht->rankD;
  const long long rankD = E->rankD;
  E->sweep_pivots = ht->st[0];
  E->sweep_tail_nnz = ht->st[1];
  E->nonpivot_nnz = (long long)ht->used_pool;
  check_cuda(cudaEventRecord(ev1, c->stream), "event");
  check_cuda(cudaEventSynchronize(ev1), "event sync");
  float ms = 0;
  cudaEventElapsedTime(&ms, ev0, ev1);
  E->numeric_ns = (int64_t)(ms * 1e6);
  static const float etrace_ms = etrace ? (float)atof(getenv("F4B_ELIM_TRACE")) : 0.f;  // print above this device time
  if (etrace && ms > etrace_ms) {
    fprintf(stderr, "[elim] r=%lld N=%lld R=%lld K=%lld dev=%.2fms allocs=%lld frees=%lld alloc_us=%.0f:", (long long)r,
            (long long)N, (long long)E->nC, (long long)E->K, ms, c->raw_allocs - a0, c->raw_frees - f0,
            c->raw_alloc_us - au0);
    for (size_t i = 0; i < marks.size(); ++i) {
      float dm = 0;
      if (i > 0 && (int)i < ntev) cudaEventElapsedTime(&dm, tev[i - 1], tev[i]);
      fprintf(stderr, " %s @%.0f (dev +%.0fus) |", marks[i].first, marks[i].second, dm * 1e3);
    }
    fprintf(stderr, "\n");
  }
  E->zero_rows = r - (E->nA + rankD);
  if (mode == F4B_FULL_RREF) run_a_sweep(c, E);
}

// pivot-row slots of a subset sweep scattered to their A positions
__global__ void k_scatter_slots(const u32* __restrict__ so, const u32* __restrict__ sl, const u32* __restrict__ pos,
                                u32 n, u32* __restrict__ off, u32* __restrict__ len) {
  const u32 i = blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    off[pos[i]] = so[i];
    len[pos[i]] = sl[i];
  }
}

// FULL_RREF's pivot rows (sparselin.py:337-349); `want` (optional, a flag
// per column) restricts the back-reduction to the pivot rows led by the
// flagged columns — the others are left empty (echelon_complete_rows)
static void run_a_sweep(Ctx* c, f4b_echelon* E, const std::vector<char>* want) {
  if (E->full && !(E->partial && !want)) return;
  Fp fp = make_fp(c);
  const long long N = E->n_cols, nA = E->nA, K = E->K;
  cudaEvent_t ev0 = timing_event(c, 2), ev1 = timing_event(c, 3);
  check_cuda(cudaEventRecord(ev0, c->stream), "event");
  ensure(c, E->a_off, (size_t)std::max<long long>(nA, 1) * sizeof(u32));
  ensure(c, E->a_len, (size_t)std::max<long long>(nA, 1) * sizeof(u32));
  ensure(c, c->errflag, 64);
  u32* err = c->errflag.as<u32>();
  if (nA) {
    DBuf arows, gacc;
    ensure(c, arows, (size_t)nA * sizeof(u32));
    // A rows in ascending lead-column order: arows[k] = prow[acols[k]]
    std::vector<u32> h_acols(nA), h_prow(N);
    check_cuda(cudaMemcpyAsync(h_acols.data(), E->acols.p, nA * sizeof(u32), cudaMemcpyDeviceToHost, c->stream), "d2h");
    check_cuda(cudaMemcpyAsync(h_prow.data(), E->prow.p, N * sizeof(u32), cudaMemcpyDeviceToHost, c->stream), "d2h");
    check_cuda(cudaStreamSynchronize(c->stream), "sync");
    std::vector<u32> h_arows, h_pos;
    h_arows.reserve(nA);
    for (long long k = 0; k < nA; ++k)
      if (!want || (*want)[h_acols[k]]) {
        h_arows.push_back(h_prow[h_acols[k]]);
        h_pos.push_back((u32)k);
      }
    const long long ns = (long long)h_arows.size();
    DBuf sub, posb;
    if (want) {  // subset: slots indexed by subset position, scattered afterwards; the rest empty
      ensure(c, sub, (size_t)std::max<long long>(2 * ns, 1) * sizeof(u32));
      ensure(c, posb, (size_t)std::max<long long>(ns, 1) * sizeof(u32));
      check_cuda(cudaMemsetAsync(E->a_off.p, 0, nA * sizeof(u32), c->stream), "memset");
      check_cuda(cudaMemsetAsync(E->a_len.p, 0, nA * sizeof(u32), c->stream), "memset");
      if (ns) check_cuda(cudaMemcpyAsync(posb.p, h_pos.data(), ns * sizeof(u32), cudaMemcpyHostToDevice, c->stream), "h2d");
    }
    if (ns) check_cuda(cudaMemcpyAsync(arows.p, h_arows.data(), ns * sizeof(u32), cudaMemcpyHostToDevice, c->stream), "h2d");
    u32* s_off = want ? sub.as<u32>() : E->a_off.as<u32>();
    u32* s_len = want ? sub.as<u32>() + std::max<long long>(ns, 1) : E->a_len.as<u32>();
    size_t base_used = (size_t)E->nonpivot_nnz;
    for (int attempt = 0; attempt < 8; ++attempt) {
      size_t need = base_used + (size_t)std::max<long long>(2 * E->M, 1 << 20);
      if (E->pool_cap < need) {
        // grow, preserving the nonpivot rows already in the pool
        E->pool_cap = std::max(need, 2 * E->pool_cap);
        ensure_keep(c, E->pool_col, E->pool_cap * sizeof(u32));
        ensure_keep(c, E->pool_val, E->pool_cap * sizeof(u32));
      }
      unsigned long long cur = base_used;
      check_cuda(cudaMemcpyAsync(E->cursor.p, &cur, 8, cudaMemcpyHostToDevice, c->stream), "h2d");
      check_cuda(cudaMemsetAsync(err, 0, 4, c->stream), "memset");
      if (ns)
        launch_sweep<1>(c, fp, E, arows.as<u32>(), (u32)ns, nullptr, (u32)K, E->rankD ? E->Rd.as<u32>() : nullptr,
                        (u32)E->rankD, E->rankD ? E->dpiv.as<u32>() : nullptr, E->pool_col.as<u32>(),
                        E->pool_val.as<u32>(), E->pool_cap, E->cursor.as<unsigned long long>(), s_off, s_len, err);
      u32 e = read_u32(c, err);
      if (!(e & DEVERR_CAPACITY)) break;
      if (attempt == 7) fail(F4B_ERR_OOM, "psge: pivot row pool still overflows after 8 resizes");
      unsigned long long tot = 0;
      check_cuda(cudaMemcpy(&tot, E->cursor.p, 8, cudaMemcpyDeviceToHost), "d2h");
      E->pool_cap = std::max<size_t>(2 * E->pool_cap, (size_t)tot + 1024);
      ensure_keep(c, E->pool_col, E->pool_cap * sizeof(u32));
      ensure_keep(c, E->pool_val, E->pool_cap * sizeof(u32));
    }
    unsigned long long tot = 0;
    check_cuda(cudaMemcpyAsync(&tot, E->cursor.p, 8, cudaMemcpyDeviceToHost, c->stream), "d2h");
    check_cuda(cudaStreamSynchronize(c->stream), "sync");
    E->pivot_nnz = (long long)tot - (long long)base_used;
    if (want && ns)
      F4B_LAUNCH(c, k_scatter_slots, nb(ns, 256), 256, 0, sub.as<u32>(), sub.as<u32>() + std::max<long long>(ns, 1),
                 posb.as<u32>(), (u32)ns, E->a_off.as<u32>(), E->a_len.as<u32>());
    release(c, arows);
    release(c, gacc);
    release(c, sub);
    release(c, posb);
  }
  check_cuda(cudaEventRecord(ev1, c->stream), "event");
  check_cuda(cudaEventSynchronize(ev1), "event sync");
  float ms = 0;
  cudaEventElapsedTime(&ms, ev0, ev1);
  E->backsub_ns = (int64_t)(ms * 1e6);
  E->full = true;
  E->partial = want != nullptr;
}

f4b_echelon* psge_plan(Ctx* c, const f4b_plan* pl, int mode) {
  f4b_echelon* E = new f4b_echelon();
  E->ctx = c;
  E->n_rows = pl->r;
  E->n_cols = pl->N;
  E->M = pl->M;
  E->rp = pl->row_ptr.as<u32>();
  E->col = pl->col_ind.as<u32>();
  E->val = pl->val.as<u32>();
  try {
    psge_run(c, E, mode);
  } catch (...) {
    echelon_release(E);
    throw;
  }
  return E;
}

f4b_echelon* psge_csr(Ctx* c, long long r, long long N, const int64_t* rp, const int64_t* col, const uint64_t* val,
                      int mode) {
  f4b_echelon* E = new f4b_echelon();
  E->ctx = c;
  E->n_rows = r;
  E->n_cols = N;
  try {
    long long M = rp[r];
    E->M = M;
    // the elimination kernels index rows, columns and nonzeros with u32
    if (M < 0 || M >= (1ll << 32) - 1 || N >= (1ll << 31) || r >= (1ll << 31))
      fail(F4B_ERR_SIZE_CAP, "psge: nnz must stay below 2^32 - 1, rows and columns below 2^31");
    std::vector<u32> hrp(r + 1), hcol(std::max<long long>(M, 1)), hval(std::max<long long>(M, 1));
    for (long long i = 0; i <= r; ++i) hrp[i] = (u32)rp[i];
    for (long long k = 0; k < M; ++k) {
      if (col[k] < 0 || col[k] >= N) fail(F4B_ERR_PROPERTY, "column out of range");
      if (val[k] == 0 || val[k] >= c->p) fail(F4B_ERR_PROPERTY, "CSR values outside [1, p)");
      hcol[k] = (u32)col[k];
      hval[k] = (u32)val[k];
    }
    ensure(c, E->own_rp, (r + 1) * sizeof(u32));
    ensure(c, E->own_col, hcol.size() * sizeof(u32));
    ensure(c, E->own_val, hval.size() * sizeof(u32));
    check_cuda(cudaMemcpyAsync(E->own_rp.p, hrp.data(), (r + 1) * sizeof(u32), cudaMemcpyHostToDevice, c->stream), "h2d");
    check_cuda(cudaMemcpyAsync(E->own_col.p, hcol.data(), hcol.size() * sizeof(u32), cudaMemcpyHostToDevice, c->stream),
               "h2d");
    check_cuda(cudaMemcpyAsync(E->own_val.p, hval.data(), hval.size() * sizeof(u32), cudaMemcpyHostToDevice, c->stream),
               "h2d");
    E->rp = E->own_rp.as<u32>();
    E->col = E->own_col.as<u32>();
    E->val = E->own_val.as<u32>();
    psge_run(c, E, mode);
    check_cuda(cudaStreamSynchronize(c->stream), "sync");
  } catch (...) {
    echelon_release(E);
    throw;
  }
  return E;
}

void echelon_complete(Ctx* c, f4b_echelon* E) { run_a_sweep(c, E); }

void echelon_complete_rows(Ctx* c, f4b_echelon* E, const int64_t* lead_cols, long long n) {
  std::vector<char> want((size_t)std::max<long long>(E->n_cols, 1), 0);
  for (long long i = 0; i < n; ++i)
    if (lead_cols[i] >= 0 && lead_cols[i] < E->n_cols) want[(size_t)lead_cols[i]] = 1;
  if (E->full && !E->partial) return;  // every pivot row is already there
  E->full = false;
  run_a_sweep(c, E, &want);
}

void echelon_info(const f4b_echelon* E, f4b_echelon_info* info) {
  info->n_rows = E->n_rows;
  info->n_cols = E->n_cols;
  info->rank = E->nA + E->rankD;
  info->zero_rows = E->zero_rows;
  info->n_pivot_rows = E->nA;
  info->n_nonpivot_rows = E->rankD;
  info->pivot_nnz = E->pivot_nnz;
  info->nonpivot_nnz = E->nonpivot_nnz;
  info->full = E->full ? (E->partial ? 2 : 1) : 0;
  info->numeric_ns = E->numeric_ns;
  info->backsub_ns = E->backsub_ns;
  info->dense_rows = E->nC;
  info->dense_cols = E->K;
  info->sweep_pivots = (int64_t)E->sweep_pivots;
  info->sweep_tail_nnz = (int64_t)E->sweep_tail_nnz;
}

void echelon_download(const f4b_echelon* E, int which, int64_t* leads, int64_t* row_ptr, int64_t* cols,
                      uint64_t* vals) {
  Ctx* c = E->ctx;
  const long long n = which == 0 ? E->nA : E->rankD;
  if (which == 0 && !E->full) fail(F4B_ERR_PRECONDITION, "pivot rows not computed (NEW_ONLY echelon)");
  std::vector<u32> off(n), len(n), lead(n);
  if (n) {
    const DBuf& o = which == 0 ? E->a_off : E->d_off;
    const DBuf& l = which == 0 ? E->a_len : E->d_len;
    check_cuda(cudaMemcpyAsync(off.data(), o.p, n * sizeof(u32), cudaMemcpyDeviceToHost, c->stream), "d2h");
    check_cuda(cudaMemcpyAsync(len.data(), l.p, n * sizeof(u32), cudaMemcpyDeviceToHost, c->stream), "d2h");
    if (which == 0) {
      check_cuda(cudaMemcpyAsync(lead.data(), E->acols.p, n * sizeof(u32), cudaMemcpyDeviceToHost, c->stream), "d2h");
    }
  }
  const long long used = E->nonpivot_nnz + (E->full ? E->pivot_nnz : 0);
  std::vector<u32> pc(std::max<long long>(used, 1)), pv(std::max<long long>(used, 1));
  if (used) {
    check_cuda(cudaMemcpyAsync(pc.data(), E->pool_col.p, used * sizeof(u32), cudaMemcpyDeviceToHost, c->stream), "d2h");
    check_cuda(cudaMemcpyAsync(pv.data(), E->pool_val.p, used * sizeof(u32), cudaMemcpyDeviceToHost, c->stream), "d2h");
  }
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  long long at = 0;
  if (row_ptr) row_ptr[0] = 0;
  for (long long k = 0; k < n; ++k) {
    if (leads) leads[k] = which == 0 ? (int64_t)lead[k] : (int64_t)pc[off[k]];
    for (u32 t = 0; t < len[k]; ++t) {
      if (cols) cols[at + t] = pc[off[k] + t];
      if (vals) vals[at + t] = pv[off[k] + t];
    }
    at += len[k];
    if (row_ptr) row_ptr[k + 1] = at;
  }
}

// ---------------------------------------------------------------------------
// Harvest on the device (reference groebner.py:285-290): the
// nonpivot rows of an echelon appended to the device basis in the driver's
// order (ascending key(LM) = descending lead column), exponents gathered from
// the plan dictionary by column, no host round trip of the terms.
// ---------------------------------------------------------------------------
__global__ void k_append_rows(const u32* __restrict__ d_off, const u32* __restrict__ d_len, u32 nnew,
                              const u32* __restrict__ noff, const u32* __restrict__ pcol, const u32* __restrict__ pval,
                              const u16* __restrict__ dict_exps, int n, long long T0, u16* __restrict__ exps,
                              u32* __restrict__ coeff, u16* __restrict__ lm, u16* __restrict__ maxe) {
  const u32 i = blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5);  // new polynomial (warp)
  const int lane = threadIdx.x & 31;
  if (i >= nnew) return;
  const u32 k = nnew - 1 - i;  // source row: descending lead
  const u32 so = d_off[k], L = d_len[k], to = noff[i];
  for (u32 t = lane; t < L; t += 32) {
    const u32 cc = pcol[so + t];
    for (int v = 0; v < n; ++v) exps[(T0 + to + t) * n + v] = dict_exps[(size_t)cc * n + v];
    coeff[T0 + to + t] = pval[so + t];
  }
  for (int v = 0; v < n; ++v) {
    u32 mx = 0;
    for (u32 t = lane; t < L; t += 32) mx = max(mx, (u32)dict_exps[(size_t)pcol[so + t] * n + v]);
    mx = __reduce_max_sync(0xffffffffu, mx);
    if (lane == 0) {
      maxe[(size_t)i * n + v] = (u16)mx;
      lm[(size_t)i * n + v] = L ? dict_exps[(size_t)pcol[so] * n + v] : (u16)0;
    }
  }
}

void basis_append_echelon(Ctx* c, const f4b_plan* pl, const f4b_echelon* E) {
  Basis& B = c->basis;
  const int n = c->n_vars;
  const long long nnew = E->rankD;
  if (!nnew) return;
  if (pl->ctx != c || E->ctx != c) fail(F4B_ERR_PRECONDITION, "plan / echelon of another context");
  std::vector<u32> len(nnew);
  check_cuda(cudaMemcpyAsync(len.data(), E->d_len.p, nnew * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  const long long T0 = B.n_terms, P0 = B.n_polys, P1 = P0 + nnew;
  std::vector<u32> noff(nnew + 1);
  long long T = 0;
  for (long long i = 0; i < nnew; ++i) {
    noff[i] = (u32)T;
    T += len[nnew - 1 - i];
  }
  noff[nnew] = (u32)T;
  const long long T1 = T0 + T;
  if (T1 >= (1ll << 31)) fail(F4B_ERR_SIZE_CAP, "basis has more than 2^31 terms");
  ensure_keep(c, B.exps, (size_t)(T1 + 1) * n * sizeof(u16));
  ensure_keep(c, B.coeff, (size_t)(T1 + 1) * sizeof(u32));
  ensure_keep(c, B.off, (size_t)(P1 + 1) * sizeof(u32));
  ensure_keep(c, B.len, (size_t)(P1 + 1) * sizeof(u32));
  ensure_keep(c, B.lmexp, (size_t)(P1 + 1) * n * sizeof(u16));
  ensure_keep(c, B.maxe, (size_t)(P1 + 1) * n * sizeof(u16));
  DBuf dno;
  ensure(c, dno, (size_t)(nnew + 1) * 4);
  check_cuda(cudaMemcpyAsync(dno.p, noff.data(), (nnew + 1) * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
  F4B_LAUNCH(c, k_append_rows, nb(nnew, 8), 256, 0, E->d_off.as<u32>(), E->d_len.as<u32>(), (u32)nnew, dno.as<u32>(),
             E->pool_col.as<u32>(), E->pool_val.as<u32>(), pl->dict_exps.as<u16>(), n, T0, B.exps.as<u16>(),
             B.coeff.as<u32>(), B.lmexp.as<u16>() + P0 * n, B.maxe.as<u16>() + P0 * n);
  // offsets / lengths of the new polynomials; LM and max-exponent mirrors back
  std::vector<u32> hoff(nnew + 1), hlen(nnew);
  for (long long i = 0; i <= nnew; ++i) hoff[i] = (u32)(B.h_off.back() + noff[i]);
  for (long long i = 0; i < nnew; ++i) hlen[i] = len[nnew - 1 - i];
  check_cuda(cudaMemcpyAsync(B.off.as<u32>() + P0, hoff.data(), (nnew + 1) * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
  check_cuda(cudaMemcpyAsync(B.len.as<u32>() + P0, hlen.data(), nnew * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
  std::vector<uint16_t> hlm((size_t)nnew * n), hmx((size_t)nnew * n);
  check_cuda(cudaMemcpyAsync(hlm.data(), B.lmexp.as<u16>() + P0 * n, hlm.size() * 2, cudaMemcpyDeviceToHost, c->stream), "d2h");
  check_cuda(cudaMemcpyAsync(hmx.data(), B.maxe.as<u16>() + P0 * n, hmx.size() * 2, cudaMemcpyDeviceToHost, c->stream), "d2h");
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  release(c, dno);
  for (long long i = 0; i < nnew; ++i) {
    B.h_len.push_back(hlen[i]);
    B.h_off.push_back(B.h_off.back() + hlen[i]);
  }
  B.h_lm.insert(B.h_lm.end(), hlm.begin(), hlm.end());
  B.h_maxe.insert(B.h_maxe.end(), hmx.begin(), hmx.end());
  B.n_polys = (int)P1;
  B.n_terms = T1;
}

// All pivot columns, ascending: A columns merged with the D' pivots.
void echelon_pivot_cols(const f4b_echelon* E, int64_t* cols) {
  Ctx* c = E->ctx;
  std::vector<u32> a(std::max<long long>(E->nA, 1)), d(std::max<long long>(E->rankD, 1)),
      nonA(std::max<long long>(E->K, 1));
  if (E->nA) check_cuda(cudaMemcpyAsync(a.data(), E->acols.p, E->nA * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
  if (E->rankD) {
    check_cuda(cudaMemcpyAsync(d.data(), E->dpiv.p, E->rankD * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
    check_cuda(cudaMemcpyAsync(nonA.data(), E->nonA.p, E->K * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
  }
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  long long i = 0, j = 0, o = 0;
  while (i < E->nA || j < E->rankD) {
    long long x = i < E->nA ? (long long)a[i] : LLONG_MAX;
    long long y = j < E->rankD ? (long long)nonA[d[j]] : LLONG_MAX;
    if (x < y) {
      cols[o++] = x;
      ++i;
    } else {
      cols[o++] = y;
      ++j;
    }
  }
}

void echelon_release(f4b_echelon* E) {
  if (!E) return;
  Ctx* c = E->ctx;
  DBuf* bufs[] = {&E->own_rp, &E->own_col, &E->own_val, &E->prow,  &E->invl, &E->desc, &E->abits, &E->acols,
                  &E->nonA,   &E->Rd,      &E->dpiv,    &E->pool_col, &E->pool_val, &E->a_off, &E->a_len,
                  &E->d_off,  &E->d_len,   &E->cursor, &E->stats, &E->apos};
  for (DBuf* b : bufs) release(c, *b);
  delete E;
}

}  // namespace f4b
