// FBSP symbolic preprocessing on the device — the ★★ path of the north star.
//
// Restates reference `compile_batch` (pkg/src/fpgb/symbolic.py:293-388) with
// `_materialize` (:204-225), `closure_expand` (:238-278),
// `_reducer_preference` (:228-235), `_merge_dict` (:281-290) and the
// dictionary join (bulk.py:207-241), producing a byte-identical LayoutPlan.
//
// Per round (round 0 = the input rows, round k = closure rows of round k):
//   K1 k_tile_dict      fill (shifted keys generated on the fly from the
//                       HBM-resident basis: key = basis_key + row delta) +
//                       shared-memory radix sort + unique of a tile of keys,
//                       runs compacted with decoupled look-back.  The M keys
//                       never round-trip through HBM.
//   K2 sort_unique      one-sweep radix sort + unique of the tile survivors
//                       (radix.cu); for closure rounds it also drops keys
//                       already in the dictionary -> the next frontier.
//   K3 k_merge_corank   dictionary ∪ new keys (disjoint, both ascending).
//   K4 k_closure_search first basis LM dividing each frontier monomial in
//                       (key(LM), index) order (warp ballot, SWAR u16x2).
//   K5 k_new_rows       compaction of the reducers found, in ascending key(m)
//                       order, with row offsets (two look-backs).
// Final: k_join_gen regenerates every key and binary-searches the
//        shared-memory dictionary -> col_ind = N-1-pos and val.
// Host round trips: one small counter read per closure round (grids of the
// round are sized by upper bounds; kernels read the true sizes on device).
#include <cooperative_groups.h>

#include <algorithm>
#include <chrono>
#include <cstdio>
#include <cstring>
#include <cstdlib>
#include <vector>

#include "block.cuh"
#include "common.cuh"
#include "engine.h"
#include "rank.cuh"
#include "fbsp_internal.cuh"

namespace f4b {

static constexpr int K1_THREADS = 512;

template <int KW>
struct K1Cfg {
  static constexpr int ITEMS = KW >= 4 ? 4 / (KW / 4) : (KW == 2 ? 8 : 16);
  static constexpr int TILE = K1_THREADS * ITEMS;
  static constexpr int SROWS = 1024;  // rows of a tile staged in shared memory
  static constexpr size_t SMEM = (size_t)2 * TILE * KW * 8 + 16 * 256 * 4 + (size_t)SROWS * (KW * 8 + 8) + 16;
};

// device-side counters of one compile_batch call
struct DevCounters {
  u32 U;     // tile survivors of the current round
  u32 N;     // dictionary size after round 0
  u32 nf;    // frontier size
  u32 R;     // new rows of the round
  u32 Mk;    // terms of the new rows
  u32 ndict; // dictionary size uploaded for the absent filter
  u32 err;
  u32 pad;
  u32 tickets[16];
};

template <int KW>
__global__ void k_encode_basis(KeyFmt f, const u16* __restrict__ exps, long long t0, long long t1,
                               u64* __restrict__ ckey) {
  long long t = t0 + (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (t >= t1) return;
  u16 e[MAXV];
  for (int v = 0; v < f.n_vars; ++v) e[v] = exps[t * f.n_vars + v];
  key_store<KW>(ckey, t, key_encode<KW>(f, e));
}

template <int KW>
__global__ void k_rows0(KeyFmt f, long long r, const int* __restrict__ rb, const u16* __restrict__ shift,
                        const u32* __restrict__ blen, u64* __restrict__ delta, u32* __restrict__ rlen) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r) return;
  u16 e[MAXV], z[MAXV];
  for (int v = 0; v < f.n_vars; ++v) {
    e[v] = shift[i * f.n_vars + v];
    z[v] = 0;
  }
  key_store<KW>(delta, i, key_sub<KW>(key_encode<KW>(f, e), key_encode<KW>(f, z)));
  rlen[i] = blen[rb[i]];
}

// row owning term t among rows [lo, hi): rstart[row] <= t < rstart[row+1]
F4B_DEV u32 row_of_term(const u32* __restrict__ rstart, u32 lo, u32 hi, u32 t) {
  while (lo + 1 < hi) {
    const u32 mid = (lo + hi) >> 1;
    if (rstart[mid] <= t) lo = mid; else hi = mid;
  }
  return lo;
}

// Keys (and optionally coefficients) of terms [t, t + cnt), walking rows forward.
template <int KW>
F4B_DEV void gen_keys(u32 t, int cnt, u32 r_lo, u32 r_hi, const int* __restrict__ rb,
                      const u64* __restrict__ delta, const u32* __restrict__ rstart, const u32* __restrict__ boff,
                      const u64* __restrict__ bckey, Key<KW>* dst, const u32* __restrict__ bcoeff, u32* vals) {
  u32 row = row_of_term(rstart, r_lo, r_hi, t);
  u32 rs = rstart[row], re = rstart[row + 1];
  int g = rb[row];
  Key<KW> d = key_load<KW>(delta, row);
  u32 bo = boff[g];
  for (int i = 0; i < cnt; ++i, ++t) {
    while (t >= re) {
      ++row;
      rs = re;
      re = rstart[row + 1];
      g = rb[row];
      d = key_load<KW>(delta, row);
      bo = boff[g];
    }
    dst[i] = key_add<KW>(key_load<KW>(bckey, (long long)bo + (t - rs)), d);
    if (vals) vals[i] = __ldg(bcoeff + bo + (t - rs));
  }
}

// K1: fill + tile sort + unique + look-back compaction.
// m_hi / r_hi may come from device counters (closure rounds: d_Mk / d_R set
// by k_new_rows), so the grid can be an upper bound; surplus tiles exit.
template <int KW>
__global__ void __launch_bounds__(K1_THREADS) k_tile_dict(u32 m_lo, u32 m_hi_host, const u32* __restrict__ d_mk,
                                                          u32 r_lo, u32 r_hi_host, const u32* __restrict__ d_r,
                                                          const int* __restrict__ rb, const u64* __restrict__ delta,
                                                          const u32* __restrict__ rstart,
                                                          const u32* __restrict__ boff, const u64* __restrict__ bckey,
                                                          int bits, u64* __restrict__ out, u32* status,
                                                          u32* ticket, u32* d_U) {
  constexpr int ITEMS = K1Cfg<KW>::ITEMS;
  constexpr int TILE = K1Cfg<KW>::TILE;
  constexpr int SROWS = K1Cfg<KW>::SROWS;
  extern __shared__ __align__(16) unsigned char smraw[];
  Key<KW>* a = reinterpret_cast<Key<KW>*>(smraw);
  Key<KW>* b = a + TILE;
  Key<KW>* sdel = b + TILE;
  u32* wh = reinterpret_cast<u32*>(sdel + SROWS);
  u32* srs = wh + 16 * 256;      // row starts of the staged rows (+1)
  u32* sbo = srs + SROWS + 1;    // basis offsets of the staged rows
  __shared__ u32 ws[33];
  __shared__ u32 s_tile, s_base, s_rf, s_nr;
  const u32 m_hi = d_mk ? m_lo + *d_mk : m_hi_host;
  const u32 r_hi = d_r ? r_lo + *d_r : r_hi_host;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const u32 tile = s_tile;
  const u32 ntiles = (m_hi - m_lo + TILE - 1) / TILE;
  if (tile >= ntiles) {
    if (tile == 0 && threadIdx.x == 0) *d_U = 0;
    return;
  }
  const u32 t0 = m_lo + tile * TILE;
  const int n = (int)min((u32)TILE, m_hi - t0);
  if (threadIdx.x == 0) {
    const u32 rf = row_of_term(rstart, r_lo, r_hi, t0);
    const u32 rl = row_of_term(rstart, rf, r_hi, t0 + n - 1);
    s_rf = rf;
    s_nr = rl - rf + 1;
  }
  __syncthreads();
  const u32 rf = s_rf, nr = s_nr;
  if (nr <= (u32)SROWS) {
    // stage the tile's rows, then generate warp-striped (coalesced basis reads)
    for (u32 i = threadIdx.x; i <= nr; i += blockDim.x) srs[i] = rstart[rf + i];
    for (u32 i = threadIdx.x; i < nr; i += blockDim.x) {
      sbo[i] = boff[rb[rf + i]];
      sdel[i] = key_load<KW>(delta, rf + i);
    }
    __syncthreads();
    for (int i = threadIdx.x; i < n; i += blockDim.x) {
      const u32 t = t0 + i;
      u32 lo = 0, hi = nr;
      while (lo + 1 < hi) {
        const u32 mid = (lo + hi) >> 1;
        if (srs[mid] <= t) lo = mid; else hi = mid;
      }
      a[i] = key_add<KW>(key_load<KW>(bckey, (long long)sbo[lo] + (t - srs[lo])), sdel[lo]);
    }
  } else {
    const int my0 = threadIdx.x * ITEMS;
    const int cnt = max(0, min(ITEMS, n - my0));
    if (cnt > 0) {
      Key<KW> tmp[ITEMS];
      gen_keys<KW>(t0 + my0, cnt, r_lo, r_hi, rb, delta, rstart, boff, bckey, tmp, nullptr, nullptr);
#pragma unroll
      for (int i = 0; i < ITEMS; ++i)
        if (i < cnt) a[my0 + i] = tmp[i];
    }
  }
  __syncthreads();
  block_sort_keys<KW, ITEMS>(a, b, n, bits, wh, ws);
  u32 o = 0;
  for (int c0 = 0; c0 < n; c0 += blockDim.x) {
    const int i = c0 + threadIdx.x;
    const bool fl = i < n && (i == 0 || !key_eq<KW>(a[i], a[i - 1]));
    u32 tot;
    const u32 pre = block_scan_excl(fl ? 1u : 0u, ws, &tot);
    if (fl) b[o + pre] = a[i];
    o += tot;
  }
  if (threadIdx.x == 0) s_base = lookback_prefix(status, tile, o);
  __syncthreads();
  const u32 base = s_base;
  for (u32 i = threadIdx.x; i < o; i += blockDim.x) key_store<KW>(out, (long long)base + i, b[i]);
  if (threadIdx.x == 0 && tile == ntiles - 1) *d_U = base + o;
}

template <int KW>
__global__ void k_mark_leads(long long r, const int* __restrict__ rb, const u64* __restrict__ delta,
                             const u32* __restrict__ boff, const u64* __restrict__ bckey, const u64* __restrict__ dict,
                             const u32* __restrict__ d_N, uint8_t* __restrict__ done) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r) return;
  const u32 N = *d_N;
  const Key<KW> k = key_add<KW>(key_load<KW>(bckey, boff[rb[i]]), key_load<KW>(delta, i));
  const u32 pos = key_lower_bound<KW>(dict, N, k);
  if (pos < N && key_eq<KW>(key_load<KW>(dict, pos), k)) done[pos] = 1;
}

// frontier of round 1: dictionary entries not covered by a lead (look-back compaction)
template <int KW>
__global__ void __launch_bounds__(256) k_front0(const u64* __restrict__ dict, const uint8_t* __restrict__ done,
                                                const u32* __restrict__ d_N, u64* __restrict__ front, u32* status,
                                                u32* ticket, u32* d_nf) {
  constexpr int ITEMS = 8;
  __shared__ u32 ws[33];
  __shared__ u32 s_tile, s_base;
  const u32 N = *d_N;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const u32 tile = s_tile;
  const u32 ntiles = (N + 256 * ITEMS - 1) / (256 * ITEMS);
  if (tile >= ntiles) {
    if (tile == 0 && threadIdx.x == 0) *d_nf = 0;
    return;
  }
  const u32 base = tile * 256 * ITEMS + threadIdx.x * ITEMS;
  u32 keep = 0;
  for (int i = 0; i < ITEMS; ++i) keep += (base + i < N && !done[base + i]) ? 1u : 0u;
  u32 tot;
  const u32 pre = block_scan_excl(keep, ws, &tot);
  if (threadIdx.x == 0) s_base = lookback_prefix(status, tile, tot);
  __syncthreads();
  u32 o = s_base + pre;
  for (int i = 0; i < ITEMS; ++i)
    if (base + i < N && !done[base + i]) key_store<KW>(front, o++, key_load<KW>(dict, base + i));
  if (tile == ntiles - 1 && threadIdx.x == 0) *d_nf = s_base + tot;
}

// K4: first divisor in preference order, warp per frontier monomial.
template <int KW>
__global__ void k_closure_search(KeyFmt f, const u64* __restrict__ front, const u32* __restrict__ d_nf,
                                 const u32* lmw, const int* __restrict__ cidx, int nc, int nw,
                                 int* __restrict__ red) {
  // candidate LM table staged in shared memory when it fits (<= 48 KB)
  extern __shared__ __align__(16) u32 slm[];
  const bool staged = (long long)nc * nw * 4 <= 48 * 1024;
  if (staged) {
    for (int i = threadIdx.x; i < nc * nw; i += blockDim.x) slm[i] = __ldg(lmw + i);
    __syncthreads();
    lmw = slm;
  }
  const long long j = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (j >= *d_nf) return;
  u16 e[MAXV + 1];
  key_decode<KW>(f, key_load<KW>(front, j), e);
  e[f.n_vars] = 0;
  u32 me[MAXV / 2];
  for (int w = 0; w < nw; ++w) me[w] = (u32)e[2 * w] | ((u32)e[2 * w + 1] << 16);
  int found = -1;
  for (int base = 0; base < nc; base += 32) {
    const int c = base + lane;
    bool ok = c < nc;
    if (ok) {
      const u32* lm = lmw + (long long)c * nw;
      for (int w = 0; w < nw; ++w) ok &= (__vcmpgeu2(me[w], lm[w]) == 0xFFFFFFFFu);
    }
    const unsigned bm = __ballot_sync(0xffffffffu, ok);
    if (bm) {
      found = cidx[base + __ffs(bm) - 1];
      break;
    }
  }
  if (lane == 0) red[j] = found;
}

// K5: compaction of the rows found (ascending key(m)) + row offsets.
template <int KW>
__global__ void __launch_bounds__(256) k_new_rows(KeyFmt f, const u64* __restrict__ front, const int* __restrict__ red,
                                                  const u32* __restrict__ d_nf, long long row_base, long long cl_base,
                                                  u32 M_base, const u32* __restrict__ boff,
                                                  const u32* __restrict__ blen, const u64* __restrict__ bckey,
                                                  const u16* __restrict__ lmexp, const u16* __restrict__ maxe,
                                                  int round, int* __restrict__ rows_basis,
                                                  u64* __restrict__ rows_delta, u32* __restrict__ rows_start,
                                                  int* __restrict__ cl_basis, u16* __restrict__ cl_shift,
                                                  int* __restrict__ cl_round, u32* status_n, u32* status_len,
                                                  u32* ticket, u32* d_R, u32* d_Mk, u32* err) {
  __shared__ u32 ws[33];
  __shared__ u32 s_tile, s_base, s_lbase;
  const u32 nf = *d_nf;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const u32 tile = s_tile;
  const u32 ntiles = (nf + 255) / 256;
  if (tile >= ntiles) {
    if (tile == 0 && threadIdx.x == 0) {
      *d_R = 0;
      *d_Mk = 0;
    }
    return;
  }
  const u32 j = tile * 256 + threadIdx.x;
  const int g = j < nf ? red[j] : -1;
  const u32 len = g >= 0 ? blen[g] : 0u;
  u32 tot, ltot;
  const u32 pre = block_scan_excl(g >= 0 ? 1u : 0u, ws, &tot);
  const u32 lpre = block_scan_excl(len, ws, &ltot);
  if (threadIdx.x == 0) {
    s_base = lookback_prefix(status_n, tile, tot);
    s_lbase = lookback_prefix(status_len, tile, ltot);
  }
  __syncthreads();
  if (g >= 0) {
    const long long q = (long long)s_base + pre;
    const long long row = row_base + q;
    const Key<KW> m = key_load<KW>(front, j);
    rows_basis[row] = g;
    key_store<KW>(rows_delta, row, key_sub<KW>(m, key_load<KW>(bckey, boff[g])));
    rows_start[row] = M_base + s_lbase + lpre;
    u16 e[MAXV];
    key_decode<KW>(f, m, e);
    bool over = false;
    for (int v = 0; v < f.n_vars; ++v) {
      const u32 s = (u32)e[v] - (u32)lmexp[(long long)g * f.n_vars + v];
      over |= (s + (u32)maxe[(long long)g * f.n_vars + v]) > 0xFFFFu;
      cl_shift[(cl_base + q) * f.n_vars + v] = (u16)s;
    }
    if (over) atomicOr(err, (u32)DEVERR_LANE_OVERFLOW);
    cl_basis[cl_base + q] = g;
    cl_round[cl_base + q] = round;
  }
  if (tile == ntiles - 1 && threadIdx.x == 0) {
    *d_R = s_base + tot;
    *d_Mk = s_lbase + ltot;
    rows_start[row_base + s_base + tot] = M_base + s_lbase + ltot;
  }
}

// K3: merge two disjoint ascending sets by co-rank; nb read from the device.
template <int KW>
__global__ void k_merge_corank(const u64* __restrict__ a, u32 na, const u64* __restrict__ b,
                               const u32* __restrict__ d_nb, u64* __restrict__ out) {
  const u32 nb = *d_nb;
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < na) {
    const Key<KW> k = key_load<KW>(a, i);
    key_store<KW>(out, i + key_lower_bound<KW>(b, nb, k), k);
  } else if (i < (long long)na + nb) {
    const long long j = i - na;
    const Key<KW> k = key_load<KW>(b, j);
    key_store<KW>(out, j + key_lower_bound<KW>(a, na, k), k);
  }
}

// Final join: regenerate every key, binary-search the (shared-memory) dictionary.
template <int KW>
__global__ void __launch_bounds__(512) k_join_gen(u32 M, u32 r, const int* __restrict__ rb,
                                                  const u64* __restrict__ delta, const u32* __restrict__ rstart,
                                                  const u32* __restrict__ boff, const u64* __restrict__ bckey,
                                                  const u32* __restrict__ bcoeff, const u64* __restrict__ dict,
                                                  u32 N, int use_smem, u32* __restrict__ col, u32* __restrict__ val,
                                                  u32* err) {
  constexpr int ITEMS = 8;
  extern __shared__ __align__(16) u64 sdict[];
  const u64* table = dict;
  if (use_smem) {
    for (u32 i = threadIdx.x; i < N * KW; i += blockDim.x) sdict[i] = __ldg(dict + i);
    __syncthreads();
    table = sdict;
  }
  bool miss = false;
  for (long long t0 = ((long long)blockIdx.x * blockDim.x + threadIdx.x) * ITEMS; t0 < M;
       t0 += (long long)gridDim.x * blockDim.x * ITEMS) {
    const int cnt = (int)min((long long)ITEMS, M - t0);
    Key<KW> k[ITEMS];
    u32 v[ITEMS];
    gen_keys<KW>((u32)t0, cnt, 0, r, rb, delta, rstart, boff, bckey, k, bcoeff, v);
#pragma unroll
    for (int i = 0; i < ITEMS; ++i) {
      if (i < cnt) {
        u32 pos = key_lower_bound<KW>(table, N, k[i]);
        if (pos >= N || !key_eq<KW>(key_load_rw<KW>(table, pos), k[i])) {
          miss = true;
          pos = 0;
        }
        col[t0 + i] = N - 1 - pos;
        val[t0 + i] = v[i];
      }
    }
  }
  if (miss) atomicOr(err, (u32)DEVERR_MISSING_KEY);
}

template <int KW>
__global__ void k_dict_exps(KeyFmt f, const u64* __restrict__ dict, u32 N, u16* __restrict__ out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  u16 e[MAXV];
  key_decode<KW>(f, key_load<KW>(dict, i), e);
  for (int v = 0; v < f.n_vars; ++v) out[((long long)N - 1 - i) * f.n_vars + v] = e[v];
}

// ---------------------------------------------------------------------------
// host orchestration
// ---------------------------------------------------------------------------
static inline unsigned nblk(long long n, int t) { return (unsigned)std::max<long long>(1, (n + t - 1) / t); }

static int mon_cmp(const uint16_t* u, const uint16_t* v, int n, int order) {
  if (order != 2) {
    long du = 0, dv = 0;
    for (int i = 0; i < n; ++i) {
      du += u[i];
      dv += v[i];
    }
    if (du != dv) return du < dv ? -1 : 1;
  }
  if (order == 0) {
    for (int i = n - 1; i >= 0; --i)
      if (u[i] != v[i]) return u[i] < v[i] ? 1 : -1;
    return 0;
  }
  for (int i = 0; i < n; ++i)
    if (u[i] != v[i]) return u[i] < v[i] ? -1 : 1;
  return 0;
}

// Candidates in preference order (key(LM), index).  The whole basis order is
// kept sorted incrementally (sort the appended polynomials, merge), so a call
// costs O(#polys) instead of a comparison sort of the candidate set.
static std::vector<int32_t> preference_order(Ctx* c, const std::vector<int32_t>& cand) {
  Basis& B = c->basis;
  const int n = c->n_vars;
  auto less = [&](int32_t x, int32_t y) {
    const int sgn = mon_cmp(&B.h_lm[(size_t)x * n], &B.h_lm[(size_t)y * n], n, c->order);
    return sgn != 0 ? sgn < 0 : x < y;
  };
  if (B.lm_sorted < B.n_polys) {
    const size_t mid = B.lm_order.size();
    for (int k = B.lm_sorted; k < B.n_polys; ++k)
      if (B.h_len[k] >= 1) B.lm_order.push_back(k);
    std::sort(B.lm_order.begin() + mid, B.lm_order.end(), less);
    std::inplace_merge(B.lm_order.begin(), B.lm_order.begin() + mid, B.lm_order.end(), less);
    B.lm_sorted = B.n_polys;
  }
  std::vector<int32_t> out;
  out.reserve(cand.size());
  bool prefix = true;  // candidates == [0, k): the common case
  for (size_t i = 0; i < cand.size() && prefix; ++i) prefix = cand[i] == (int32_t)i;
  if (prefix) {
    const int32_t k = (int32_t)cand.size();
    for (int32_t x : B.lm_order)
      if (x < k) out.push_back(x);
  } else {
    std::vector<char> in((size_t)B.n_polys, 0);
    for (int32_t x : cand) in[(size_t)x] = 1;
    for (int32_t x : B.lm_order)
      if (in[(size_t)x]) out.push_back(x);
  }
  return out;
}

template <int KW>
static void encode_basis(Ctx* c, const KeyFmt& f) {
  Basis& B = c->basis;
  if (B.ckey_lane_bits != f.lane_bits || B.ckey_words != KW) {
    B.ckey_terms = 0;
    B.ckey_lane_bits = f.lane_bits;
    B.ckey_words = KW;
  }
  if (B.ckey_terms == B.n_terms) return;
  ensure_keep(c, B.ckey, (size_t)(B.n_terms + 1) * KW * sizeof(u64));
  const long long t0 = B.ckey_terms, t1 = B.n_terms;
  F4B_LAUNCH(c, k_encode_basis<KW>, nblk(t1 - t0, 256), 256, 0, f, B.exps.as<u16>(), t0, t1, B.ckey.as<u64>());
  B.ckey_terms = t1;
}

static void read_counters(Ctx* c, const DevCounters* dc, DevCounters* h) {
  check_cuda(cudaMemcpyAsync(c->h_stat, dc, sizeof(DevCounters), cudaMemcpyDeviceToHost, c->stream), "d2h counters");
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  memcpy(h, c->h_stat, sizeof(DevCounters));
}

// Look-back scratch of one round: [tickets | status regions], zeroed per round.
struct RoundScratch {
  u32* tile_st;
  u32* front_st;
  u32* rows_n_st;
  u32* rows_l_st;
  size_t words;
};

template <int KW>
static void compile_t(Ctx* c, const KeyFmt& f, long long r0, const int32_t* h_rb, const uint16_t* h_shift,
                      int closure, const std::vector<int32_t>& cand, long long dict_cap, f4b_plan* pl) {
  Basis& B = c->basis;
  const int n = c->n_vars;
  const int bits = f.lane_bits * f.n_lanes;
  c->launches = 0;
  cudaEvent_t ev0, ev1, ev2;
  check_cuda(cudaEventCreate(&ev0), "event");
  check_cuda(cudaEventCreate(&ev1), "event");
  check_cuda(cudaEventCreate(&ev2), "event");
  check_cuda(cudaEventRecord(ev0, c->stream), "event record");
  encode_basis<KW>(c, f);

  std::vector<uint32_t> h_start(r0 + 1);
  long long M = 0;
  for (long long i = 0; i < r0; ++i) {
    h_start[i] = (uint32_t)M;
    M += B.h_len[h_rb[i]];
  }
  h_start[r0] = (uint32_t)M;
  if (M >= (1ll << 30)) fail(F4B_ERR_SIZE_CAP, "batch has more than 2^30 terms");
  const u32 M0 = (u32)M;

  // counters + per-round look-back scratch
  DevCounters* dc = nullptr;
  RoundScratch rs{};
  auto reset_round = [&](u32 m_terms, u32 m_front) {
    const size_t a = m_terms / K1Cfg<KW>::TILE + 4, b = m_front / 2048 + 4, cc = m_front / 256 + 4;
    const size_t words = a + b + 2 * cc + 64;
    const size_t bytes = sizeof(DevCounters) + words * 4;
    if (bytes > c->errflag.cap) {
      ensure_keep(c, c->errflag, bytes);
    }
    dc = reinterpret_cast<DevCounters*>(c->errflag.p);
    u32* lb = reinterpret_cast<u32*>(dc + 1);
    rs.tile_st = lb;
    rs.front_st = lb + a;
    rs.rows_n_st = rs.front_st + b;
    rs.rows_l_st = rs.rows_n_st + cc;
    rs.words = words;
    check_cuda(cudaMemsetAsync(dc->tickets, 0, sizeof(dc->tickets), c->stream), "memset tickets");
    check_cuda(cudaMemsetAsync(lb, 0, words * 4, c->stream), "memset lb");
  };
  ensure(c, c->errflag, sizeof(DevCounters) + 4096);
  check_cuda(cudaMemsetAsync(c->errflag.p, 0, sizeof(DevCounters), c->stream), "memset counters");
  reset_round(M0, M0);

  // ---- round 0 ----------------------------------------------------------
  long long rcap = std::max<long long>(2 * r0 + 1024, 4096);
  ensure(c, c->rows_basis, rcap * sizeof(int));
  ensure(c, c->rows_delta, rcap * KW * sizeof(u64));
  ensure(c, c->rows_len, rcap * sizeof(u32));
  ensure(c, c->rows_start, (rcap + 1) * sizeof(u32));
  ensure(c, c->shift_in, (size_t)std::max<long long>(r0, 1) * n * sizeof(u16));
  check_cuda(cudaMemcpyAsync(c->rows_basis.p, h_rb, r0 * sizeof(int), cudaMemcpyHostToDevice, c->stream), "h2d rows");
  check_cuda(cudaMemcpyAsync(c->shift_in.p, h_shift, r0 * n * sizeof(u16), cudaMemcpyHostToDevice, c->stream), "h2d");
  check_cuda(cudaMemcpyAsync(c->rows_start.p, h_start.data(), (r0 + 1) * sizeof(u32), cudaMemcpyHostToDevice,
                             c->stream), "h2d starts");
  F4B_LAUNCH(c, k_rows0<KW>, nblk(r0, 256), 256, 0, f, r0, c->rows_basis.as<int>(), c->shift_in.as<u16>(),
             B.len.as<u32>(), c->rows_delta.as<u64>(), c->rows_len.as<u32>());
  static bool attr = false;
  if (!attr) {
    check_cuda(cudaFuncSetAttribute(k_tile_dict<KW>, cudaFuncAttributeMaxDynamicSharedMemorySize, (int)K1Cfg<KW>::SMEM),
               "attr");
    check_cuda(cudaFuncSetAttribute(k_join_gen<KW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024),
               "attr");
    attr = true;
  }
  // m_hi / r_hi either host-known (d_mk = d_r = nullptr) or device counters
  // with `m_bound` bounding m_hi - m_lo (grid upper bound, surplus tiles exit)
  auto tile_dict = [&](u32 m_lo, u32 m_hi, u32 m_bound, const u32* d_mk, u32 r_lo, u32 r_hi, const u32* d_r,
                       u64* out) {
    const u32 tiles = std::max<u32>(1, (m_bound + K1Cfg<KW>::TILE - 1) / K1Cfg<KW>::TILE);
    F4B_LAUNCH(c, k_tile_dict<KW>, tiles, K1_THREADS, K1Cfg<KW>::SMEM, m_lo, m_hi, d_mk, r_lo, r_hi, d_r,
               c->rows_basis.as<int>(), c->rows_delta.as<u64>(), c->rows_start.as<u32>(), B.off.as<u32>(),
               B.ckey.as<u64>(), bits, out, rs.tile_st, &dc->tickets[0], &dc->U);
  };
  ensure(c, c->uniq, (size_t)(M0 + 1) * KW * sizeof(u64));
  tile_dict(0, M0, M0, nullptr, 0, (u32)r0, nullptr, c->uniq.as<u64>());
  pl->sort_passes += (bits + 7) / 8;
  ensure(c, c->dict_a, (size_t)(M0 + 1) * KW * sizeof(u64));
  sort_unique(c, KW, c->uniq.as<u64>(), &dc->U, M0, bits, nullptr, nullptr, c->dict_a.as<u64>(), &dc->N);
  u64* dict = c->dict_a.as<u64>();
  long long r = r0, rounds = 0, n_cl = 0;
  DevCounters hc;
  long long N = 0;

  if (closure && M0 > 0) {
    // leads of the input rows are covered (symbolic.py:339); the rest is the frontier
    ensure(c, c->flags, (size_t)M0 + 16);
    ensure(c, c->front, (size_t)(M0 + 1) * KW * sizeof(u64));
    uint8_t* done = c->flags.as<uint8_t>();
    check_cuda(cudaMemsetAsync(done, 0, M0, c->stream), "memset done");
    F4B_LAUNCH(c, k_mark_leads<KW>, nblk(r0, 256), 256, 0, r0, c->rows_basis.as<int>(), c->rows_delta.as<u64>(),
               B.off.as<u32>(), B.ckey.as<u64>(), dict, &dc->N, done);
    F4B_LAUNCH(c, k_front0<KW>, nblk(M0, 2048), 256, 0, dict, done, &dc->N, c->front.as<u64>(), rs.front_st,
               &dc->tickets[1], &dc->nf);
    // candidate LMs in preference order (key(LM), index) (symbolic.py:228-235)
    std::vector<int32_t> pref(cand);
    std::stable_sort(pref.begin(), pref.end(), [&](int32_t x, int32_t y) {
      int s = mon_cmp(&B.h_lm[(size_t)x * n], &B.h_lm[(size_t)y * n], n, c->order);
      return s != 0 ? s < 0 : x < y;
    });
    const int nc = (int)pref.size();
    const int nw = (n + 1) / 2;
    std::vector<uint32_t> h_lmw((size_t)std::max(nc, 1) * nw, 0u);
    for (int q = 0; q < nc; ++q)
      for (int v = 0; v < n; ++v)
        h_lmw[(size_t)q * nw + v / 2] |= (uint32_t)B.h_lm[(size_t)pref[q] * n + v] << (16 * (v & 1));
    ensure(c, c->lmpref, h_lmw.size() * sizeof(u32));
    ensure(c, c->cand_idx, (size_t)std::max(nc, 1) * sizeof(int));
    check_cuda(cudaMemcpyAsync(c->lmpref.p, h_lmw.data(), h_lmw.size() * sizeof(u32), cudaMemcpyHostToDevice,
                               c->stream), "h2d lm");
    if (nc)
      check_cuda(cudaMemcpyAsync(c->cand_idx.p, pref.data(), nc * sizeof(int), cudaMemcpyHostToDevice, c->stream),
                 "h2d cand");
    read_counters(c, dc, &hc);
    N = hc.N;
    long long nf = hc.nf;
    long long clcap = std::max<long long>(N + 1024, 4096);
    ensure(c, c->cl_basis, clcap * sizeof(int));
    ensure(c, c->cl_shift, clcap * n * sizeof(u16));
    ensure(c, c->cl_round, clcap * sizeof(int));
    u32 Mcur = M0;
    long long maxlen = 1;
    for (int32_t k : pref) maxlen = std::max<long long>(maxlen, B.h_len[k]);

    // One host round trip per closure round: every kernel of the round reads
    // the sizes it needs (nf, R, Mk, U) from device counters; grids are
    // sized by upper bounds (new rows <= nf, terms <= nf * max length).
    while (nf > 0 && nc > 0) {
      const long long mk_bound = std::max<long long>(1, std::min<long long>(nf * maxlen, (1ll << 30) - Mcur));
      if (r + nf + 2 > rcap) {
        rcap = 2 * (r + nf + 2);
        ensure_keep(c, c->rows_basis, rcap * sizeof(int));
        ensure_keep(c, c->rows_delta, rcap * KW * sizeof(u64));
        ensure_keep(c, c->rows_len, rcap * sizeof(u32));
        ensure_keep(c, c->rows_start, (rcap + 1) * sizeof(u32));
      }
      if (n_cl + nf > clcap) {
        clcap = 2 * (n_cl + nf);
        ensure_keep(c, c->cl_basis, clcap * sizeof(int));
        ensure_keep(c, c->cl_shift, clcap * n * sizeof(u16));
        ensure_keep(c, c->cl_round, clcap * sizeof(int));
      }
      ensure(c, c->red, (size_t)nf * sizeof(int));
      reset_round((u32)mk_bound, (u32)nf);
      ensure(c, c->uniq, (size_t)(mk_bound + 1) * KW * sizeof(u64));
      ensure(c, c->front_new, (size_t)(mk_bound + 1) * KW * sizeof(u64));
      DBuf& cur = (dict == c->dict_a.as<u64>()) ? c->dict_a : c->dict_b;
      DBuf& oth = (dict == c->dict_a.as<u64>()) ? c->dict_b : c->dict_a;
      ensure(c, oth, (size_t)(N + mk_bound + 1) * KW * sizeof(u64));
      const size_t lm_smem = (size_t)nc * nw * 4 <= 48 * 1024 ? (size_t)nc * nw * 4 : 0;
      F4B_LAUNCH(c, k_closure_search<KW>, nblk(nf * 32, 256), 256, lm_smem, f, c->front.as<u64>(), &dc->nf,
                 c->lmpref.as<u32>(), c->cand_idx.as<int>(), nc, nw, c->red.as<int>());
      F4B_LAUNCH(c, k_new_rows<KW>, nblk(nf, 256), 256, 0, f, c->front.as<u64>(), c->red.as<int>(), &dc->nf, r, n_cl,
                 Mcur, B.off.as<u32>(), B.len.as<u32>(), B.ckey.as<u64>(), B.lmexp.as<u16>(), B.maxe.as<u16>(),
                 (int)rounds + 1, c->rows_basis.as<int>(), c->rows_delta.as<u64>(), c->rows_start.as<u32>(),
                 c->cl_basis.as<int>(), c->cl_shift.as<u16>(), c->cl_round.as<int>(), rs.rows_n_st, rs.rows_l_st,
                 &dc->tickets[2], &dc->R, &dc->Mk, &dc->err);
      // fill + dictionary of the new rows; keys absent from the dictionary -> next frontier
      tile_dict(Mcur, 0, (u32)mk_bound, &dc->Mk, (u32)r, 0, &dc->R, c->uniq.as<u64>());
      c->h_stat[512] = (u32)N;
      check_cuda(cudaMemcpyAsync(&dc->ndict, &c->h_stat[512], 4, cudaMemcpyHostToDevice, c->stream), "h2d N");
      sort_unique(c, KW, c->uniq.as<u64>(), &dc->U, (u32)mk_bound, bits, dict, &dc->ndict, c->front_new.as<u64>(),
                  &dc->nf);
      // merged dictionary (symbolic.py:281-290); the new keys are the next frontier
      F4B_LAUNCH(c, k_merge_corank<KW>, nblk(N + mk_bound, 256), 256, 0, cur.as<u64>(), (u32)N,
                 c->front_new.as<u64>(), &dc->nf, oth.as<u64>());
      read_counters(c, dc, &hc);
      const long long R = hc.R, Mk = hc.Mk;
      if (R == 0) break;
      if ((long long)Mcur + Mk >= (1ll << 30)) fail(F4B_ERR_SIZE_CAP, "batch has more than 2^30 terms");
      ++rounds;
      pl->sort_passes += (bits + 7) / 8;
      std::swap(c->front, c->front_new);
      nf = hc.nf;
      dict = oth.as<u64>();
      N += nf;
      M += Mk;
      Mcur += (u32)Mk;
      r += R;
      n_cl += R;
      if (N > dict_cap)
        fail(F4B_ERR_SIZE_CAP, "dictionary exceeded the cap after " + std::to_string(rounds) + " closure rounds");
    }
  } else {
    read_counters(c, dc, &hc);
    N = hc.N;
  }
  check_cuda(cudaEventRecord(ev1, c->stream), "event record");

  // ---- row assembly ------------------------------------------------------
  pl->KW = KW;
  pl->lane_bits = f.lane_bits;
  pl->r = r;
  pl->r0 = r0;
  pl->N = N;
  pl->M = M;
  pl->closure_rounds = rounds;
  ensure(c, pl->row_ptr, (size_t)(r + 1) * sizeof(u32));
  ensure(c, pl->col_ind, (size_t)std::max<long long>(M, 1) * sizeof(u32));
  ensure(c, pl->val, (size_t)std::max<long long>(M, 1) * sizeof(u32));
  ensure(c, pl->dict, (size_t)std::max<long long>(N, 1) * KW * sizeof(u64));
  ensure(c, pl->dict_exps, (size_t)std::max<long long>(N, 1) * n * sizeof(u16));
  ensure(c, pl->cl_basis, (size_t)std::max<long long>(n_cl, 1) * sizeof(int));
  ensure(c, pl->cl_shift, (size_t)std::max<long long>(n_cl, 1) * n * sizeof(u16));
  ensure(c, pl->cl_round, (size_t)std::max<long long>(n_cl, 1) * sizeof(int));
  check_cuda(cudaMemcpyAsync(pl->row_ptr.p, c->rows_start.p, (r + 1) * sizeof(u32), cudaMemcpyDeviceToDevice,
                             c->stream), "d2d row_ptr");
  if (N)
    check_cuda(cudaMemcpyAsync(pl->dict.p, dict, N * KW * sizeof(u64), cudaMemcpyDeviceToDevice, c->stream), "d2d");
  if (n_cl) {
    check_cuda(cudaMemcpyAsync(pl->cl_basis.p, c->cl_basis.p, n_cl * sizeof(int), cudaMemcpyDeviceToDevice, c->stream),
               "d2d");
    check_cuda(cudaMemcpyAsync(pl->cl_shift.p, c->cl_shift.p, n_cl * n * sizeof(u16), cudaMemcpyDeviceToDevice,
                               c->stream), "d2d");
    check_cuda(cudaMemcpyAsync(pl->cl_round.p, c->cl_round.p, n_cl * sizeof(int), cudaMemcpyDeviceToDevice, c->stream),
               "d2d");
  }
  if (M) {
    size_t smem = (size_t)N * KW * sizeof(u64);
    const int use_smem = smem <= 200 * 1024 ? 1 : 0;
    if (!use_smem) smem = 0;
    const int per_sm = use_smem ? (int)std::max<size_t>(1, std::min<size_t>(4, (220 * 1024) / (smem + 8 * 1024))) : 4;
    const int blocks = (int)std::min<long long>(nblk(M, 512 * 8), (long long)c->num_sms * per_sm);
    F4B_LAUNCH(c, k_join_gen<KW>, blocks, 512, smem, (u32)M, (u32)r, c->rows_basis.as<int>(),
               c->rows_delta.as<u64>(), c->rows_start.as<u32>(), B.off.as<u32>(), B.ckey.as<u64>(),
               B.coeff.as<u32>(), pl->dict.as<u64>(), (u32)N, use_smem, pl->col_ind.as<u32>(), pl->val.as<u32>(),
               &dc->err);
  }
  if (N) F4B_LAUNCH(c, k_dict_exps<KW>, nblk(N, 256), 256, 0, f, pl->dict.as<u64>(), (u32)N, pl->dict_exps.as<u16>());
  check_cuda(cudaEventRecord(ev2, c->stream), "event record");
  read_counters(c, dc, &hc);
  float ms1 = 0, ms2 = 0;
  check_cuda(cudaEventElapsedTime(&ms1, ev0, ev1), "elapsed");
  check_cuda(cudaEventElapsedTime(&ms2, ev1, ev2), "elapsed");
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  cudaEventDestroy(ev2);
  pl->dict_ns = (int64_t)(ms1 * 1e6);
  pl->asm_ns = (int64_t)(ms2 * 1e6);
  pl->launches = c->launches;
  if (hc.err & DEVERR_LANE_OVERFLOW) fail(F4B_ERR_LANE_OVERFLOW, "shifted exponent overflows a 16-bit lane");
  if (hc.err & DEVERR_MISSING_KEY) fail(F4B_ERR_MISSING_KEY, "row key absent from dictionary (closure defect)");
}

// ===========================================================================
// Rank-bitmap dictionary (grevlex fast path)
// ---------------------------------------------------------------------------
// A counting sort over the dense monomial rank space: for grevlex and batch
// degree <= D every monomial m has a combinatorial rank
//   rank(m) = C(n+d-1, n) + sum_{i=n-1..1} [s_i > e_i] C(s_i - e_i - 1 + i, i),
//   d = deg m, s_{n-1} = d, s_{i-1} = s_i - e_i,
// that is order-isomorphic to the term order on [0, C(n+D, n)).  The
// dictionary is then a STATIC presence bitmap over that range (idempotent
// ORs into a preallocated array — no dynamic insertion, no hashing, fully
// deterministic), unique is the bitmap itself, the ascending dictionary is the
// set bits in rank order, and the column map is a popcount prefix:
//   col(m) = N - 1 - (prefix[rank >> 5] + popc(word & below(rank))).
// The radix-sort path above stays for lex / deglex and huge rank spaces.
// ===========================================================================
static constexpr int RK_THREADS = 256;
static constexpr int RK_TILE = 4096;
static constexpr int RK_SROWS = 1024;

// Fill: every term of rows [r_lo, r_hi) -> its rank -> one bit.  Private
// shared-memory bitmaps per CTA (written out as partials) when the rank space
// fits, otherwise atomicOr straight into one global bitmap.  Closure rounds
// pass `known` (the dictionary so far): only absent monomials are ORed into
// the global new-bits map, so a round costs O(Mk) instead of O(grid * words).
template <int KW>
__global__ void __launch_bounds__(RK_THREADS) k_rank_fill(
    KeyFmt f, u32 m_lo, u32 m_hi_host, const u32* __restrict__ d_mk, u32 r_lo, u32 r_hi_host,
    const u32* __restrict__ d_r, const int* __restrict__ rb, const u64* __restrict__ delta,
    const u32* __restrict__ rstart, const u32* __restrict__ boff, const u64* __restrict__ bckey,
    const u32* __restrict__ bt_g, int st, int bt_words, u32 words, int use_smem, u32* __restrict__ partial,
    const u32* __restrict__ known) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Key<KW>* sdel = reinterpret_cast<Key<KW>*>(smraw);
  u32* srs = reinterpret_cast<u32*>(sdel + RK_SROWS);
  u32* sbo = srs + RK_SROWS + 1;
  u32* bt = sbo + RK_SROWS;
  u32* sbits = bt + bt_words;
  __shared__ u32 s_rf, s_nr;
  const u32 m_hi = d_mk ? m_lo + *d_mk : m_hi_host;
  const u32 r_hi = d_r ? r_lo + *d_r : r_hi_host;
  for (int i = threadIdx.x; i < bt_words; i += blockDim.x) bt[i] = bt_g[i];
  u32* bits = partial;
  if (use_smem) {
    for (u32 w = threadIdx.x; w < words; w += blockDim.x) sbits[w] = 0;
    bits = sbits;
  }
  __syncthreads();
  const u32 ntiles = (m_hi - m_lo + RK_TILE - 1) / RK_TILE;
  for (u32 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const u32 t0 = m_lo + tile * RK_TILE;
    const u32 n = min((u32)RK_TILE, m_hi - t0);
    if (threadIdx.x == 0) {
      const u32 rf = row_of_term(rstart, r_lo, r_hi, t0);
      s_rf = rf;
      s_nr = row_of_term(rstart, rf, r_hi, t0 + n - 1) - rf + 1;
    }
    __syncthreads();
    const u32 rf = s_rf, nr = s_nr;
    if (nr <= (u32)RK_SROWS) {
      for (u32 i = threadIdx.x; i <= nr; i += blockDim.x) srs[i] = rstart[rf + i];
      for (u32 i = threadIdx.x; i < nr; i += blockDim.x) {
        sbo[i] = boff[rb[rf + i]];
        sdel[i] = key_load<KW>(delta, rf + i);
      }
      __syncthreads();
      for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
        const u32 t = t0 + i;
        u32 lo = 0, hi = nr;
        while (lo + 1 < hi) {
          const u32 mid = (lo + hi) >> 1;
          if (srs[mid] <= t) lo = mid; else hi = mid;
        }
        const Key<KW> k = key_add<KW>(key_load<KW>(bckey, (long long)sbo[lo] + (t - srs[lo])), sdel[lo]);
        const u32 rk = key_rank<KW>(f, bt, st, k);
        if (!known || !((__ldg(known + (rk >> 5)) >> (rk & 31)) & 1u)) atomicOr(bits + (rk >> 5), 1u << (rk & 31));
      }
    } else {
      for (u32 i = threadIdx.x * 8; i < n; i += blockDim.x * 8) {
        Key<KW> k[8];
        const int cnt = (int)min(8u, n - i);
        gen_keys<KW>(t0 + i, cnt, r_lo, r_hi, rb, delta, rstart, boff, bckey, k, nullptr, nullptr);
        for (int q = 0; q < cnt; ++q) {
          const u32 rk = key_rank<KW>(f, bt, st, k[q]);
          if (!known || !((__ldg(known + (rk >> 5)) >> (rk & 31)) & 1u)) atomicOr(bits + (rk >> 5), 1u << (rk & 31));
        }
      }
    }
    __syncthreads();
  }
  // merge the private map: OR only words that add bits (most are already in)
  if (use_smem)
    for (u32 w = threadIdx.x; w < words; w += blockDim.x) {
      const u32 v = sbits[w];
      if (v && (v & ~__ldcg(partial + w))) atomicOr(partial + w, v);
    }
}

// OR the partial bitmaps.  mode 0: dict = OR.  mode 1: newbits = OR & ~dict,
// dict |= OR.  Adds the popcount of the result (dict / newbits) to *d_count.
__global__ void __launch_bounds__(256) k_rank_reduce(const u32* __restrict__ partial, int nparts, u32 words, int mode,
                                                     u32* __restrict__ dict, u32* __restrict__ newbits,
                                                     u32* d_count) {
  __shared__ u32 ws[33];
  const u32 w = blockIdx.x * blockDim.x + threadIdx.x;
  u32 cnt = 0;
  if (w < words) {
    u32 v = 0;
    for (int p = 0; p < nparts; ++p) v |= partial[(size_t)p * words + w];
    if (mode == 0) {
      dict[w] = v;
      cnt = __popc(v);
    } else {
      const u32 old = dict[w];
      const u32 nw = v & ~old;
      newbits[w] = nw;
      dict[w] = old | v;
      cnt = __popc(nw);
    }
  }
  u32 tot;
  block_scan_excl(cnt, ws, &tot);
  if (threadIdx.x == 0 && tot) atomicAdd(d_count, tot);
}

template <int KW>
__global__ void k_rank_leads(KeyFmt f, long long r, const int* __restrict__ rb, const u64* __restrict__ delta,
                             const u32* __restrict__ boff, const u64* __restrict__ bckey, const u32* __restrict__ bt,
                             int st, u32* __restrict__ done) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r) return;
  const Key<KW> k = key_add<KW>(key_load<KW>(bckey, boff[rb[i]]), key_load<KW>(delta, i));
  const u32 rk = key_rank<KW>(f, bt, st, k);
  atomicOr(done + (rk >> 5), 1u << (rk & 31));
}

// Set bits of (A & ~B) in ascending rank order (look-back compaction).
// mode 0 (frontier): out_keys[pos] = device key of the monomial.
// mode 1 (final dictionary): out_keys ascending, out_exps[(N-1-pos)] (column
//   order), wprefix[w] = number of set bits before word w.
template <int KW>
__global__ void __launch_bounds__(256) k_rank_extract(KeyFmt f, const u32* __restrict__ A, const u32* __restrict__ B,
                                                      u32 words, int mode, const u32* __restrict__ bt_g, int st,
                                                      int bt_words, u32* __restrict__ ranks,
                                                      u32* __restrict__ wprefix, u32* status, u32* ticket,
                                                      u32* d_count) {
  constexpr int WPT = 4;  // words per thread
  extern __shared__ u32 bt[];
  __shared__ u32 ws[33];
  __shared__ u32 s_tile, s_base;
  for (int i = threadIdx.x; i < bt_words; i += blockDim.x) bt[i] = bt_g[i];
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const u32 tile = s_tile;
  const u32 ntiles = (words + 256 * WPT - 1) / (256 * WPT);
  if (tile >= ntiles) {
    if (tile == 0 && threadIdx.x == 0) *d_count = 0;
    return;
  }
  const u32 w0 = tile * 256 * WPT + threadIdx.x * WPT;
  u32 v[WPT];
  u32 cnt = 0;
#pragma unroll
  for (int q = 0; q < WPT; ++q) {
    const u32 w = w0 + q;
    v[q] = w < words ? (A[w] & (B ? ~B[w] : 0xFFFFFFFFu)) : 0u;
    cnt += __popc(v[q]);
  }
  u32 tot;
  const u32 pre = block_scan_excl(cnt, ws, &tot);
  if (threadIdx.x == 0) s_base = lookback_prefix(status, tile, tot);
  __syncthreads();
  u32 pos = s_base + pre;
#pragma unroll
  for (int q = 0; q < WPT; ++q) {
    const u32 w = w0 + q;
    if (mode == 1 && w < words) wprefix[w] = pos;
    u32 m = v[q];
    while (m) {
      const int bit = __ffs(m) - 1;
      m &= m - 1;
      ranks[pos++] = w * 32 + bit;
    }
  }
  if (tile == ntiles - 1 && threadIdx.x == 0) *d_count = s_base + tot;
}

// ranks -> device keys (and, for the final dictionary, exponents in column
// order).  Grid-stride over the device-side count.
template <int KW>
__global__ void __launch_bounds__(256) k_rank_unrank(KeyFmt f, const u32* __restrict__ ranks,
                                                     const u32* __restrict__ d_count, const u32* __restrict__ bt_g,
                                                     int st, int bt_words, int D, u64* __restrict__ out_keys,
                                                     u16* __restrict__ out_exps) {
  extern __shared__ u32 bts[];
  for (int i = threadIdx.x; i < bt_words; i += blockDim.x) bts[i] = bt_g[i];
  __syncthreads();
  const u32 cnt = *d_count;
  const int n = f.n_vars;
  for (u32 j = blockIdx.x * blockDim.x + threadIdx.x; j < cnt; j += gridDim.x * blockDim.x) {
    u16 e[MAXV];
    unrank_exps(ranks[j], n, D, bts, st, e);
    key_store<KW>(out_keys, j, key_encode<KW>(f, e));
    if (out_exps)
      for (int x = 0; x < n; ++x) out_exps[((long long)cnt - 1 - j) * n + x] = e[x];
  }
}

// Fused round tail: OR the fill partials (mode 0: dict = OR, frontier = dict &
// ~done; mode 1: frontier = OR & ~dict, dict |= OR), then emit the frontier
// monomials in ascending rank order (look-back over word tiles) as device
// keys, unranked cooperatively by the whole CTA.  Replaces reduce + extract +
// unrank (three launches) per round.
static constexpr int RX_WPT = 1;
static constexpr int RX_LIST = 4096;
template <int KW>
__global__ void __launch_bounds__(256) k_rank_round(KeyFmt f, const u32* __restrict__ partial, int nparts, u32 words,
                                                    int mode, u32* __restrict__ dict, const u32* __restrict__ done,
                                                    const u32* __restrict__ bt_g, int st, int bt_words, int D,
                                                    u64* __restrict__ front, u32* status, u32* ticket, u32* d_nf,
                                                    u32* d_ndict) {
  extern __shared__ __align__(16) u32 rsm[];
  u32* bt = rsm;
  u32* list = rsm + bt_words;
  __shared__ u32 ws[33];
  __shared__ u32 s_tile, s_base;
  for (int i = threadIdx.x; i < bt_words; i += blockDim.x) bt[i] = bt_g[i];
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const u32 tile = s_tile;
  const u32 ntiles = (words + 256 * RX_WPT - 1) / (256 * RX_WPT);
  if (tile >= ntiles) return;
  const u32 w0 = tile * 256 * RX_WPT + threadIdx.x * RX_WPT;
  u32 x[RX_WPT];
  u32 cnt = 0, dcnt = 0;
#pragma unroll
  for (int q = 0; q < RX_WPT; ++q) {
    const u32 w = w0 + q;
    x[q] = 0;
    if (w < words) {
      u32 v = 0;
      for (int pp = 0; pp < nparts; ++pp) v |= partial[(size_t)pp * words + w];
      if (mode == 0) {
        dict[w] = v;
        dcnt += __popc(v);
        x[q] = v & ~done[w];
      } else {
        const u32 old = dict[w];
        x[q] = v & ~old;
        dict[w] = old | v;
        dcnt += __popc(x[q]);
      }
      cnt += __popc(x[q]);
    }
  }
  u32 tot, dtot;
  const u32 pre = block_scan_excl(cnt, ws, &tot);
  block_scan_excl(dcnt, ws, &dtot);
  if (threadIdx.x == 0) {
    s_base = lookback_prefix(status, tile, tot);
    if (dtot) atomicAdd(d_ndict, dtot);
  }
  __syncthreads();
  const u32 base = s_base;
  // unrank the tile's frontier monomials: ranks staged in shared memory
  for (u32 done_cnt = 0; done_cnt < tot; done_cnt += RX_LIST) {
    u32 p = pre;
#pragma unroll
    for (int q = 0; q < RX_WPT; ++q) {
      u32 m = x[q];
      while (m) {
        const int bit = __ffs(m) - 1;
        m &= m - 1;
        if (p >= done_cnt && p < done_cnt + RX_LIST) list[p - done_cnt] = (w0 + q) * 32 + bit;
        ++p;
      }
    }
    __syncthreads();
    const u32 chunk = min((u32)RX_LIST, tot - done_cnt);
    for (u32 j = threadIdx.x; j < chunk; j += blockDim.x) {
      u16 e[MAXV];
      unrank_exps(list[j], f.n_vars, D, bt, st, e);
      key_store<KW>(front, (long long)base + done_cnt + j, key_encode<KW>(f, e));
    }
    __syncthreads();
  }
  if (tile == ntiles - 1 && threadIdx.x == 0) *d_nf = base + tot;
}

// Fused closure round: first LM divisor per frontier monomial (warp per
// monomial, SWAR u16x2 over the shared-memory LM table) and compaction of the
// reducer rows in ascending key(m) with their row offsets (two look-backs).
static constexpr int CR_TILE = 64;
template <int KW>
__global__ void __launch_bounds__(256) k_closure_rows(KeyFmt f, const u64* __restrict__ front,
                                                      const u32* __restrict__ d_nf, const u32* lmw_g,
                                                      const int* __restrict__ cidx, int nc, int nw, int stage_lm,
                                                      long long row_base, long long cl_base, u32 M_base,
                                                      const u32* __restrict__ boff, const u32* __restrict__ blen,
                                                      const u64* __restrict__ bckey, const u16* __restrict__ lmexp,
                                                      const u16* __restrict__ maxe, int round,
                                                      int* __restrict__ rows_basis, u64* __restrict__ rows_delta,
                                                      u32* __restrict__ rows_start, int* __restrict__ cl_basis,
                                                      u16* __restrict__ cl_shift, int* __restrict__ cl_round,
                                                      u32* status_n, u32* status_len, u32* ticket, u32* d_R, u32* d_Mk,
                                                      u32* err) {
  extern __shared__ __align__(16) u32 slm[];
  __shared__ int sred[CR_TILE];
  __shared__ u32 ws[33];
  __shared__ u32 s_tile, s_base, s_lbase;
  const u32* lmw = lmw_g;
  if (stage_lm) {
    for (int i = threadIdx.x; i < nc * nw; i += blockDim.x) slm[i] = __ldg(lmw_g + i);
    lmw = slm;
  }
  const u32 nf = *d_nf;
  if (threadIdx.x == 0) s_tile = atomicAdd(ticket, 1u);
  __syncthreads();
  const u32 tile = s_tile;
  const u32 ntiles = (nf + CR_TILE - 1) / CR_TILE;
  if (tile >= ntiles) {
    if (tile == 0 && threadIdx.x == 0) {
      *d_R = 0;
      *d_Mk = 0;
    }
    return;
  }
  const int lane = threadIdx.x & 31, warp = threadIdx.x >> 5;
  for (int t = warp; t < CR_TILE; t += 8) {
    const u32 j = tile * CR_TILE + t;
    int found = -1;
    if (j < nf) {
      u16 e[MAXV + 1];
      key_decode<KW>(f, key_load<KW>(front, j), e);
      e[f.n_vars] = 0;
      u32 me[MAXV / 2];
      for (int w = 0; w < nw; ++w) me[w] = (u32)e[2 * w] | ((u32)e[2 * w + 1] << 16);
      for (int b0 = 0; b0 < nc; b0 += 32) {
        const int cc = b0 + lane;
        bool ok = cc < nc;
        if (ok) {
          const u32* lm = lmw + (long long)cc * nw;
          for (int w = 0; w < nw; ++w) ok &= (__vcmpgeu2(me[w], lm[w]) == 0xFFFFFFFFu);
        }
        const unsigned bm = __ballot_sync(0xffffffffu, ok);
        if (bm) {
          found = cidx[b0 + __ffs(bm) - 1];
          break;
        }
      }
    }
    if (lane == 0) sred[t] = found;
  }
  __syncthreads();
  const int t = threadIdx.x;
  const u32 j = tile * CR_TILE + t;
  const int g = (t < CR_TILE && j < nf) ? sred[t] : -1;
  const u32 len = g >= 0 ? blen[g] : 0u;
  u32 tot, ltot;
  const u32 pre = block_scan_excl(g >= 0 ? 1u : 0u, ws, &tot);
  const u32 lpre = block_scan_excl(len, ws, &ltot);
  if (threadIdx.x == 0) {
    s_base = lookback_prefix(status_n, tile, tot);
    s_lbase = lookback_prefix(status_len, tile, ltot);
  }
  __syncthreads();
  if (g >= 0) {
    const long long q = (long long)s_base + pre;
    const long long row = row_base + q;
    const Key<KW> m = key_load<KW>(front, j);
    rows_basis[row] = g;
    key_store<KW>(rows_delta, row, key_sub<KW>(m, key_load<KW>(bckey, boff[g])));
    rows_start[row] = M_base + s_lbase + lpre;
    u16 e[MAXV];
    key_decode<KW>(f, m, e);
    bool over = false;
    for (int v = 0; v < f.n_vars; ++v) {
      const u32 s = (u32)e[v] - (u32)lmexp[(long long)g * f.n_vars + v];
      over |= (s + (u32)maxe[(long long)g * f.n_vars + v]) > 0xFFFFu;
      cl_shift[(cl_base + q) * f.n_vars + v] = (u16)s;
    }
    if (over) atomicOr(err, (u32)DEVERR_LANE_OVERFLOW);
    cl_basis[cl_base + q] = g;
    cl_round[cl_base + q] = round;
  }
  if (tile == ntiles - 1 && threadIdx.x == 0) {
    *d_R = s_base + tot;
    *d_Mk = s_lbase + ltot;
    rows_start[row_base + s_base + tot] = M_base + s_lbase + ltot;
  }
}

// ---------------------------------------------------------------------------
// Persistent closure loop (cooperative launch): every closure round of
// symbolic.py:250-290 in ONE kernel, grid barriers between the phases, no
// host round trip per round.  Per round:
//   A  reducer search, warp per frontier monomial; per-tile (rows, terms)
//      counts                                                   | grid.sync
//   B  totals + tile bases (every CTA scans the tile counts), rows written
//      in frontier order, and their terms ranked straight away by the CTA
//      that wrote them: absent monomials ORed into `newbits`    | grid.sync
//   D1 per-CTA word chunk popcounts                             | grid.sync
//   D2 chunk bases; set bits -> next frontier (ascending rank = ascending
//      key), dict |= newbits, newbits = 0                       | grid.sync
// Every CTA derives the same loop state (R, Mk, nf) from the same global
// counts, so all exits are grid-uniform.  Capacity overflows stop the loop
// with a flag; the host grows the buffers and recompiles.
// ---------------------------------------------------------------------------
struct LoopOut {
  u32 r, n_cl, M, N, rounds, nf, flags, sel;
  unsigned long long t_start, t_epi, t_end;  // %globaltimer (fused kernel)
};
enum : u32 { LOOP_OVERFLOW = 1u, LOOP_SIZE_CAP = 2u, LOOP_DICT_CAP = 4u };

struct LoopArgs {
  KeyFmt f;
  int D, st, bt_words;
  u32 words;
  const u32* bt;
  u32* dict;
  u32* newbits;
  u64* front0;
  u64* front1;
  u32 front_cap;
  int* red;
  u32* tilecnt;
  u32* chunkcnt;
  const u32* lmw;
  const int* cidx;
  int nc, nw, stage_lm;
  const u32* boff;
  const u32* blen;
  const u64* bckey;
  const u16* lmexp;
  const u16* maxe;
  int* rows_basis;
  u64* rows_delta;
  u32* rows_start;
  long long rows_cap;
  int* cl_basis;
  u16* cl_shift;
  int* cl_round;
  long long cl_cap;
  long long r0;
  u32 M0, maxlen;
  long long dict_cap;
  const u32* d_nf0;
  const u32* d_N0;
  u32* err;
  LoopOut* out;
  unsigned long long* trace;  // optional: [round][5] %globaltimer stamps + nf (F4B_LOOP_TRACE)
  // full pipeline (compile_rank_fused): round 0 before the loop, the final
  // dictionary and the join after it
  int full, closure;
  const int* rb_in;
  const u32* start_in;
  const u16* shift_in;
  const u32* bcoeff;
  u32* done;
  u64* dict_out;
  u16* dict_exps;
  uint2* dwp;
  u32* col;
  u32* val;
  u32 N_cap, M_cap;
};

F4B_DEV unsigned long long gtimer() {
  unsigned long long t;
  asm volatile("mov.u64 %0, %globaltimer;" : "=l"(t));
  return t;
}

static constexpr int CL_THREADS = 256;
// k_fbsp: 512 threads, one CTA per SM slot pair (256: 3.08e9, 512: 3.11e9 nnz/s)
static constexpr int FB_THREADS = 512;
static constexpr int CL_LIST = 2048;

F4B_DEV u32 block_sum_u32(u32 v, u32* ws) {
  u32 tot;
  block_scan_excl(v, ws, &tot);
  return tot;
}

template <int KW>
__global__ void __launch_bounds__(CL_THREADS) k_closure_loop(const LoopArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) u32 csm[];
  u32* bt = csm;
  u32* list = csm + a.bt_words;             // CL_LIST ranks (D2)
  u32* slm = list + CL_LIST;                // LM table (optional)
  __shared__ u32 ws[33];
  __shared__ u32 s_wn[CL_THREADS / 32], s_wl[CL_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NWARP = CL_THREADS / 32;
  const int n = a.f.n_vars;
  for (int i = tid; i < a.bt_words; i += blockDim.x) bt[i] = a.bt[i];
  const u32* lmw = a.lmw;
  if (a.stage_lm) {
    for (int i = tid; i < a.nc * a.nw; i += blockDim.x) slm[i] = __ldg(a.lmw + i);
    lmw = slm;
  }
  __syncthreads();
  u32 nf = a.full ? 0u : __ldcg(a.d_nf0), N = a.full ? 0u : __ldcg(a.d_N0);
  long long r = a.r0, n_cl = 0;
  u32 Mcur = a.M0, rounds = 0, flags = 0;
  int sel = 0;
  const u32 G = gridDim.x, W = G * NWARP, gw = blockIdx.x * NWARP + warp;
  const u32 CH = (a.maxlen + 31) / 32;  // 32-term chunks per row (upper bound)
  const u32 cw = (((a.words + G - 1) / G) + 31) & ~31u;
  const u32 w_lo = min(a.words, blockIdx.x * cw), w_hi = min(a.words, w_lo + cw);
  // emit the set bits of x(w) over this CTA's word chunk, ascending, from
  // position `base`: keys to out_keys[pos]; with out_exps also exponents to
  // out_exps[N_all - 1 - pos] (column order) and the word prefix to dwp
  auto emit_chunk = [&](auto getx, u32 base, u64* out_keys, u16* out_exps, u32 N_all) {
    for (u32 w0 = w_lo; w0 < w_hi; w0 += blockDim.x) {
      const u32 w = w0 + tid;
      const u32 x = w < w_hi ? getx(w) : 0u;
      u32 tt;
      const u32 pre = block_scan_excl(__popc(x), ws, &tt);
      if (out_exps && w < w_hi) a.dwp[w] = make_uint2(x, base + pre);
      auto put = [&](u32 pos, u32 rk) {
        u16 e[MAXV];
        unrank_exps(rk, n, a.D, bt, a.st, e);
        key_store<KW>(out_keys, pos, key_encode<KW>(a.f, e));
        if (out_exps)
          for (int v = 0; v < n; ++v) out_exps[((long long)N_all - 1 - pos) * n + v] = e[v];
      };
      if (tt <= (u32)CL_LIST) {
        u32 p = pre, m = x;
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          list[p++] = w * 32 + b;
        }
        __syncthreads();
        for (u32 q = tid; q < tt; q += blockDim.x) put(base + q, list[q]);
        __syncthreads();
      } else {
        u32 p = base + pre, m = x;
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          put(p++, w * 32 + b);
        }
      }
      base += tt;
    }
  };
  // exclusive base of this CTA and the grand total of per-CTA counts cnt[0, G)
  auto chunk_bases = [&](const u32* cnt, u32& base, u32& total) {
    u32 sb = 0, st = 0;
    for (u32 b = tid; b < G; b += blockDim.x) {
      const u32 v = __ldcg(cnt + b);
      st += v;
      if (b < blockIdx.x) sb += v;
    }
    base = block_sum_u32(sb, ws);
    total = block_sum_u32(st, ws);
  };
  unsigned long long t_start = 0, t_epi = 0;
  if (blockIdx.x == 0 && tid == 0) t_start = gtimer();
  if (a.full) {
    const long long gt = (long long)blockIdx.x * blockDim.x + tid, GT = (long long)G * blockDim.x;
    // P0: clear the maps; shift deltas key(t) - key(1) of the input rows
    for (long long w = gt; w < a.words; w += GT) {
      a.dict[w] = 0;
      a.done[w] = 0;
      a.newbits[w] = 0;
    }
    for (long long i = gt; i <= a.r0; i += GT) {
      a.rows_start[i] = a.start_in[i];
      if (i == a.r0) break;
      a.rows_basis[i] = a.rb_in[i];
      u16 e[MAXV], z[MAXV];
      for (int v = 0; v < n; ++v) {
        e[v] = a.shift_in[i * n + v];
        z[v] = 0;
      }
      key_store<KW>(a.rows_delta, i, key_sub<KW>(key_encode<KW>(a.f, e), key_encode<KW>(a.f, z)));
    }
    grid.sync();
    if (a.trace && blockIdx.x == 0 && tid == 0) a.trace[384] = gtimer();
    // P1: leads of the input rows are covered (symbolic.py:339); every term
    // of the input rows -> its dictionary bit (a stale L1 read of the map
    // only costs a redundant atomic)
    if (a.closure)
      for (long long i = gt; i < a.r0; i += GT) {
        const int g = __ldcg(a.rows_basis + i);
        const Key<KW> k = key_add<KW>(key_load<KW>(a.bckey, __ldg(a.boff + g)), key_load_cg<KW>(a.rows_delta, i));
        const u32 rk = key_rank<KW>(a.f, bt, a.st, k);
        atomicOr(a.done + (rk >> 5), 1u << (rk & 31));
      }
    for (long long i = gw; i < a.r0; i += W) {
      const int g = __ldcg(a.rows_basis + i);
      const u32 off = __ldg(a.boff + g), len = __ldg(a.blen + g);
      const Key<KW> dl = key_load_cg<KW>(a.rows_delta, i);
      for (u32 t = lane; t < len; t += 32) {
        const Key<KW> kk = key_add<KW>(key_load<KW>(a.bckey, (long long)off + t), dl);
        const u32 rk = key_rank<KW>(a.f, bt, a.st, kk);
        const u32 bit = 1u << (rk & 31);
        if (!(a.dict[rk >> 5] & bit)) atomicOr(a.dict + (rk >> 5), bit);
      }
    }
    grid.sync();
    if (a.trace && blockIdx.x == 0 && tid == 0) a.trace[385] = gtimer();
    // P2: dictionary size and the round-1 frontier dict & ~done (ascending)
    {
      u32 cf = 0, cd = 0;
      for (u32 w = w_lo + tid; w < w_hi; w += blockDim.x) {
        const u32 d = __ldcg(a.dict + w);
        cd += __popc(d);
        if (a.closure) cf += __popc(d & ~__ldcg(a.done + w));
      }
      cf = block_sum_u32(cf, ws);
      cd = block_sum_u32(cd, ws);
      if (tid == 0) {
        a.chunkcnt[blockIdx.x] = cf;
        a.chunkcnt[G + blockIdx.x] = cd;
      }
    }
    grid.sync();
    u32 base, dummy;
    chunk_bases(a.chunkcnt, base, nf);
    chunk_bases(a.chunkcnt + G, dummy, N);
    if (nf > a.front_cap) {
      flags |= LOOP_OVERFLOW;
      nf = 0;
    } else if (a.closure && nf) {
      emit_chunk([&](u32 w) { return __ldcg(a.dict + w) & ~__ldcg(a.done + w); }, base, a.front0, nullptr, 0u);
    }
    if (!a.closure) nf = 0;
    grid.sync();
    if (a.trace && blockIdx.x == 0 && tid == 0) a.trace[386] = gtimer();
  }
  while (nf > 0 && a.nc > 0) {
    const u64* front = sel ? a.front1 : a.front0;
    u64* fnext = sel ? a.front0 : a.front1;
    const bool tr = a.trace && blockIdx.x == 0 && tid == 0 && rounds < 64;
    if (tr) {
      a.trace[rounds * 6] = gtimer();
      a.trace[rounds * 6 + 5] = nf;
    }
    // ---- A: first LM divisor in preference order (symbolic.py:228-235),
    // warp per monomial over contiguous per-warp ranges; per-warp counts.
    const u32 per = (nf + W - 1) / W;
    const u32 j0 = min(nf, gw * per), j1 = min(nf, j0 + per);
    {
      u32 cn = 0, cl = 0;
      for (u32 j = j0; j < j1; ++j) {
        int found = -1;
        u16 e[MAXV + 1];
        key_decode<KW>(a.f, key_load_cg<KW>(front, j), e);
        e[n] = 0;
        u32 me[MAXV / 2];
        for (int w = 0; w < a.nw; ++w) me[w] = (u32)e[2 * w] | ((u32)e[2 * w + 1] << 16);
        for (int b0 = 0; b0 < a.nc; b0 += 32) {
          const int cc = b0 + lane;
          bool ok = cc < a.nc;
          if (ok) {
            const u32* lm = lmw + (long long)cc * a.nw;
            for (int w = 0; w < a.nw; ++w) ok &= (__vcmpgeu2(me[w], lm[w]) == 0xFFFFFFFFu);
          }
          const unsigned bm = __ballot_sync(0xffffffffu, ok);
          if (bm) {
            found = __ldg(a.cidx + b0 + __ffs(bm) - 1);
            break;
          }
        }
        if (lane == 0) a.red[j] = found;
        if (found >= 0) {
          ++cn;
          cl += __ldg(a.blen + found);
        }
      }
      if (lane == 0) {
        a.tilecnt[2 * gw] = cn;
        a.tilecnt[2 * gw + 1] = cl;
      }
    }
    grid.sync();
    if (tr) a.trace[rounds * 6 + 1] = gtimer();
    // ---- totals and this warp's row / term bases
    u32 R, Mk, bn, bl;
    {
      u32 tn = 0, tl = 0, pn = 0, pl = 0;
      const u32 mine = blockIdx.x * NWARP;
      for (u32 w = tid; w < W; w += blockDim.x) {
        const u32 vn = __ldcg(a.tilecnt + 2 * w), vl = __ldcg(a.tilecnt + 2 * w + 1);
        tn += vn;
        tl += vl;
        if (w < mine) {
          pn += vn;
          pl += vl;
        }
        if (w >= mine && w < mine + NWARP) {
          s_wn[w - mine] = vn;
          s_wl[w - mine] = vl;
        }
      }
      R = block_sum_u32(tn, ws);
      Mk = block_sum_u32(tl, ws);
      bn = block_sum_u32(pn, ws);
      bl = block_sum_u32(pl, ws);
      for (int q = 0; q < warp; ++q) {
        bn += s_wn[q];
        bl += s_wl[q];
      }
    }
    if (R == 0) break;
    if (r + R + 1 > a.rows_cap || n_cl + R > a.cl_cap) {
      flags |= LOOP_OVERFLOW;
      break;
    }
    if ((unsigned long long)Mcur + Mk >= (1ull << 30)) {
      flags |= LOOP_SIZE_CAP;
      break;
    }
    if (blockIdx.x == 0 && tid == 0) a.rows_start[r + R] = Mcur + Mk;
    // ---- B: the warp's rows, in frontier order
    for (u32 jb = j0; jb < j1; jb += 32) {
      const u32 j = jb + lane;
      const int g = j < j1 ? __ldcg(a.red + j) : -1;
      const u32 len = g >= 0 ? __ldg(a.blen + g) : 0u;
      const unsigned bm = __ballot_sync(0xffffffffu, g >= 0);
      u32 lp = len;
#pragma unroll
      for (int o = 1; o < 32; o <<= 1) {
        const u32 y = __shfl_up_sync(0xffffffffu, lp, o);
        if (lane >= o) lp += y;
      }
      const u32 ltot = __shfl_sync(0xffffffffu, lp, 31);
      if (g >= 0) {
        const long long q = (long long)bn + __popc(bm & lanemask_lt());
        const long long row = r + q;
        const Key<KW> m = key_load_cg<KW>(front, j);
        a.rows_basis[row] = g;
        key_store<KW>(a.rows_delta, row, key_sub<KW>(m, key_load<KW>(a.bckey, __ldg(a.boff + g))));
        a.rows_start[row] = Mcur + bl + lp - len;
        u16 e[MAXV];
        key_decode<KW>(a.f, m, e);
        bool over = false;
        for (int v = 0; v < n; ++v) {
          const u32 s = (u32)e[v] - (u32)a.lmexp[(long long)g * n + v];
          over |= (s + (u32)a.maxe[(long long)g * n + v]) > 0xFFFFu;
          a.cl_shift[(n_cl + q) * n + v] = (u16)s;
        }
        if (over) atomicOr(a.err, (u32)DEVERR_LANE_OVERFLOW);
        a.cl_basis[n_cl + q] = g;
        a.cl_round[n_cl + q] = (int)rounds + 1;
      }
      bn += __popc(bm);
      bl += ltot;
    }
    // ---- C: every term of the new rows -> rank; absent monomials into
    // newbits.  Items (frontier entry, 32-term chunk) over all warps of the
    // grid.  The dictionary test is only a filter (a stale hit just costs an
    // extra atomic; D masks with the dictionary), so it may use the L1 path.
    for (u32 it = gw; it < nf * CH; it += W) {
      const u32 j = it / CH, ch = it - j * CH;
      const int g = __ldcg(a.red + j);
      if (g < 0) continue;
      const u32 len = __ldg(a.blen + g);
      if (ch * 32 >= len) continue;
      const u32 off = __ldg(a.boff + g);
      const Key<KW> dl = key_sub<KW>(key_load_cg<KW>(front, j), key_load<KW>(a.bckey, off));
      const u32 t = ch * 32 + lane;
      if (t < len) {
        const Key<KW> kk = key_add<KW>(key_load<KW>(a.bckey, (long long)off + t), dl);
        const u32 rk = key_rank<KW>(a.f, bt, a.st, kk);
        const u32 bit = 1u << (rk & 31);
        if (!(__ldg(a.dict + (rk >> 5)) & bit)) atomicOr(a.newbits + (rk >> 5), bit);
      }
    }
    grid.sync();
    if (tr) a.trace[rounds * 6 + 2] = gtimer();
    // ---- D1: popcount of the CTA's word chunk (new = newbits & ~dict)
    {
      u32 cnt = 0;
      for (u32 w = w_lo + tid; w < w_hi; w += blockDim.x) cnt += __popc(__ldcg(a.newbits + w) & ~__ldcg(a.dict + w));
      cnt = block_sum_u32(cnt, ws);
      if (tid == 0) a.chunkcnt[blockIdx.x] = cnt;
    }
    grid.sync();
    if (tr) a.trace[rounds * 6 + 3] = gtimer();
    // ---- D2: next frontier (ascending rank), dictionary update
    u32 base, total;
    {
      u32 sb = 0, st = 0;
      for (u32 b = tid; b < G; b += blockDim.x) {
        const u32 v = __ldcg(a.chunkcnt + b);
        st += v;
        if (b < blockIdx.x) sb += v;
      }
      base = block_sum_u32(sb, ws);
      total = block_sum_u32(st, ws);
    }
    if (total > a.front_cap) {
      flags |= LOOP_OVERFLOW;
      break;
    }
    for (u32 w0 = w_lo; w0 < w_hi; w0 += blockDim.x) {
      const u32 w = w0 + tid;
      u32 x = 0;
      if (w < w_hi) {
        const u32 nb = __ldcg(a.newbits + w);
        if (nb) {
          const u32 d = __ldcg(a.dict + w);
          x = nb & ~d;
          a.dict[w] = d | nb;
          a.newbits[w] = 0;
        }
      }
      u32 tt;
      const u32 pre = block_scan_excl(__popc(x), ws, &tt);
      if (tt <= (u32)CL_LIST) {
        u32 p = pre, m = x;
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          list[p++] = w * 32 + b;
        }
        __syncthreads();
        for (u32 q = tid; q < tt; q += blockDim.x) {
          u16 e[MAXV];
          unrank_exps(list[q], n, a.D, bt, a.st, e);
          key_store<KW>(fnext, base + q, key_encode<KW>(a.f, e));
        }
        __syncthreads();
      } else {
        u32 p = base + pre, m = x;
        while (m) {
          const int b = __ffs(m) - 1;
          m &= m - 1;
          u16 e[MAXV];
          unrank_exps(w * 32 + b, n, a.D, bt, a.st, e);
          key_store<KW>(fnext, p++, key_encode<KW>(a.f, e));
        }
      }
      base += tt;
    }
    r += R;
    n_cl += R;
    Mcur += Mk;
    ++rounds;
    nf = total;
    N += total;
    sel ^= 1;
    if ((long long)N > a.dict_cap) {
      flags |= LOOP_DICT_CAP;
      break;
    }
    grid.sync();
    if (tr) a.trace[(rounds - 1) * 6 + 4] = gtimer();
  }
  if (blockIdx.x == 0 && tid == 0) t_epi = gtimer();
  if (a.full && !flags) {
    if (N > a.N_cap || Mcur > a.M_cap || r + 1 > a.rows_cap) {
      flags |= LOOP_OVERFLOW;
    } else {
      // P3: final dictionary: keys ascending, exponents in column order
      // (descending), word prefix for the column map
      {
        u32 cd = 0;
        for (u32 w = w_lo + tid; w < w_hi; w += blockDim.x) cd += __popc(__ldcg(a.dict + w));
        cd = block_sum_u32(cd, ws);
        if (tid == 0) a.chunkcnt[blockIdx.x] = cd;
      }
      grid.sync();
      u32 base, tot;
      chunk_bases(a.chunkcnt, base, tot);
      emit_chunk([&](u32 w) { return __ldcg(a.dict + w); }, base, a.dict_out, a.dict_exps, N);
      grid.sync();
      if (a.trace && blockIdx.x == 0 && tid == 0) a.trace[387] = gtimer();
      // P4: join (symbolic.py:360-388): every term -> rank -> column
      //   col = N - 1 - (prefix[rank >> 5] + popc(word & below(rank)))
      bool miss = false;
      for (long long i = gw; i < r; i += W) {
        const int g = __ldcg(a.rows_basis + i);
        const u32 off = __ldg(a.boff + g), len = __ldg(a.blen + g);
        const u32 rs = __ldcg(a.rows_start + i);
        const Key<KW> dl = key_load_cg<KW>(a.rows_delta, i);
        for (u32 t = lane; t < len; t += 32) {
          const Key<KW> kk = key_add<KW>(key_load<KW>(a.bckey, (long long)off + t), dl);
          const u32 rk = key_rank<KW>(a.f, bt, a.st, kk);
          const uint2 dw = __ldcg(a.dwp + (rk >> 5));
          if (!((dw.x >> (rk & 31)) & 1u)) miss = true;
          a.col[rs + t] = N - 1 - (dw.y + __popc(dw.x & ((1u << (rk & 31)) - 1u)));
          a.val[rs + t] = __ldg(a.bcoeff + off + t);
        }
      }
      if (miss) atomicOr(a.err, (u32)DEVERR_MISSING_KEY);
    }
  }
  if (blockIdx.x == 0 && tid == 0) {
    LoopOut o;
    o.r = (u32)r;
    o.n_cl = (u32)n_cl;
    o.M = Mcur;
    o.N = N;
    o.rounds = rounds;
    o.nf = nf;
    o.flags = flags;
    o.sel = (u32)sel;
    o.t_start = t_start;
    o.t_epi = t_epi;
    o.t_end = gtimer();
    *a.out = o;
  }
}

// ===========================================================================
// k_fbsp: the whole rank-path compile_batch (symbolic.py:293-388) in ONE
// cooperative launch.  Grid barriers:
//   P1  input rows: shift deltas, row table, lead bits, dictionary bits
//       (first setter of a bit counts it for the owning word chunk)   | sync
//   P2  round-1 frontier = dict & ~done: chunk counts | sync | emit  | sync
//   per closure round (2 barriers):
//     AC  reducer search (symbolic.py:228-235) and, in the same warps,
//         ranking of the reducer rows' terms: absent monomials into
//         newbits, first setters counted per word chunk              | sync
//     BD  row bases -> rows written in frontier order; chunk bases ->
//         next frontier (ascending rank = ascending key), dict |= new | sync
//   P3  final dictionary: keys ascending, exponents in column order, word
//       prefix for the column map                                     | sync
//   P4  join: every term -> rank -> column (symbolic.py:360-388)      | sync
// The presence maps and the per-chunk counters are zero on entry and left
// zero on exit (the host clears them after an aborted run).  All exits are
// grid-uniform: every CTA derives the loop state from the same counters.
// ===========================================================================
struct FbspArgs {
  KeyFmt f;
  int D, st, bt_words, closure, nc, nw, stage_lm;
  unsigned long long prefetch_terms;  // basis terms to pull into L2 up front (0 = none)
  u32 words, maxlen, front_cap, N_cap, M_cap, M0;
  long long r0, rows_cap, cl_cap, dict_cap;
  const u32* bt;
  const int* rb_in;
  const u32* start_in;
  const u16* shift_in;
  const u32* lmw;
  const int* cidx;
  const u32* boff;
  const u32* blen;
  const u64* bckey;
  const u32* bcoeff;
  const u16* lmexp;
  const u16* maxe;
  u32* dict;
  u32* done;
  u32* newbits;
  uint2* dwp;
  u64* front0;
  u64* front1;
  int* red;
  u32* tilecnt;  // [2 * warps]
  u32* cnt;      // [4 * G] this call: new-bit counts (two parities), dictionary and lead counts per chunk
  u32* cnt_next; // the next call's set, cleared here ([0, cnt_clear))
  u32 cnt_clear;
  u32 big_nf;    // frontier size from which a round ranks over balanced term ranges (0: one per warp of the grid)
  int* rows_basis;
  u64* rows_delta;
  u32* rows_start;
  int* cl_basis;
  u16* cl_shift;
  int* cl_round;
  u64* dict_out;
  u16* dict_exps;
  u32* col;
  u32* val;
  u32* err;
  LoopOut* out;
  unsigned long long* trace;
};

template <int KW, int NV>
__global__ void __launch_bounds__(FB_THREADS) k_fbsp(const FbspArgs a) {
  namespace cg = cooperative_groups;
  cg::grid_group grid = cg::this_grid();
  extern __shared__ __align__(16) u32 csm[];
  u32* bt = csm;
  u32* list = csm + ((a.bt_words + 3) & ~3);  // 16-byte aligned
  u32* slm = list + CL_LIST;
  __shared__ u32 ws[33];
  __shared__ u32 s_red6[FB_THREADS / 32][6];  // fused BD reductions of a small round
  __shared__ u32 s_wn[FB_THREADS / 32], s_wl[FB_THREADS / 32];
  // a group's reducer and exponent words per frontier monomial (small rounds,
  // up to 32 monomials per group), kept from the search for the row writer
  constexpr bool STASH = NV <= 16;
  constexpr int JW = STASH ? (NV + 1) / 2 : 1;
  __shared__ int s_jf[STASH ? FB_THREADS / 32 : 1][32];
  __shared__ u32 s_je[STASH ? FB_THREADS / 32 : 1][32][JW];
  __shared__ u32 s_jl[STASH ? FB_THREADS / 32 : 1][32];                       // reducer length
  __shared__ unsigned long long s_jd[STASH ? FB_THREADS / 32 : 1][32][KW];  // row key delta (small rounds)
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  constexpr int NWARP = FB_THREADS / 32;
  constexpr int U = 1;  // 32-term chunks per warp step (U = 4 / 2 / 1 measured 2.90e9 / 3.04e9 / 3.08e9 nnz/s: finer term ranges)
  const int n = a.f.n_vars;
  const u32 G = gridDim.x, W = G * NWARP, gw = blockIdx.x * NWARP + warp;
  // pull the basis keys / coefficients into L2 (one 128-byte line per
  // thread-step): the per-warp chains below then start from L2, not HBM
  if (a.prefetch_terms) {
    const char* kp = reinterpret_cast<const char*>(a.bckey);
    const char* cp = reinterpret_cast<const char*>(a.bcoeff);
    const unsigned long long kb_ = a.prefetch_terms * KW * 8, cb_ = a.prefetch_terms * 4;
    const unsigned long long gt = (unsigned long long)blockIdx.x * blockDim.x + tid, GT = (unsigned long long)G * blockDim.x;
    for (unsigned long long o = gt * 128; o < kb_; o += GT * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(kp + o));
    for (unsigned long long o = gt * 128; o < cb_; o += GT * 128) asm volatile("prefetch.global.L2 [%0];" ::"l"(cp + o));
  }
  // stage the binomial and LM tables (16-byte loads, all in flight)
  for (int i = tid; i < a.bt_words; i += blockDim.x) bt[i] = a.bt[i];
  const u32* lmw = a.lmw;
  if (a.stage_lm) {
    const int nv = (a.nc * a.nw) >> 2;
    const uint4* src = reinterpret_cast<const uint4*>(a.lmw);
    uint4* dst = reinterpret_cast<uint4*>(slm);
    int i = tid;
    for (; i + 3 * (int)blockDim.x < nv; i += 4 * blockDim.x) {
      const uint4 v0 = src[i], v1 = src[i + blockDim.x], v2 = src[i + 2 * blockDim.x], v3 = src[i + 3 * blockDim.x];
      dst[i] = v0;
      dst[i + blockDim.x] = v1;
      dst[i + 2 * blockDim.x] = v2;
      dst[i + 3 * blockDim.x] = v3;
    }
    for (; i < nv; i += blockDim.x) dst[i] = src[i];
    for (int w = (nv << 2) + tid; w < a.nc * a.nw; w += blockDim.x) slm[w] = a.lmw[w];
    lmw = slm;
  }
  // the next call's counters are idle now: clear them
  for (u32 i = blockIdx.x * blockDim.x + tid; i < a.cnt_clear; i += G * blockDim.x) a.cnt_next[i] = 0;
  if (blockIdx.x == 0 && tid == 0) *a.err = 0;  // nothing sets it before the first grid barrier
  __syncthreads();
  const u32 CH = max(1u, (a.maxlen + 31) / 32);
  const u32 cw = (((a.words + G - 1) / G) + 31) & ~31u;
  const u32 w_lo = min(a.words, blockIdx.x * cw), w_hi = min(a.words, w_lo + cw);
  u32* cnt_a = a.cnt;
  u32* cnt_b = a.cnt + G;
  u32* dcount = a.cnt + 2 * G;
  u32* lcount = a.cnt + 3 * G;
  const bool t0th = blockIdx.x == 0 && tid == 0;
  unsigned long long t_start = t0th ? gtimer() : 0ull, t_epi = 0;
  auto stamp = [&](int slot) {
    if (a.trace && t0th) a.trace[slot] = gtimer();
  };
  // exclusive base of this CTA and the total over per-CTA values v(b)
  auto cta_bases = [&](auto v, u32& base, u32& total) {
    u32 sb = 0, stt = 0;
    for (u32 b = tid; b < G; b += blockDim.x) {
      const u32 x = v(b);
      stt += x;
      if (b < blockIdx.x) sb += x;
    }
    base = block_sum_u32(sb, ws);
    total = block_sum_u32(stt, ws);
  };
  // k warps per item (k = W / n_items clamped to [1, kmax]); each group of k
  // warps owns a contiguous item range; `sub` is the warp's rank in it
  auto groups_of = [&](u32 nitems, u32 kmax, u32& k, u32& i0, u32& i1, u32& sub) {
    k = nitems >= W ? 1u : max(1u, min(W / max(nitems, 1u), kmax));
    const u32 ng = W / k, g = gw / k;
    sub = gw - g * k;
    const u32 per = (nitems + ng - 1) / ng;
    i0 = g < ng ? min(nitems, g * per) : nitems;
    i1 = g < ng ? min(nitems, i0 + per) : nitems;
  };
  // set bits of getx(w) over this CTA's chunk, ascending from `base`: their
  // RANKS to out[pos] (a u32 list; the frontier consumers and the final
  // dictionary pass unrank them, balanced over the grid) and, with dwp, the
  // word prefix for the join.  One store per monomial: a chunk owning most of
  // the dictionary no longer serialises the unranking.
  auto emit_chunk = [&](auto getx, u32 base, u32* out, bool with_dwp, u32 stride) {
    for (u32 w0 = w_lo; w0 < w_hi; w0 += blockDim.x) {
      const u32 w = w0 + tid;
      const u32 x = w < w_hi ? getx(w) : 0u;
      u32 tt;
      const u32 pre = block_scan_excl(__popc(x), ws, &tt);
      if (with_dwp && w < w_hi) a.dwp[w] = make_uint2(x, base + pre);
      u32 p = base + pre, m = x;
      while (m) {
        const int b = __ffs(m) - 1;
        m &= m - 1;
        out[(size_t)(p++) * stride] = w * 32 + b;
      }
      base += tt;
    }
  };
  // ranks of terms [0, len) of the basis polynomial at `off` times the shift
  // `dl`, chunks sub, sub + k, ... with U chunks in flight per lane
  auto rank_chunks = [&](u32 off, u32 len, const Key<KW>& dl, u32 sub, u32 k, u32 c, u32* tt, u32* rk) {
    Key<KW> kk[U];
#pragma unroll
    for (int q = 0; q < U; ++q) {
      tt[q] = (c + q * k) * 32 + lane;
      if (tt[q] < len) kk[q] = key_load<KW>(a.bckey, (long long)off + tt[q]);
    }
#pragma unroll
    for (int q = 0; q < U; ++q)
      if (tt[q] < len) rk[q] = key_rank<KW>(a.f, bt, a.st, key_add<KW>(kk[q], dl));
  };
  // Balanced term ranges: terms [t_begin, t_end) of rows [row_lo, row_hi)
  // (row i owns [rs(i), rs(i) + len_i), rs ascending).  Warp gw takes the
  // contiguous range [a0, a1) of T terms, finds its first row with a 32-ary
  // warp search, then walks rows: body(i, rs_i, from, to).
  auto term_ranges = [&](u32 row_lo, u32 row_hi, u32 t_begin, u32 t_end, auto rs_of, auto body) {
    if (t_end <= t_begin || row_hi <= row_lo) return;
    const u32 T = (((t_end - t_begin) + W - 1) / W + 31) & ~31u;
    const unsigned long long a0l = (unsigned long long)t_begin + (unsigned long long)gw * T;
    if (a0l >= t_end) return;
    const u32 a0 = (u32)a0l, a1 = min(t_end, a0 + T);
    u32 lo = row_lo, hi = row_hi;  // rs(lo) <= a0 < rs(hi)
    while (hi - lo > 1) {
      const u32 step = (hi - lo + 31) / 32;
      const u32 pr = lo + step * (lane + 1);
      const bool le = pr < hi && rs_of(pr) <= a0;
      const u32 c = __popc(__ballot_sync(0xffffffffu, le));
      lo += step * c;
      hi = min(hi, lo + step);
    }
    for (u32 i = lo; i < row_hi; ++i) {
      const u32 rsi = rs_of(i);
      if (rsi >= a1) break;
      body(i, rsi, max(a0, rsi), a1);
    }
  };

  // ---- P1: input rows: shift deltas, row table, lead bits, dictionary bits
  // (balanced term ranges; the first setter of a bit counts it for the
  // owning word chunk; the warp owning a row's first term writes its entry)
  term_ranges(0u, (u32)a.r0, 0u, a.M0, [&](u32 i) { return a.start_in[i]; }, [&](u32 i, u32 rsi, u32 from, u32 to) {
    const int g = a.rb_in[i];
    u16 e[NV], z[NV];
#pragma unroll
    for (int v = 0; v < NV; ++v) {
      e[v] = v < n ? a.shift_in[(long long)i * n + v] : (u16)0;
      z[v] = 0;
    }
    const Key<KW> dl = key_sub<KW>(gl_encode<KW, NV>(a.f, e), gl_encode<KW, NV>(a.f, z));
    const u32 off = __ldg(a.boff + g), len = __ldg(a.blen + g);
    if (from == rsi && lane == 0) {
      a.rows_basis[i] = g;
      key_store<KW>(a.rows_delta, i, dl);
      a.rows_start[i] = rsi;
      if (a.closure) {
        // leads of the input rows are covered (symbolic.py:339)
        const u32 rk = key_rank<KW>(a.f, bt, a.st, key_add<KW>(key_load<KW>(a.bckey, off), dl));
        const u32 bit = 1u << (rk & 31);
        if (!(atomicOr(a.done + (rk >> 5), bit) & bit)) atomicAdd(lcount + (rk >> 5) / cw, 1u);
      }
    }
    const u32 t_lo = from - rsi, t_hi = min(len, to - rsi);
    for (u32 tb = t_lo; tb < t_hi; tb += 32 * U) {
      u32 tt[U], rk[U], dw[U];
      Key<KW> kk[U];
#pragma unroll
      for (int q = 0; q < U; ++q) {
        tt[q] = tb + q * 32 + lane;
        if (tt[q] < t_hi) kk[q] = key_load<KW>(a.bckey, (long long)off + tt[q]);
      }
#pragma unroll
      for (int q = 0; q < U; ++q)
        if (tt[q] < t_hi) {
          rk[q] = key_rank<KW>(a.f, bt, a.st, key_add<KW>(kk[q], dl));
          a.col[rsi + tt[q]] = rk[q];  // parked for the join (P4 turns it into the column)
        }
#pragma unroll
      for (int q = 0; q < U; ++q) dw[q] = tt[q] < t_hi ? __ldcg(a.dict + (rk[q] >> 5)) : 0xFFFFFFFFu;  // L2 filter
      // lanes whose bits fall in the same word combine them: one atomicOr
      // per distinct word of the warp (a row's consecutive terms often share
      // a word), the new bits counted by the lane that issued it
#pragma unroll
      for (int q = 0; q < U; ++q) {
        const u32 w = rk[q] >> 5, bit = 1u << (rk[q] & 31);
        const bool need = tt[q] < t_hi && !(dw[q] & bit);
        const unsigned grp = __match_any_sync(0xffffffffu, need ? w : 0xFFFFFFFFu);
        const u32 gb = __reduce_or_sync(grp, need ? bit : 0u);
        if (need && lane == __ffs(grp) - 1) {
          const u32 nb = gb & ~atomicOr(a.dict + w, gb);
          if (nb) atomicAdd(dcount + w / cw, (u32)__popc(nb));
        }
      }
    }
  });
  if (t0th) a.rows_start[a.r0] = a.start_in[a.r0];
  grid.sync();
  stamp(384);
  // ---- P2: dictionary size, round-1 frontier = dict & ~done (every lead is
  // a dictionary monomial, so the chunk counts are dcount - lcount)
  u32 nf = 0, N = 0, flags = 0, rounds = 0;
  {
    // N, nf and this CTA's frontier base in one pass (one CTA barrier)
    u32 v3[3] = {0u, 0u, 0u};
    for (u32 b = tid; b < G; b += blockDim.x) {
      const u32 d = __ldcg(dcount + b), f = a.closure ? d - __ldcg(lcount + b) : 0u;
      v3[0] += d;
      v3[1] += f;
      if (b < blockIdx.x) v3[2] += f;
    }
#pragma unroll
    for (int q = 0; q < 3; ++q)
#pragma unroll
      for (int o = 16; o; o >>= 1) v3[q] += __shfl_xor_sync(0xffffffffu, v3[q], o);
    if (lane == 0)
#pragma unroll
      for (int q = 0; q < 3; ++q) s_red6[warp][q] = v3[q];
    __syncthreads();
#pragma unroll
    for (int q = 0; q < 3; ++q) {
      u32 t = 0;
#pragma unroll
      for (int w = 0; w < NWARP; ++w) t += s_red6[w][q];
      v3[q] = t;
    }
    N = v3[0];
    const u32 base = v3[2];
    if (a.closure) {
      nf = v3[1];
      if (nf > a.front_cap) {
        flags |= LOOP_OVERFLOW;
      } else {
        emit_chunk([&](u32 w) {
          const u32 d = __ldcg(a.dict + w), dn = __ldcg(a.done + w);
          if (dn) a.done[w] = 0;
          return d & ~dn;
        }, base, reinterpret_cast<u32*>(a.front0), false, 1u);
      }
      grid.sync();
    }
  }
  stamp(385);
  // ---- closure rounds ------------------------------------------------------
  long long r = a.r0, n_cl = 0;
  u32 Mcur = a.M0;
  int sel = 0;
  while (!flags && nf > 0 && a.nc > 0) {
    const u32* front = reinterpret_cast<const u32*>(sel ? a.front1 : a.front0);  // ranks, ascending
    u32* fnext = reinterpret_cast<u32*>(sel ? a.front0 : a.front1);
    u32* cur = (rounds & 1) ? cnt_b : cnt_a;
    u32* nxt = (rounds & 1) ? cnt_a : cnt_b;
    const bool tr = a.trace && t0th && rounds < 64;
    if (tr) {
      a.trace[rounds * 6] = gtimer();
      a.trace[rounds * 6 + 5] = nf;
    }
    // big rounds (nf >= W): search only here, the reducer rows' terms are
    // ranked after the rows are written, over balanced term ranges (two more
    // barriers); small rounds rank inside the search groups
    const bool big = nf >= (a.big_nf ? a.big_nf : W);
    u32 k, j0, j1, sub;
    groups_of(nf, big ? 1u : CH, k, j0, j1, sub);
    const bool leader = sub == 0;
    // ---- AC: reducer search (every warp of the group) + ranking of the
    // reducer row's terms (chunks split across the group)
    {
      u32 cn = 0, cl = 0;
      for (u32 j = j0; j < j1; ++j) {
        int found = -1;
        u16 e[NV];
        gl_unrank<NV>(__ldcg(front + j), n, a.D, bt, a.st, e);
        const Key<KW> m = gl_encode<KW, NV>(a.f, e);
        constexpr int NW2 = (NV + 1) / 2;
        u32 me[NW2];
#pragma unroll
        for (int w = 0; w < NW2; ++w)
          me[w] = (u32)e[2 * w] | (2 * w + 1 < NV ? ((u32)e[2 * w + 1] << 16) : 0u);
        for (int b0 = 0; b0 < a.nc; b0 += 32) {
          const int cc = b0 + lane;
          bool ok = cc < a.nc;
          if (ok) {
            const u32* lm = lmw + (long long)cc * a.nw;
#pragma unroll
            for (int w = 0; w < NW2; ++w)
              if (w < a.nw) ok &= (__vcmpgeu2(me[w], lm[w]) == 0xFFFFFFFFu);
          }
          const unsigned bm = __ballot_sync(0xffffffffu, ok);
          if (bm) {
            found = a.cidx[b0 + __ffs(bm) - 1];
            break;
          }
        }
        if (leader) {
          if (lane == 0) a.red[j] = found;
          if (found >= 0) {
            ++cn;
            cl += __ldg(a.blen + found);
          }
          if (STASH && j1 - j0 <= 32u) {
            if (lane == 0) {
              s_jf[warp][j - j0] = found;
              s_jl[warp][j - j0] = found >= 0 ? __ldg(a.blen + found) : 0u;
            }
#pragma unroll
            for (int w = 0; w < JW; ++w)
              if (lane == w) s_je[warp][j - j0][w] = me[w];
          }
        }
        if (found < 0 || big) continue;
        const u32 off = __ldg(a.boff + found), len = __ldg(a.blen + found);
        const Key<KW> dl = key_sub<KW>(m, key_load<KW>(a.bckey, off));
        if (STASH && leader && lane == 0 && j1 - j0 <= 32u)
#pragma unroll
          for (int w = 0; w < KW; ++w) s_jd[warp][j - j0][w] = dl.w[w];
        for (u32 c = sub; c * 32 < len; c += U * k) {
          u32 tt[U], rk[U], dw[U];
          rank_chunks(off, len, dl, sub, k, c, tt, rk);
#pragma unroll
          for (int q = 0; q < U; ++q)
            dw[q] = tt[q] < len ? (__ldcg(a.dict + (rk[q] >> 5)) | __ldcg(a.newbits + (rk[q] >> 5))) : 0xFFFFFFFFu;
#pragma unroll
          for (int q = 0; q < U; ++q) {
            if (tt[q] >= len) continue;
            const u32 w = rk[q] >> 5, bit = 1u << (rk[q] & 31);
            if (!(dw[q] & bit) && !(atomicOr(a.newbits + w, bit) & bit)) atomicAdd(cur + w / cw, 1u);
          }
        }
      }
      if (lane == 0) {
        s_wn[warp] = cn;
        s_wl[warp] = cl;
      }
      __syncthreads();
      if (tid == 0) {
        u32 sn = 0, sl = 0;
        for (int q = 0; q < NWARP; ++q) {
          sn += s_wn[q];
          sl += s_wl[q];
        }
        a.tilecnt[2 * blockIdx.x] = sn;
        a.tilecnt[2 * blockIdx.x + 1] = sl;
      }
    }
    grid.sync();
    if (tr) a.trace[rounds * 6 + 1] = gtimer();
    // ---- BD: totals, this warp's row / term bases; a small round's new
    // monomial counts are final here too, so the CTA's frontier base comes
    // out of the same pass (one CTA barrier for all six sums)
    u32 R, Mk, bn, bl, base = 0, total = 0;
    {
      u32 v6[6] = {0u, 0u, 0u, 0u, 0u, 0u};  // tn, tl, pn, pl, total, base
      for (u32 b = tid; b < G; b += blockDim.x) {
        const uint2 v = __ldcg(reinterpret_cast<const uint2*>(a.tilecnt) + b);
        const u32 x = big ? 0u : __ldcg(cur + b);
        v6[0] += v.x;
        v6[1] += v.y;
        v6[4] += x;
        if (b < blockIdx.x) {
          v6[2] += v.x;
          v6[3] += v.y;
          v6[5] += x;
        }
      }
#pragma unroll
      for (int q = 0; q < 6; ++q)
#pragma unroll
        for (int o = 16; o; o >>= 1) v6[q] += __shfl_xor_sync(0xffffffffu, v6[q], o);
      if (lane == 0)
#pragma unroll
        for (int q = 0; q < 6; ++q) s_red6[warp][q] = v6[q];
      __syncthreads();
#pragma unroll
      for (int q = 0; q < 6; ++q) {
        u32 t = 0;
#pragma unroll
        for (int w = 0; w < NWARP; ++w) t += s_red6[w][q];
        v6[q] = t;
      }
      R = v6[0];
      Mk = v6[1];
      bn = v6[2];
      bl = v6[3];
      total = v6[4];
      base = v6[5];
      for (int q = 0; q < warp; ++q) {
        bn += s_wn[q];
        bl += s_wl[q];
      }
    }
    if (R == 0) break;
    if (r + R + 1 > a.rows_cap || n_cl + R > a.cl_cap) {
      flags |= LOOP_OVERFLOW;
      break;
    }
    if ((unsigned long long)Mcur + Mk >= (1ull << 30)) {
      flags |= LOOP_SIZE_CAP;
      break;
    }
    if (t0th) a.rows_start[r + R] = Mcur + Mk;
    // B: the group's rows, in frontier order (leader warp)
    if (leader) {
      const bool stashed = STASH && j1 - j0 <= 32u;
      for (u32 jb = j0; jb < j1; jb += 32) {
        const u32 j = jb + lane;
        const int g = j < j1 ? (stashed ? s_jf[warp][lane] : __ldcg(a.red + j)) : -1;
        const u32 len = g >= 0 ? (stashed ? s_jl[warp][lane] : __ldg(a.blen + g)) : 0u;
        const unsigned bm = __ballot_sync(0xffffffffu, g >= 0);
        u32 lp = len;
#pragma unroll
        for (int o = 1; o < 32; o <<= 1) {
          const u32 y = __shfl_up_sync(0xffffffffu, lp, o);
          if (lane >= o) lp += y;
        }
        const u32 ltot = __shfl_sync(0xffffffffu, lp, 31);
        if (g >= 0) {
          const long long q = (long long)bn + __popc(bm & lanemask_lt());
          const long long row = r + q;
          u16 e[NV];
          if (stashed) {
#pragma unroll
            for (int v = 0; v < NV; ++v) e[v] = (u16)(s_je[warp][lane][v / 2 < JW ? v / 2 : 0] >> (16 * (v & 1)));
          } else {
            gl_unrank<NV>(__ldcg(front + j), n, a.D, bt, a.st, e);
          }
          const Key<KW> m = gl_encode<KW, NV>(a.f, e);
          a.rows_basis[row] = big ? g : ~g;  // ~g: ranks not parked in col (ranked in AC), the join ranks them
          if (stashed && !big) {
            Key<KW> dl;
#pragma unroll
            for (int w = 0; w < KW; ++w) dl.w[w] = s_jd[warp][lane][w];
            key_store<KW>(a.rows_delta, row, dl);
          } else {
            key_store<KW>(a.rows_delta, row, key_sub<KW>(m, key_load<KW>(a.bckey, __ldg(a.boff + g))));
          }
          a.rows_start[row] = Mcur + bl + lp - len;
          bool over = false;
#pragma unroll
          for (int v = 0; v < NV; ++v) {
            if (v < n) {
              const u32 sft = (u32)e[v] - (u32)a.lmexp[(long long)g * n + v];
              over |= (sft + (u32)a.maxe[(long long)g * n + v]) > 0xFFFFu;
              a.cl_shift[(n_cl + q) * n + v] = (u16)sft;
            }
          }
          if (over) atomicOr(a.err, (u32)DEVERR_LANE_OVERFLOW);
          a.cl_basis[n_cl + q] = g;
          a.cl_round[n_cl + q] = (int)rounds + 1;
        }
        bn += __popc(bm);
        bl += ltot;
      }
    }
    if (big) {
      grid.sync();
      if (tr) a.trace[rounds * 6 + 2] = gtimer();
      // C: the new rows' terms -> rank -> absent monomials into newbits
      term_ranges((u32)r, (u32)(r + R), Mcur, Mcur + Mk, [&](u32 i) { return __ldcg(a.rows_start + i); },
                  [&](u32 i, u32 rsi, u32 from, u32 to) {
        const int g = __ldcg(a.rows_basis + i);
        const u32 off = __ldg(a.boff + g), len = __ldg(a.blen + g);
        const Key<KW> dl = key_load_cg<KW>(a.rows_delta, i);
        const u32 t_lo = from - rsi, t_hi = min(len, to - rsi);
        for (u32 tb = t_lo; tb < t_hi; tb += 32 * U) {
          u32 tt[U], rk[U], dw[U];
          Key<KW> kk[U];
#pragma unroll
          for (int q = 0; q < U; ++q) {
            tt[q] = tb + q * 32 + lane;
            if (tt[q] < t_hi) kk[q] = key_load<KW>(a.bckey, (long long)off + tt[q]);
          }
#pragma unroll
          for (int q = 0; q < U; ++q)
            if (tt[q] < t_hi) {
              rk[q] = key_rank<KW>(a.f, bt, a.st, key_add<KW>(kk[q], dl));
              if (rsi + tt[q] < a.M_cap) a.col[rsi + tt[q]] = rk[q];  // parked for the join
            }
#pragma unroll
          for (int q = 0; q < U; ++q)
            dw[q] = tt[q] < t_hi ? (__ldcg(a.dict + (rk[q] >> 5)) | __ldcg(a.newbits + (rk[q] >> 5))) : 0xFFFFFFFFu;
#pragma unroll
          for (int q = 0; q < U; ++q) {
            if (tt[q] >= t_hi) continue;
            const u32 w = rk[q] >> 5, bit = 1u << (rk[q] & 31);
            if (!(dw[q] & bit) && !(atomicOr(a.newbits + w, bit) & bit)) atomicAdd(cur + w / cw, 1u);
          }
        }
      });
      grid.sync();
      if (tr) a.trace[rounds * 6 + 3] = gtimer();
    }
    if (big) cta_bases([&](u32 b) { return __ldcg(cur + b); }, base, total);
    if (total > a.front_cap) {
      flags |= LOOP_OVERFLOW;
      break;
    }
    // D: next frontier from this CTA's chunk; dict |= newbits; newbits = 0
    emit_chunk([&](u32 w) {
      const u32 nb = __ldcg(a.newbits + w);
      if (!nb) return 0u;
      const u32 d = __ldcg(a.dict + w);
      a.dict[w] = d | nb;
      a.newbits[w] = 0;
      return nb & ~d;
    }, base, fnext, false, 1u);
    if (tid == 0) {
      dcount[blockIdx.x] += __ldcg(cur + blockIdx.x);
      nxt[blockIdx.x] = 0;
    }
    r += R;
    n_cl += R;
    Mcur += Mk;
    ++rounds;
    nf = total;
    N += total;
    sel ^= 1;
    if ((long long)N > a.dict_cap) flags |= LOOP_DICT_CAP;
    grid.sync();
    if (tr) a.trace[(rounds - 1) * 6 + 4] = gtimer();
  }
  if (t0th) t_epi = gtimer();
  if (!flags && (N > a.N_cap || Mcur > a.M_cap || r + 1 > a.rows_cap)) flags |= LOOP_OVERFLOW;
  if (!flags) {
    // ---- P3: final dictionary (the map is cleared behind us)
    u32 base, tot;
    cta_bases([&](u32 b) { return __ldcg(dcount + b); }, base, tot);
    // ranks of the final dictionary parked in the first word of each
    // dict_out slot; the same thread turns slot i into the key below
    u32* drank = reinterpret_cast<u32*>(a.dict_out);
    emit_chunk([&](u32 w) {
      const u32 d = __ldcg(a.dict + w);
      if (d) a.dict[w] = 0;
      return d;
    }, base, drank, true, 2u * KW);
    grid.sync();
    stamp(387);
    // final dictionary: keys ascending, exponents in column order (grid-stride,
    // every thread of the grid)
    for (u32 i = blockIdx.x * blockDim.x + tid; i < N; i += G * blockDim.x) {
      const u32 rk = __ldcg(drank + (size_t)i * 2 * KW);
      u16 e[NV];
      gl_unrank<NV>(rk, n, a.D, bt, a.st, e);
      key_store<KW>(a.dict_out, i, gl_encode<KW, NV>(a.f, e));
#pragma unroll
      for (int v = 0; v < NV; ++v)
        if (v < n) a.dict_exps[((long long)N - 1 - i) * n + v] = e[v];
    }
    // ---- P4: join: col = N - 1 - (prefix[rank >> 5] + popc(word & below))
    bool miss = false;
    term_ranges(0u, (u32)r, 0u, Mcur, [&](u32 i) { return __ldcg(a.rows_start + i); },
                [&](u32 i, u32 rsi, u32 from, u32 to) {
      int g = __ldcg(a.rows_basis + i);
      const bool parked = g >= 0;  // ranks parked in col by P1 / a big round's C
      if (!parked) g = ~g;
      const u32 off = __ldg(a.boff + g), len = __ldg(a.blen + g);
      const Key<KW> dl = key_load_cg<KW>(a.rows_delta, i);
      const u32 t_lo = from - rsi, t_hi = min(len, to - rsi);
      for (u32 tb = t_lo; tb < t_hi; tb += 32 * U) {
        u32 tt[U], rk[U], cf[U];
        uint2 dw[U];
        Key<KW> kk[U];
#pragma unroll
        for (int q = 0; q < U; ++q) {
          tt[q] = tb + q * 32 + lane;
          if (tt[q] < t_hi) {
            if (parked) rk[q] = __ldcg(a.col + rsi + tt[q]);
            else kk[q] = key_load<KW>(a.bckey, (long long)off + tt[q]);
            cf[q] = __ldg(a.bcoeff + off + tt[q]);
          }
        }
        if (!parked) {
#pragma unroll
          for (int q = 0; q < U; ++q)
            if (tt[q] < t_hi) rk[q] = key_rank<KW>(a.f, bt, a.st, key_add<KW>(kk[q], dl));
        }
#pragma unroll
        for (int q = 0; q < U; ++q)
          if (tt[q] < t_hi) dw[q] = __ldcg(a.dwp + (rk[q] >> 5));
#pragma unroll
        for (int q = 0; q < U; ++q)
          if (tt[q] < t_hi) {
            const u32 sh = rk[q] & 31;
            if (!((dw[q].x >> sh) & 1u)) miss = true;
            a.col[rsi + tt[q]] = N - 1 - (dw[q].y + __popc(dw[q].x & ((1u << sh) - 1u)));
            a.val[rsi + tt[q]] = cf[q];
          }
      }
    });
    if (miss) atomicOr(a.err, (u32)DEVERR_MISSING_KEY);
  }
  if (t0th) {
    LoopOut o;
    o.r = (u32)r;
    o.n_cl = (u32)n_cl;
    o.M = Mcur;
    o.N = N;
    o.rounds = rounds;
    o.nf = nf;
    o.flags = flags;
    o.sel = (u32)sel;
    o.t_start = t_start;
    o.t_epi = t_epi;
    o.t_end = gtimer();
    *a.out = o;
  }
}

// Join: every term -> rank -> column via the popcount prefix.
template <int KW>
__global__ void __launch_bounds__(RK_THREADS) k_rank_join(KeyFmt f, u32 M, u32 r, const int* __restrict__ rb,
                                                          const u64* __restrict__ delta, const u32* __restrict__ rstart,
                                                          const u32* __restrict__ boff, const u64* __restrict__ bckey,
                                                          const u32* __restrict__ bcoeff, const u32* __restrict__ bt_g,
                                                          int st, int bt_words, const u32* __restrict__ dict_g,
                                                          const u32* __restrict__ wpre_g, u32 words, int use_smem,
                                                          u32 N, u32* __restrict__ col, u32* __restrict__ val,
                                                          u32* err) {
  extern __shared__ __align__(16) unsigned char smraw[];
  Key<KW>* sdel = reinterpret_cast<Key<KW>*>(smraw);
  u32* srs = reinterpret_cast<u32*>(sdel + RK_SROWS);
  u32* sbo = srs + RK_SROWS + 1;
  u32* bt = sbo + RK_SROWS;
  u32* sd = bt + bt_words;
  u32* sp = sd + words;
  __shared__ u32 s_rf, s_nr;
  for (int i = threadIdx.x; i < bt_words; i += blockDim.x) bt[i] = bt_g[i];
  const u32* dict = dict_g;
  const u32* wpre = wpre_g;
  if (use_smem) {
    for (u32 w = threadIdx.x; w < words; w += blockDim.x) {
      sd[w] = dict_g[w];
      sp[w] = wpre_g[w];
    }
    dict = sd;
    wpre = sp;
  }
  __syncthreads();
  bool miss = false;
  const u32 ntiles = (M + RK_TILE - 1) / RK_TILE;
  for (u32 tile = blockIdx.x; tile < ntiles; tile += gridDim.x) {
    const u32 t0 = tile * RK_TILE;
    const u32 n = min((u32)RK_TILE, M - t0);
    if (threadIdx.x == 0) {
      const u32 rf = row_of_term(rstart, 0, r, t0);
      s_rf = rf;
      s_nr = row_of_term(rstart, rf, r, t0 + n - 1) - rf + 1;
    }
    __syncthreads();
    const u32 rf = s_rf, nr = s_nr;
    const bool staged = nr <= (u32)RK_SROWS;
    if (staged) {
      for (u32 i = threadIdx.x; i <= nr; i += blockDim.x) srs[i] = rstart[rf + i];
      for (u32 i = threadIdx.x; i < nr; i += blockDim.x) {
        sbo[i] = boff[rb[rf + i]];
        sdel[i] = key_load<KW>(delta, rf + i);
      }
    }
    __syncthreads();
    for (u32 i = threadIdx.x; i < n; i += blockDim.x) {
      const u32 t = t0 + i;
      u32 row, rs, bo;
      Key<KW> d;
      if (staged) {
        u32 lo = 0, hi = nr;
        while (lo + 1 < hi) {
          const u32 mid = (lo + hi) >> 1;
          if (srs[mid] <= t) lo = mid; else hi = mid;
        }
        rs = srs[lo];
        bo = sbo[lo];
        d = sdel[lo];
      } else {
        row = row_of_term(rstart, rf, r, t);
        rs = rstart[row];
        bo = boff[rb[row]];
        d = key_load<KW>(delta, row);
      }
      const Key<KW> k = key_add<KW>(key_load<KW>(bckey, (long long)bo + (t - rs)), d);
      const u32 rk = key_rank<KW>(f, bt, st, k);
      const u32 word = dict[rk >> 5];
      const u32 below = word & ((1u << (rk & 31)) - 1u);
      if (!((word >> (rk & 31)) & 1u)) miss = true;
      col[t] = N - 1 - (wpre[rk >> 5] + __popc(below));
      val[t] = __ldg(bcoeff + bo + (t - rs));
    }
    __syncthreads();
  }
  if (miss) atomicOr(err, (u32)DEVERR_MISSING_KEY);
}


// Eligibility of the rank path: grevlex and a rank space of <= 2^26 monomials.
static bool rank_path_ok(const Ctx* c, int order, int n, long long D) {
  if (order != 0 || D > 255 || c->opt_dict_sort) return false;
  return binom_ull(n + (int)D, n) <= (1ull << 26);
}

// ===========================================================================
// Fused rank-path compile: ONE cooperative launch runs round 0, every closure
// round, the final dictionary and the join (k_closure_loop with full = 1);
// the host packs its inputs into one page-locked upload and reads the
// counters back once.  Plan buffers are sized from capacity hints; an
// overflow (flagged by the kernel) grows the hints and recompiles.
// ===========================================================================
template <int KW, int NV>
static void compile_rank_fused(Ctx* c, const KeyFmt& f, int D, long long r0, const int32_t* h_rb,
                               const uint16_t* h_shift, int closure, const std::vector<int32_t>& cand,
                               long long dict_cap, f4b_plan* pl) {
  Basis& B = c->basis;
  const int n = c->n_vars;
  c->launches = 0;
  static const bool htrace = getenv("F4B_HOST_TRACE") != nullptr;
  const auto h0 = std::chrono::steady_clock::now();
  std::vector<std::pair<const char*, double>> hmarks;
  auto mark = [&](const char* what) {
    if (htrace)
      hmarks.push_back({what, std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count()});
  };
  cudaEvent_t ev0 = timing_event(c, 0), ev1 = timing_event(c, 1);
  check_cuda(cudaEventRecord(ev0, c->stream), "event record");
  mark("ev0");
  encode_basis<KW>(c, f);
  mark("encode");

  const int st = n + 1;
  const int rows_bt = D + n + 2;
  const int bt_words = rows_bt * st;
  const unsigned long long Rsp = binom_ull(n + D, n);
  const u32 words = (u32)((Rsp + 31) / 32);

  long long M = 0;
  for (long long i = 0; i < r0; ++i) M += B.h_len[h_rb[i]];
  if (M >= (1ll << 30)) fail(F4B_ERR_SIZE_CAP, "batch has more than 2^30 terms");
  const u32 M0 = (u32)M;

  // candidate LMs in preference order (key(LM), index) (symbolic.py:228-235)
  std::vector<int32_t> pref;
  if (closure) pref = preference_order(c, cand);
  mark("pref sort");
  const int nc = closure ? (int)pref.size() : 0;
  const int nw = (n + 1) / 2;
  u32 maxlen = 1;
  for (int32_t k : pref) maxlen = std::max<u32>(maxlen, (u32)B.h_len[k]);

  // one page-locked staging block: binomials | rb | row starts | shifts | LM table | candidate ids
  auto al = [](size_t x) { return (x + 15) & ~(size_t)15; };
  const size_t o_bt = 0, o_rb = o_bt + al((size_t)bt_words * 4), o_st = o_rb + al((size_t)r0 * 4),
               o_sh = o_st + al((size_t)(r0 + 1) * 4), o_lm = o_sh + al((size_t)r0 * n * 2),
               o_ci = o_lm + al((size_t)std::max(nc, 1) * nw * 4), stage_bytes = o_ci + al((size_t)std::max(nc, 1) * 4);
  if (c->h_stage_cap < stage_bytes) {
    if (c->h_stage) cudaFreeHost(c->h_stage);
    c->h_stage = nullptr;
    c->h_stage_cap = 0;
    const size_t cap = std::max<size_t>(stage_bytes + stage_bytes / 2, 1 << 20);
    check_cuda(cudaHostAlloc(&c->h_stage, cap, cudaHostAllocDefault), "cudaHostAlloc stage");
    c->h_stage_cap = cap;
  }
  unsigned char* hs = static_cast<unsigned char*>(c->h_stage);
  {
    // binomials: cached per (rows, n) in the context
    if (c->h_binom_rows != rows_bt || c->h_binom_n != n) {
      c->h_binom.resize((size_t)bt_words);
      for (int x = 0; x < rows_bt; ++x)
        for (int y = 0; y <= n; ++y)
          c->h_binom[(size_t)x * st + y] = (u32)std::min<unsigned long long>(binom_ull(x, y), 0xFFFFFFFFull);
      c->h_binom_rows = rows_bt;
      c->h_binom_n = n;
    }
    memcpy(hs + o_bt, c->h_binom.data(), (size_t)bt_words * 4);
    mark("binom");
    memcpy(hs + o_rb, h_rb, (size_t)r0 * 4);
    u32* hst = reinterpret_cast<u32*>(hs + o_st);
    u32 acc = 0;
    for (long long i = 0; i < r0; ++i) {
      hst[i] = acc;
      acc += (u32)B.h_len[h_rb[i]];
    }
    hst[r0] = acc;
    memcpy(hs + o_sh, h_shift, (size_t)r0 * n * 2);
    // LM table in preference order, from the per-polynomial packed LMs
    // (packed once per appended polynomial)
    if (B.lmw_polys < B.n_polys) {
      B.h_lmw.resize((size_t)B.n_polys * nw, 0u);
      for (int k = B.lmw_polys; k < B.n_polys; ++k) {
        u32* w = &B.h_lmw[(size_t)k * nw];
        for (int v = 0; v < nw; ++v) w[v] = 0;
        for (int v = 0; v < n; ++v) w[v / 2] |= (u32)B.h_lm[(size_t)k * n + v] << (16 * (v & 1));
      }
      B.lmw_polys = B.n_polys;
    }
    u32* hlm = reinterpret_cast<u32*>(hs + o_lm);
    if (!nc) memset(hlm, 0, (size_t)nw * 4);
    for (int q = 0; q < nc; ++q) memcpy(hlm + (size_t)q * nw, &B.h_lmw[(size_t)pref[q] * nw], (size_t)nw * 4);
    if (nc) memcpy(hs + o_ci, pref.data(), (size_t)nc * 4);
  }
  mark("pack");
  ensure(c, c->dstage, stage_bytes);
  check_cuda(cudaMemcpyAsync(c->dstage.p, hs, stage_bytes, cudaMemcpyHostToDevice, c->stream), "h2d stage");
  unsigned char* ds = c->dstage.as<unsigned char>();
  mark("stage packed + h2d");

  // capacities
  const long long cap = (long long)std::min<unsigned long long>(
      Rsp + 1, (unsigned long long)std::max<long long>({1ll << 16, c->closure_cap_hint, 2 * r0}));
  const long long rows_cap = r0 + (closure ? cap : 0) + 1;
  const long long M_cap = std::min<long long>((1ll << 30) + 1, std::max<long long>({3ll * M0 + (1 << 16), c->m_cap_hint}));
  const long long N_cap = (long long)std::min<unsigned long long>(
      Rsp + 1, (unsigned long long)std::max<long long>({1ll << 16, c->n_cap_hint}));
  ensure(c, c->rows_basis, rows_cap * sizeof(int));
  ensure(c, c->rows_delta, rows_cap * KW * sizeof(u64));
  ensure(c, pl->row_ptr, (size_t)(rows_cap + 1) * sizeof(u32));
  ensure(c, pl->col_ind, (size_t)M_cap * sizeof(u32));
  ensure(c, pl->val, (size_t)M_cap * sizeof(u32));
  ensure(c, pl->dict, (size_t)N_cap * KW * sizeof(u64));
  ensure(c, pl->dict_exps, (size_t)N_cap * n * sizeof(u16));
  const long long clc = closure ? cap : 1;
  ensure(c, pl->cl_basis, clc * sizeof(int));
  ensure(c, pl->cl_shift, clc * n * sizeof(u16));
  ensure(c, pl->cl_round, clc * sizeof(int));
  ensure(c, c->front, (size_t)cap * KW * sizeof(u64));
  ensure(c, c->front_new, (size_t)cap * KW * sizeof(u64));
  ensure(c, c->red, (size_t)cap * sizeof(int));
  ensure(c, c->errflag, sizeof(DevCounters) + 4096);
  DevCounters* dc = reinterpret_cast<DevCounters*>(c->errflag.p);
  LoopOut* d_out = reinterpret_cast<LoopOut*>(dc + 1);
  // dc->err is cleared by k_fbsp itself (CTA 0, before its first barrier)

  mark("ensure");
  const int stage_lm = (size_t)nc * nw * 4 <= 48 * 1024 ? 1 : 0;
  // dynamic shared memory rounded up to 8 KB steps: the occupancy query below
  // (tens of microseconds of host time) then runs once per step, not once per
  // call as the LM table grows
  const size_t lsm = ((((size_t)((bt_words + 3) & ~3) + CL_LIST) * 4 + (stage_lm ? (size_t)nc * nw * 4 : 0)) + 8191) &
                     ~(size_t)8191;
  static bool lattr = false;
  if (!lattr) {
    check_cuda(cudaFuncSetAttribute((k_fbsp<KW, NV>), cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024), "attr");
    lattr = true;
  }
  static int bps_by_step[16] = {-1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1, -1};
  const int lstep = (int)std::min<size_t>(15, lsm / 8192);
  if (bps_by_step[lstep] < 0)
    check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps_by_step[lstep], (k_fbsp<KW, NV>), FB_THREADS, lsm),
               "occupancy");
  const int bps_cached = bps_by_step[lstep];
  static const int bps_max = getenv("F4B_LOOP_BPS") ? atoi(getenv("F4B_LOOP_BPS")) : 2;
  // as many CTAs per SM as fit, up to F4B_LOOP_BPS (2): with FB_THREADS =
  // 512 that is one.  F4B_FBSP_SMALL_M0 (experiment knob, default 0 = never)
  // drops batches below that many input terms to one CTA per SM; with
  // 256-thread CTAs this measured 2 % slower over the 38 cyclic-8 batches
  // than two per SM for every batch.  Fewer than one per SM was slower (the
  // closure rounds' search and ranking spread over all warps).
  static const int g_env = getenv("F4B_FBSP_G") ? atoi(getenv("F4B_FBSP_G")) : 0;
  const int G_full = c->num_sms * std::max(1, std::min(bps_cached, bps_max));
  static const unsigned small_m0 = getenv("F4B_FBSP_SMALL_M0") ? (unsigned)atoi(getenv("F4B_FBSP_SMALL_M0")) : 0u;
  const int G = g_env > 0 ? std::min(g_env, G_full) : (M0 < small_m0 ? std::min(c->num_sms, G_full) : G_full);
  const size_t W = (size_t)G * (FB_THREADS / 32);
  ensure(c, c->loop_scratch, (2 * W + 16) * sizeof(u32));
  // presence maps dict | done | newbits: zero on entry (kept zero by the
  // kernel; cleared here after growth or an aborted run)
  const size_t maps_bytes = ((size_t)3 * words + 64) * 4;
  if (c->maps.cap < maps_bytes) c->maps_clean = 0;
  ensure(c, c->maps, maps_bytes);
  if (c->maps_clean < maps_bytes) {
    check_cuda(cudaMemsetAsync(c->maps.p, 0, c->maps.cap, c->stream), "memset maps");
    c->maps_clean = c->maps.cap;
  }
  u32* d_dict = c->maps.as<u32>();
  u32* d_done = d_dict + words;
  u32* d_new = d_done + words;
  // chunk counters: set `parity` for this call (zero), the other set is
  // cleared by the kernel for the next call
  // two sets of per-CTA counters at a fixed stride for any G up to the
  // buffer's: the kernel clears the whole next set, so a change of G between
  // calls needs no memset (only growth does)
  const int Gset = std::max(G, 2 * c->num_sms);
  if (c->fcnt_G < Gset || !c->fcnt.p) {
    ensure(c, c->fcnt, (size_t)8 * Gset * sizeof(u32));
    check_cuda(cudaMemsetAsync(c->fcnt.p, 0, (size_t)8 * Gset * sizeof(u32), c->stream), "memset counters");
    c->fcnt_G = Gset;
    c->fcnt_parity = 0;
  }
  u32* d_cnt = c->fcnt.as<u32>() + (size_t)4 * c->fcnt_G * c->fcnt_parity;
  u32* d_cnt_next = c->fcnt.as<u32>() + (size_t)4 * c->fcnt_G * (1 - c->fcnt_parity);
  c->fcnt_parity ^= 1;
  ensure(c, c->dwp, (size_t)(words + 1) * sizeof(uint2));

  mark("occ+maps");
  FbspArgs fa;
  memset(&fa, 0, sizeof(fa));
  fa.f = f;
  fa.D = D;
  fa.st = st;
  fa.bt_words = bt_words;
  fa.closure = closure;
  fa.nc = nc;
  fa.nw = nw;
  fa.stage_lm = stage_lm;
  {
    // L2 prefetch of the whole basis stream (experiment, F4B_L2_PREFETCH=1):
    // measured 1.7 % slower on the cyclic-8 replays (a batch touches a few
    // reducers, the prefetch pulls every term) and neutral on Katsura-11
    static const bool l2pf = getenv("F4B_L2_PREFETCH") != nullptr;
    const unsigned long long bytes = (unsigned long long)B.n_terms * (KW * 8 + 4);
    fa.prefetch_terms = l2pf && bytes <= (48ull << 20) ? (unsigned long long)B.n_terms : 0ull;
  }
  fa.words = words;
  fa.maxlen = maxlen;
  fa.front_cap = (u32)cap;
  fa.N_cap = (u32)std::min<long long>(N_cap, 0xFFFFFFFFll);
  fa.M_cap = (u32)std::min<long long>(M_cap, 0xFFFFFFFFll);
  fa.M0 = M0;
  fa.r0 = r0;
  fa.rows_cap = rows_cap;
  fa.cl_cap = clc;
  fa.dict_cap = dict_cap;
  fa.bt = reinterpret_cast<const u32*>(ds + o_bt);
  fa.rb_in = reinterpret_cast<const int*>(ds + o_rb);
  fa.start_in = reinterpret_cast<const u32*>(ds + o_st);
  fa.shift_in = reinterpret_cast<const u16*>(ds + o_sh);
  fa.lmw = reinterpret_cast<const u32*>(ds + o_lm);
  fa.cidx = reinterpret_cast<const int*>(ds + o_ci);
  fa.boff = B.off.as<u32>();
  fa.blen = B.len.as<u32>();
  fa.bckey = B.ckey.as<u64>();
  fa.bcoeff = B.coeff.as<u32>();
  fa.lmexp = B.lmexp.as<u16>();
  fa.maxe = B.maxe.as<u16>();
  fa.dict = d_dict;
  fa.done = d_done;
  fa.newbits = d_new;
  fa.dwp = c->dwp.as<uint2>();
  fa.front0 = c->front.as<u64>();
  fa.front1 = c->front_new.as<u64>();
  fa.red = c->red.as<int>();
  fa.tilecnt = c->loop_scratch.as<u32>();
  fa.cnt = d_cnt;
  fa.cnt_next = d_cnt_next;
  fa.cnt_clear = (u32)(4 * c->fcnt_G);
  static const int big_env = getenv("F4B_FBSP_BIG_NF") ? atoi(getenv("F4B_FBSP_BIG_NF")) : 0;  // experiment knob
  fa.big_nf = (u32)std::max(0, big_env);
  fa.rows_basis = c->rows_basis.as<int>();
  fa.rows_delta = c->rows_delta.as<u64>();
  fa.rows_start = pl->row_ptr.as<u32>();
  fa.cl_basis = pl->cl_basis.as<int>();
  fa.cl_shift = pl->cl_shift.as<u16>();
  fa.cl_round = pl->cl_round.as<int>();
  fa.dict_out = pl->dict.as<u64>();
  fa.dict_exps = pl->dict_exps.as<u16>();
  fa.col = pl->col_ind.as<u32>();
  fa.val = pl->val.as<u32>();
  fa.err = &dc->err;
  fa.out = d_out;
  static const bool trace_on = getenv("F4B_LOOP_TRACE") != nullptr;
  DBuf trb;
  if (trace_on) {
    ensure(c, trb, 400 * 8);
    check_cuda(cudaMemsetAsync(trb.p, 0, 400 * 8, c->stream), "memset");
    fa.trace = trb.as<unsigned long long>();
  }
  {
    void* args[] = {&fa};
    ProfScope ps(c, "k_fbsp");
    check_cuda(cudaLaunchCooperativeKernel((void*)(k_fbsp<KW, NV>), G, FB_THREADS, args, lsm, c->stream), "k_fbsp");
  }
  mark("launched");
  check_cuda(cudaEventRecord(ev1, c->stream), "event record");
  // LayoutPlan.validate (symbolic.py:383-387) fused behind the kernel: sizes
  // from LoopOut on the device, its flag read back with the counters
  unsigned long long* vflag = reinterpret_cast<unsigned long long*>(d_out + 1);
  validate_launch_dev(c, pl, reinterpret_cast<const uint32_t*>(d_out), vflag);
  check_cuda(cudaMemcpyAsync(c->h_stat, dc, sizeof(DevCounters) + sizeof(LoopOut) + 8, cudaMemcpyDeviceToHost,
                             c->stream),
             "d2h");
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  mark("synced");
  if (htrace) {
    fprintf(stderr, "[host] r0=%lld M0=%u:", r0, M0);
    for (auto& m : hmarks) fprintf(stderr, " %s @%.1f |", m.first, m.second);
    fprintf(stderr, "\n");
  }
  DevCounters hc;
  LoopOut ho;
  memcpy(&hc, c->h_stat, sizeof(DevCounters));
  memcpy(&ho, reinterpret_cast<unsigned char*>(c->h_stat) + sizeof(DevCounters), sizeof(LoopOut));
  if (trace_on) {
    std::vector<unsigned long long> ht(400);
    check_cuda(cudaMemcpy(ht.data(), trb.p, ht.size() * 8, cudaMemcpyDeviceToHost), "d2h");
    auto us = [&](unsigned long long a1, unsigned long long b1) { return a1 && b1 ? (b1 - a1) / 1e3 : -1.0; };
    fprintf(stderr, "[fused] G=%d nc=%d r0=%lld M0=%u rounds=%u N=%u M=%u | P1 %.1f P2 %.1f | loop %.1f | P3 %.1f P4 %.1f us\n",
            G, nc, r0, M0, ho.rounds, ho.N, ho.M, us(ho.t_start, ht[384]), us(ht[384], ht[385]),
            us(ht[385], ho.t_epi), us(ho.t_epi, ht[387]), us(ht[387], ho.t_end));
    for (u32 q = 0; q < std::min<u32>(ho.rounds + 1, 64); ++q) {
      const unsigned long long* t = &ht[q * 6];
      if (!t[0]) break;
      fprintf(stderr, "[fused]  rnd %u nf=%llu AC=%.1fus BD=%.1fus (B %.1f C %.1f)\n", q, t[5], us(t[0], t[1]),
              us(t[1], t[4]), us(t[1], t[2]), us(t[2], t[3]));
    }
    release(c, trb);
  }
  float ms = 0;
  check_cuda(cudaEventElapsedTime(&ms, ev0, ev1), "elapsed");
  if (ho.flags) {
    // aborted run: maps and counters may be dirty
    c->maps_clean = 0;
    c->fcnt_G = 0;
  }
  if (ho.flags & LOOP_OVERFLOW) {
    c->closure_cap_hint = std::max<long long>(4 * cap, c->closure_cap_hint);
    c->m_cap_hint = std::max<long long>(c->m_cap_hint, std::max<long long>(2 * M_cap, (long long)ho.M + ho.M / 4));
    c->n_cap_hint = std::max<long long>(c->n_cap_hint, std::max<long long>(2 * N_cap, (long long)ho.N + ho.N / 4));
    compile_rank_fused<KW, NV>(c, f, D, r0, h_rb, h_shift, closure, cand, dict_cap, pl);
    return;
  }
  if (ho.flags & LOOP_SIZE_CAP) fail(F4B_ERR_SIZE_CAP, "batch has more than 2^30 terms");
  if (ho.flags & LOOP_DICT_CAP)
    fail(F4B_ERR_SIZE_CAP, "dictionary exceeded the cap after " + std::to_string(ho.rounds) + " closure rounds");
  if (hc.err & DEVERR_LANE_OVERFLOW) fail(F4B_ERR_LANE_OVERFLOW, "shifted exponent overflows a 16-bit lane");
  if (hc.err & DEVERR_MISSING_KEY) fail(F4B_ERR_MISSING_KEY, "row key absent from dictionary (closure defect)");
  // remember the sizes so later batches rarely overflow
  c->m_cap_hint = std::max<long long>(c->m_cap_hint, (long long)ho.M + ho.M / 4);
  c->n_cap_hint = std::max<long long>(c->n_cap_hint, (long long)ho.N + ho.N / 4);
  pl->KW = KW;
  pl->lane_bits = f.lane_bits;
  pl->r = ho.r;
  pl->r0 = r0;
  pl->N = ho.N;
  pl->M = ho.M;
  pl->closure_rounds = ho.rounds;
  pl->sort_passes = 0;
  const double asm_ns = ho.t_end > ho.t_epi ? (double)(ho.t_end - ho.t_epi) : 0.0;
  pl->asm_ns = (int64_t)asm_ns;
  pl->dict_ns = (int64_t)std::max(0.0, ms * 1e6 - asm_ns);
  pl->launches = c->launches;
  unsigned long long vf;
  memcpy(&vf, reinterpret_cast<unsigned char*>(c->h_stat) + sizeof(DevCounters) + sizeof(LoopOut), 8);
  if (vf != ~0ull) fail(F4B_ERR_PROPERTY, validate_message(vf, pl->row_lo));
  pl->validated = true;
}

template <int KW>
static void compile_rank(Ctx* c, const KeyFmt& f, int D, long long r0, const int32_t* h_rb, const uint16_t* h_shift,
                         int closure, const std::vector<int32_t>& cand, long long dict_cap, f4b_plan* pl) {
  Basis& B = c->basis;
  const int n = c->n_vars;
  c->launches = 0;
  static const bool htrace = getenv("F4B_HOST_TRACE") != nullptr;
  const auto h0 = std::chrono::steady_clock::now();
  std::vector<std::pair<const char*, double>> hmarks;
  auto mark = [&](const char* what) {
    if (htrace)
      hmarks.push_back({what, std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - h0).count()});
  };
  cudaEvent_t ev0, ev1, ev2;
  check_cuda(cudaEventCreate(&ev0), "event");
  check_cuda(cudaEventCreate(&ev1), "event");
  check_cuda(cudaEventCreate(&ev2), "event");
  check_cuda(cudaEventRecord(ev0, c->stream), "event record");
  encode_basis<KW>(c, f);

  // binomial table C(a, b), a <= D + n + 1, b <= n
  const int st = n + 1;
  const int rows_bt = D + n + 2;
  const int bt_words = rows_bt * st;
  std::vector<u32> hbt((size_t)bt_words, 0u);
  for (int a = 0; a < rows_bt; ++a)
    for (int b = 0; b <= n; ++b) hbt[(size_t)a * st + b] = (u32)std::min<unsigned long long>(binom_ull(a, b), 0xFFFFFFFFull);
  const unsigned long long Rsp = binom_ull(n + D, n);
  const u32 words = (u32)((Rsp + 31) / 32);

  std::vector<uint32_t> h_start(r0 + 1);
  long long M = 0;
  for (long long i = 0; i < r0; ++i) {
    h_start[i] = (uint32_t)M;
    M += B.h_len[h_rb[i]];
  }
  h_start[r0] = (uint32_t)M;
  if (M >= (1ll << 30)) fail(F4B_ERR_SIZE_CAP, "batch has more than 2^30 terms");
  const u32 M0 = (u32)M;

  // buffers: counters+lookback | bt | dict | aux (done / newbits) | wprefix | partials
  const size_t fill_smem_bits = (size_t)words * 4;
  const int use_smem = fill_smem_bits <= 96 * 1024 ? 1 : 0;
  const size_t fill_smem = (size_t)RK_SROWS * (KW * 8 + 8) + 16 + (size_t)bt_words * 4 + (use_smem ? fill_smem_bits : 0);
  const int per_sm = use_smem ? (int)std::max<size_t>(1, std::min<size_t>(4, (220 * 1024) / (fill_smem + 4096))) : 4;
  const int max_grid = c->num_sms * per_sm;
  ensure(c, c->errflag, sizeof(DevCounters) + 4096);
  DevCounters* dc = reinterpret_cast<DevCounters*>(c->errflag.p);
  check_cuda(cudaMemsetAsync(dc, 0, sizeof(DevCounters), c->stream), "memset counters");
  // look-back status regions: A/B for k_new_rows (<= N/256 tiles), C for k_rank_extract
  const size_t lbAB = (size_t)words / 2 + 64, lbC = (size_t)words / 256 + 64;
  ensure(c, c->dict_b, ((size_t)bt_words + 3 * (size_t)words + 2 * lbAB + lbC + 64) * 4);
  u32* base = c->dict_b.as<u32>();
  u32* d_bt = base;
  u32* d_dict = d_bt + bt_words;
  u32* d_aux = d_dict + words;
  u32* d_wpre = d_aux + words;
  u32* d_lbA = d_wpre + words + 1;
  u32* d_lbB = d_lbA + lbAB;
  u32* d_lbC = d_lbB + lbAB;
  check_cuda(cudaMemcpyAsync(d_bt, hbt.data(), (size_t)bt_words * 4, cudaMemcpyHostToDevice, c->stream), "h2d binom");
  auto zero_lb = [&]() {
    check_cuda(cudaMemsetAsync(dc->tickets, 0, sizeof(dc->tickets), c->stream), "memset tickets");
    check_cuda(cudaMemsetAsync(d_lbA, 0, (2 * lbAB + lbC) * 4, c->stream), "memset lb");
  };

  // rows of round 0
  long long rcap = std::max<long long>(2 * r0 + 1024, 4096);
  ensure(c, c->rows_basis, rcap * sizeof(int));
  ensure(c, c->rows_delta, rcap * KW * sizeof(u64));
  ensure(c, c->rows_len, rcap * sizeof(u32));
  ensure(c, c->rows_start, (rcap + 1) * sizeof(u32));
  ensure(c, c->shift_in, (size_t)std::max<long long>(r0, 1) * n * sizeof(u16));
  check_cuda(cudaMemcpyAsync(c->rows_basis.p, h_rb, r0 * sizeof(int), cudaMemcpyHostToDevice, c->stream), "h2d rows");
  check_cuda(cudaMemcpyAsync(c->shift_in.p, h_shift, r0 * n * sizeof(u16), cudaMemcpyHostToDevice, c->stream), "h2d");
  check_cuda(cudaMemcpyAsync(c->rows_start.p, h_start.data(), (r0 + 1) * sizeof(u32), cudaMemcpyHostToDevice,
                             c->stream), "h2d starts");
  F4B_LAUNCH(c, k_rows0<KW>, nblk(r0, 256), 256, 0, f, r0, c->rows_basis.as<int>(), c->shift_in.as<u16>(),
             B.len.as<u32>(), c->rows_delta.as<u64>(), c->rows_len.as<u32>());
  mark("rows h2d + rows0");
  static bool attr = false;
  if (!attr) {
    check_cuda(cudaFuncSetAttribute(k_rank_fill<KW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024), "attr");
    check_cuda(cudaFuncSetAttribute(k_rank_join<KW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024), "attr");
    check_cuda(cudaFuncSetAttribute(k_rank_extract<KW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 64 * 1024),
               "attr");
    check_cuda(cudaFuncSetAttribute(k_rank_round<KW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024),
               "attr");
    attr = true;
  }
  // known == nullptr: round 0 (private partials when they fit);
  // known == dict: closure round, absent monomials only, one global map.
  auto fill = [&](u32 m_lo, u32 m_hi, u32 m_bound, const u32* d_mk, u32 r_lo, u32 r_hi, const u32* d_r,
                  const u32* known) -> int {
    const int sm = known ? 0 : use_smem;
    const u32 tiles = std::max<u32>(1, (m_bound + RK_TILE - 1) / RK_TILE);
    const int grid = (int)std::min<long long>(tiles, sm ? std::min(max_grid, 2 * c->num_sms) : 4 * c->num_sms);
    const int nparts = 1;
    ensure(c, c->uniq, (size_t)words * 4 + 16);
    check_cuda(cudaMemsetAsync(c->uniq.p, 0, (size_t)words * 4, c->stream), "memset bits");
    F4B_LAUNCH(c, k_rank_fill<KW>, grid, RK_THREADS, sm ? fill_smem : fill_smem - (use_smem ? fill_smem_bits : 0), f,
               m_lo, m_hi, d_mk, r_lo, r_hi, d_r, c->rows_basis.as<int>(), c->rows_delta.as<u64>(),
               c->rows_start.as<u32>(), B.off.as<u32>(), B.ckey.as<u64>(), d_bt, st, bt_words, words, sm,
               c->uniq.as<u32>(), known);
    return nparts;
  };
  const size_t ex_smem = (size_t)bt_words * 4;
  // (caller zeroes region C and ticket 3 first)
  // set bits of A & ~Bm -> rank list (ascending) -> device keys (+ exponents)
  ensure(c, c->tmp_u32c, ((size_t)std::min<unsigned long long>(Rsp, (unsigned long long)M0 + (1ull << 22)) + 16) * 4);
  auto extract = [&](const u32* A, const u32* Bm, int mode, u64* out_keys, u16* out_exps, u32 N_final, u32* d_count) {
    (void)N_final;
    const u32 tiles = std::max<u32>(1, (words + 1023) / 1024);
    F4B_LAUNCH(c, k_rank_extract<KW>, tiles, 256, 0, f, A, Bm, words, mode, d_bt, st, 0, c->tmp_u32c.as<u32>(), d_wpre,
               d_lbC, &dc->tickets[3], d_count);
    F4B_LAUNCH(c, k_rank_unrank<KW>, c->num_sms * 2, 256, ex_smem, f, c->tmp_u32c.as<u32>(), d_count, d_bt, st,
               bt_words, D, out_keys, out_exps);
  };

  zero_lb();
  check_cuda(cudaMemsetAsync(&dc->N, 0, 4, c->stream), "memset");
  // leads of the input rows are covered (symbolic.py:339): "done" bitmap
  check_cuda(cudaMemsetAsync(d_aux, closure ? 0 : 0xFF, (size_t)words * 4, c->stream), "memset done");
  if (closure)
    F4B_LAUNCH(c, k_rank_leads<KW>, nblk(r0, 256), 256, 0, f, r0, c->rows_basis.as<int>(), c->rows_delta.as<u64>(),
               B.off.as<u32>(), B.ckey.as<u64>(), d_bt, st, d_aux);
  int nparts = fill(0, M0, M0, nullptr, 0, (u32)r0, nullptr, nullptr);
  ensure(c, c->front, (size_t)(std::min<unsigned long long>(Rsp, M0) + 1) * KW * sizeof(u64));
  const size_t rr_smem = ((size_t)bt_words + RX_LIST) * 4;
  const u32 rr_tiles = std::max<u32>(1, (words + 256 * RX_WPT - 1) / (256 * RX_WPT));
  // dictionary (= OR of the partials), its size, and the round-1 frontier
  F4B_LAUNCH(c, k_rank_round<KW>, rr_tiles, 256, rr_smem, f, c->uniq.as<u32>(), nparts, words, 0, d_dict, d_aux, d_bt,
             st, bt_words, D, c->front.as<u64>(), d_lbC, &dc->tickets[3], &dc->nf, &dc->N);
  long long r = r0, rounds = 0, n_cl = 0, N = 0;
  mark("fill + round0 launched");
  DevCounters hc;
  if (closure) {
    // candidate LMs in preference order (key(LM), index) (symbolic.py:228-235)
    std::vector<int32_t> pref(cand);
    std::stable_sort(pref.begin(), pref.end(), [&](int32_t x, int32_t y) {
      int s = mon_cmp(&B.h_lm[(size_t)x * n], &B.h_lm[(size_t)y * n], n, c->order);
      return s != 0 ? s < 0 : x < y;
    });
    const int nc = (int)pref.size();
    const int nw = (n + 1) / 2;
    std::vector<uint32_t> h_lmw((size_t)std::max(nc, 1) * nw, 0u);
    for (int q = 0; q < nc; ++q)
      for (int v = 0; v < n; ++v)
        h_lmw[(size_t)q * nw + v / 2] |= (uint32_t)B.h_lm[(size_t)pref[q] * n + v] << (16 * (v & 1));
    ensure(c, c->lmpref, h_lmw.size() * sizeof(u32));
    ensure(c, c->cand_idx, (size_t)std::max(nc, 1) * sizeof(int));
    check_cuda(cudaMemcpyAsync(c->lmpref.p, h_lmw.data(), h_lmw.size() * sizeof(u32), cudaMemcpyHostToDevice,
                               c->stream), "h2d lm");
    if (nc)
      check_cuda(cudaMemcpyAsync(c->cand_idx.p, pref.data(), nc * sizeof(int), cudaMemcpyHostToDevice, c->stream),
                 "h2d cand");
    mark("LM pref sorted + h2d");
    if (!getenv("F4B_CLOSURE_ROUNDS")) {
      // persistent closure loop: one cooperative launch for every round
      const long long cap = (long long)std::min<unsigned long long>(
          Rsp + 1, (unsigned long long)std::max<long long>({1ll << 16, c->closure_cap_hint, 2 * r0}));
      const long long rows_cap = r0 + cap + 1;
      if (rows_cap > rcap) {
        rcap = rows_cap;
        ensure_keep(c, c->rows_basis, rcap * sizeof(int));
        ensure_keep(c, c->rows_delta, rcap * KW * sizeof(u64));
        ensure_keep(c, c->rows_len, rcap * sizeof(u32));
        ensure_keep(c, c->rows_start, (rcap + 1) * sizeof(u32));
      }
      ensure(c, c->cl_basis, cap * sizeof(int));
      ensure(c, c->cl_shift, cap * n * sizeof(u16));
      ensure(c, c->cl_round, cap * sizeof(int));
      ensure_keep(c, c->front, (size_t)(std::max<unsigned long long>(cap, std::min<unsigned long long>(Rsp, M0) + 1)) *
                                   KW * sizeof(u64));
      ensure(c, c->front_new, (size_t)cap * KW * sizeof(u64));
      ensure(c, c->red, (size_t)cap * sizeof(int));
      const int stage_lm = (size_t)nc * nw * 4 <= 48 * 1024 ? 1 : 0;
      const size_t lsm = ((size_t)bt_words + CL_LIST) * 4 + (stage_lm ? (size_t)nc * nw * 4 : 0);
      static bool lattr = false;
      if (!lattr) {
        check_cuda(cudaFuncSetAttribute(k_closure_loop<KW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 96 * 1024),
                   "attr");
        lattr = true;
      }
      int bps = 0;
      check_cuda(cudaOccupancyMaxActiveBlocksPerMultiprocessor(&bps, k_closure_loop<KW>, CL_THREADS, lsm), "occupancy");
      static const int bps_max = getenv("F4B_LOOP_BPS") ? atoi(getenv("F4B_LOOP_BPS")) : 2;
      const int G = c->num_sms * std::max(1, std::min(bps, bps_max));
      const size_t ntile_cap = (size_t)G * (CL_THREADS / 32);
      ensure(c, c->loop_scratch, (2 * ntile_cap + G + 16) * sizeof(u32));
      LoopOut* d_out = reinterpret_cast<LoopOut*>(dc + 1);
      check_cuda(cudaMemsetAsync(d_aux, 0, (size_t)words * 4, c->stream), "memset newbits");
      LoopArgs la;
      memset(&la, 0, sizeof(la));
      la.f = f;
      la.D = D;
      la.st = st;
      la.bt_words = bt_words;
      la.words = words;
      la.bt = d_bt;
      la.dict = d_dict;
      la.newbits = d_aux;
      la.front0 = c->front.as<u64>();
      la.front1 = c->front_new.as<u64>();
      la.front_cap = (u32)cap;
      la.red = c->red.as<int>();
      la.tilecnt = c->loop_scratch.as<u32>();
      la.chunkcnt = la.tilecnt + 2 * ntile_cap;
      la.lmw = c->lmpref.as<u32>();
      la.cidx = c->cand_idx.as<int>();
      la.nc = nc;
      la.nw = nw;
      la.stage_lm = stage_lm;
      la.boff = B.off.as<u32>();
      la.blen = B.len.as<u32>();
      la.bckey = B.ckey.as<u64>();
      la.lmexp = B.lmexp.as<u16>();
      la.maxe = B.maxe.as<u16>();
      la.rows_basis = c->rows_basis.as<int>();
      la.rows_delta = c->rows_delta.as<u64>();
      la.rows_start = c->rows_start.as<u32>();
      la.rows_cap = rcap;
      la.cl_basis = c->cl_basis.as<int>();
      la.cl_shift = c->cl_shift.as<u16>();
      la.cl_round = c->cl_round.as<int>();
      la.cl_cap = cap;
      la.r0 = r0;
      la.M0 = M0;
      u32 maxlen_c = 1;
      for (int32_t k : pref) maxlen_c = std::max<u32>(maxlen_c, (u32)B.h_len[k]);
      la.maxlen = maxlen_c;
      la.dict_cap = dict_cap;
      la.d_nf0 = &dc->nf;
      la.d_N0 = &dc->N;
      la.err = &dc->err;
      la.out = d_out;
      static const bool trace_on = getenv("F4B_LOOP_TRACE") != nullptr;
      DBuf trb;
      la.trace = nullptr;
      if (trace_on) {
        ensure(c, trb, 64 * 6 * 8);
        check_cuda(cudaMemsetAsync(trb.p, 0, 64 * 6 * 8, c->stream), "memset");
        la.trace = trb.as<unsigned long long>();
      }
      {
        void* args[] = {&la};
        ProfScope ps(c, "k_closure_loop");
        check_cuda(cudaLaunchCooperativeKernel((void*)k_closure_loop<KW>, G, CL_THREADS, args, lsm, c->stream),
                   "k_closure_loop");
      }
      mark("loop launched");
      LoopOut ho;
      check_cuda(cudaMemcpyAsync(c->h_stat, d_out, sizeof(LoopOut), cudaMemcpyDeviceToHost, c->stream), "d2h");
      check_cuda(cudaStreamSynchronize(c->stream), "sync");
      memcpy(&ho, c->h_stat, sizeof(LoopOut));
      mark("loop synced");
      if (trace_on) {
        std::vector<unsigned long long> ht(64 * 6);
        check_cuda(cudaMemcpy(ht.data(), trb.p, ht.size() * 8, cudaMemcpyDeviceToHost), "d2h");
        fprintf(stderr, "[loop] G=%d nc=%d rounds=%u N=%u\n", G, nc, ho.rounds, ho.N);
        for (u32 q = 0; q < std::min<u32>(ho.rounds + 1, 64); ++q) {
          const unsigned long long* t = &ht[q * 6];
          if (!t[0]) break;
          fprintf(stderr, "[loop]  round %u nf=%llu A=%.1fus B=%.1fus D1=%.1fus D2=%.1fus\n", q, t[5],
                  t[1] ? (t[1] - t[0]) / 1e3 : 0.0, t[2] ? (t[2] - t[1]) / 1e3 : 0.0, t[3] ? (t[3] - t[2]) / 1e3 : 0.0,
                  t[4] ? (t[4] - t[3]) / 1e3 : 0.0);
        }
        release(c, trb);
      }
      if (ho.flags & LOOP_OVERFLOW) {
        // frontier / closure rows outgrew the buffers: grow and recompile
        c->closure_cap_hint = std::max<long long>(4 * cap, c->closure_cap_hint);
        cudaEventDestroy(ev0);
        cudaEventDestroy(ev1);
        cudaEventDestroy(ev2);
        compile_rank<KW>(c, f, D, r0, h_rb, h_shift, closure, cand, dict_cap, pl);
        return;
      }
      if (ho.flags & LOOP_SIZE_CAP) fail(F4B_ERR_SIZE_CAP, "batch has more than 2^30 terms");
      if (ho.flags & LOOP_DICT_CAP)
        fail(F4B_ERR_SIZE_CAP, "dictionary exceeded the cap after " + std::to_string(ho.rounds) + " closure rounds");
      r = ho.r;
      n_cl = ho.n_cl;
      M = ho.M;
      N = ho.N;
      rounds = ho.rounds;
    } else {
    read_counters(c, dc, &hc);
    N = hc.N;
    long long nf = hc.nf;
    long long clcap = std::max<long long>(N + 1024, 4096);
    ensure(c, c->cl_basis, clcap * sizeof(int));
    ensure(c, c->cl_shift, clcap * n * sizeof(u16));
    ensure(c, c->cl_round, clcap * sizeof(int));
    u32 Mcur = M0;
    long long maxlen = 1;
    for (int32_t k : pref) maxlen = std::max<long long>(maxlen, B.h_len[k]);
    while (nf > 0 && nc > 0) {
      const long long mk_bound = std::max<long long>(1, std::min<long long>(nf * maxlen, (1ll << 30) - Mcur));
      if (r + nf + 2 > rcap) {
        rcap = 2 * (r + nf + 2);
        ensure_keep(c, c->rows_basis, rcap * sizeof(int));
        ensure_keep(c, c->rows_delta, rcap * KW * sizeof(u64));
        ensure_keep(c, c->rows_len, rcap * sizeof(u32));
        ensure_keep(c, c->rows_start, (rcap + 1) * sizeof(u32));
      }
      if (n_cl + nf > clcap) {
        clcap = 2 * (n_cl + nf);
        ensure_keep(c, c->cl_basis, clcap * sizeof(int));
        ensure_keep(c, c->cl_shift, clcap * n * sizeof(u16));
        ensure_keep(c, c->cl_round, clcap * sizeof(int));
      }
      ensure(c, c->red, (size_t)nf * sizeof(int));
      ensure(c, c->front_new, (size_t)(std::min<unsigned long long>(Rsp, (unsigned long long)mk_bound) + 1) * KW *
                                  sizeof(u64));
      zero_lb();
      const int stage_lm = (size_t)nc * nw * 4 <= 48 * 1024 ? 1 : 0;
      F4B_LAUNCH(c, k_closure_rows<KW>, std::max<long long>(1, (nf + CR_TILE - 1) / CR_TILE), 256,
                 stage_lm ? (size_t)nc * nw * 4 : 0, f, c->front.as<u64>(), &dc->nf, c->lmpref.as<u32>(),
                 c->cand_idx.as<int>(), nc, nw, stage_lm, r, n_cl, Mcur, B.off.as<u32>(), B.len.as<u32>(),
                 B.ckey.as<u64>(), B.lmexp.as<u16>(), B.maxe.as<u16>(), (int)rounds + 1, c->rows_basis.as<int>(),
                 c->rows_delta.as<u64>(), c->rows_start.as<u32>(), c->cl_basis.as<int>(), c->cl_shift.as<u16>(),
                 c->cl_round.as<int>(), d_lbA, d_lbB, &dc->tickets[2], &dc->R, &dc->Mk, &dc->err);
      nparts = fill(Mcur, 0, (u32)mk_bound, &dc->Mk, (u32)r, 0, &dc->R, d_dict);
      F4B_LAUNCH(c, k_rank_round<KW>, rr_tiles, 256, rr_smem, f, c->uniq.as<u32>(), nparts, words, 1, d_dict, nullptr,
                 d_bt, st, bt_words, D, c->front_new.as<u64>(), d_lbC, &dc->tickets[3], &dc->nf, &dc->N);
      read_counters(c, dc, &hc);
      const long long R = hc.R, Mk = hc.Mk;
      if (R == 0) break;
      if ((long long)Mcur + Mk >= (1ll << 30)) fail(F4B_ERR_SIZE_CAP, "batch has more than 2^30 terms");
      ++rounds;
      std::swap(c->front, c->front_new);
      nf = hc.nf;
      N += nf;
      M += Mk;
      Mcur += (u32)Mk;
      r += R;
      n_cl += R;
      if (N > dict_cap)
        fail(F4B_ERR_SIZE_CAP, "dictionary exceeded the cap after " + std::to_string(rounds) + " closure rounds");
    }
    }
  } else {
    read_counters(c, dc, &hc);
    N = hc.N;
  }
  check_cuda(cudaEventRecord(ev1, c->stream), "event record");

  // ---- row assembly ------------------------------------------------------
  pl->KW = KW;
  pl->lane_bits = f.lane_bits;
  pl->r = r;
  pl->r0 = r0;
  pl->N = N;
  pl->M = M;
  pl->closure_rounds = rounds;
  pl->sort_passes = 0;
  ensure(c, pl->row_ptr, (size_t)(r + 1) * sizeof(u32));
  ensure(c, pl->col_ind, (size_t)std::max<long long>(M, 1) * sizeof(u32));
  ensure(c, pl->val, (size_t)std::max<long long>(M, 1) * sizeof(u32));
  ensure(c, pl->dict, (size_t)std::max<long long>(N, 1) * KW * sizeof(u64));
  ensure(c, pl->dict_exps, (size_t)std::max<long long>(N, 1) * n * sizeof(u16));
  ensure(c, pl->cl_basis, (size_t)std::max<long long>(n_cl, 1) * sizeof(int));
  ensure(c, pl->cl_shift, (size_t)std::max<long long>(n_cl, 1) * n * sizeof(u16));
  ensure(c, pl->cl_round, (size_t)std::max<long long>(n_cl, 1) * sizeof(int));
  check_cuda(cudaMemcpyAsync(pl->row_ptr.p, c->rows_start.p, (r + 1) * sizeof(u32), cudaMemcpyDeviceToDevice,
                             c->stream), "d2d row_ptr");
  if (n_cl) {
    check_cuda(cudaMemcpyAsync(pl->cl_basis.p, c->cl_basis.p, n_cl * sizeof(int), cudaMemcpyDeviceToDevice, c->stream),
               "d2d");
    check_cuda(cudaMemcpyAsync(pl->cl_shift.p, c->cl_shift.p, n_cl * n * sizeof(u16), cudaMemcpyDeviceToDevice,
                               c->stream), "d2d");
    check_cuda(cudaMemcpyAsync(pl->cl_round.p, c->cl_round.p, n_cl * sizeof(int), cudaMemcpyDeviceToDevice, c->stream),
               "d2d");
  }
  // final dictionary: keys ascending, exponents in column order, word prefix
  zero_lb();
  extract(d_dict, nullptr, 1, pl->dict.as<u64>(), pl->dict_exps.as<u16>(), (u32)N, &dc->U);
  if (M) {
    const size_t js = (size_t)RK_SROWS * (KW * 8 + 8) + 16 + (size_t)bt_words * 4;
    const int use_s = js + (size_t)words * 8 <= 200 * 1024 ? 1 : 0;
    const size_t jsmem = js + (use_s ? (size_t)words * 8 : 0);
    const int jper = (int)std::max<size_t>(1, std::min<size_t>(4, (220 * 1024) / (jsmem + 4096)));
    const int grid = (int)std::min<long long>(nblk(M, RK_TILE), (long long)c->num_sms * jper);
    F4B_LAUNCH(c, k_rank_join<KW>, grid, RK_THREADS, jsmem, f, (u32)M, (u32)r, c->rows_basis.as<int>(),
               c->rows_delta.as<u64>(), c->rows_start.as<u32>(), B.off.as<u32>(), B.ckey.as<u64>(),
               B.coeff.as<u32>(), d_bt, st, bt_words, d_dict, d_wpre, words, use_s, (u32)N, pl->col_ind.as<u32>(),
               pl->val.as<u32>(), &dc->err);
  }
  check_cuda(cudaEventRecord(ev2, c->stream), "event record");
  mark("join launched");
  read_counters(c, dc, &hc);
  float ms1 = 0, ms2 = 0;
  check_cuda(cudaEventElapsedTime(&ms1, ev0, ev1), "elapsed");
  check_cuda(cudaEventElapsedTime(&ms2, ev1, ev2), "elapsed");
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  cudaEventDestroy(ev2);
  mark("final sync");
  if (htrace) {
    fprintf(stderr, "[host] r0=%lld M=%lld:", r0, (long long)M);
    for (auto& m : hmarks) fprintf(stderr, " %s @%.1f |", m.first, m.second);
    fprintf(stderr, " dev dict %.1fus asm %.1fus\n", ms1 * 1e3, ms2 * 1e3);
  }
  pl->dict_ns = (int64_t)(ms1 * 1e6);
  pl->asm_ns = (int64_t)(ms2 * 1e6);
  pl->launches = c->launches;
  if (hc.U != (u32)N) fail(F4B_ERR_PROPERTY, "dictionary extraction count mismatch");
  if (hc.err & DEVERR_LANE_OVERFLOW) fail(F4B_ERR_LANE_OVERFLOW, "shifted exponent overflows a 16-bit lane");
  if (hc.err & DEVERR_MISSING_KEY) fail(F4B_ERR_MISSING_KEY, "row key absent from dictionary (closure defect)");
}

BatchFormat batch_format(Ctx* c, long long r0, const int32_t* rb, const uint16_t* shift, const int32_t* cands,
                         long long n_cands) {
  Basis& B = c->basis;
  const int n = c->n_vars;
  BatchFormat bf;
  long long D = 0;
  for (long long i = 0; i < r0; ++i) {
    const int g = rb[i];
    if (g < 0 || g >= B.n_polys) fail(F4B_ERR_PRECONDITION, "row references unknown basis index");
    if (B.h_len[g] < 1) fail(F4B_ERR_PROPERTY, "zero polynomial referenced as a reducer");
    long long d = 0;
    for (int v = 0; v < n; ++v) {
      const long long s = shift[i * n + v];
      if (s + B.h_maxe[(size_t)g * n + v] > 0xFFFF) {
        // h_maxe may still hold the deg(LM) bounds of a pending key append:
        // decide on the exact maximum exponents
        if (c->pend.active && c->pend.applied) {
          basis_finish(c);
          return batch_format(c, r0, rb, shift, cands, n_cands);
        }
        fail(F4B_ERR_LANE_OVERFLOW, "shifted exponent overflows a 16-bit lane");
      }
      d += s + B.h_lm[(size_t)g * n + v];
    }
    D = std::max(D, d);
  }
  bf.D = D;
  std::vector<int32_t>& cand = bf.cand;
  if (cands) {
    cand.assign(cands, cands + n_cands);
    for (int32_t k : cand)
      if (k < 0 || k >= B.n_polys) fail(F4B_ERR_PRECONDITION, "candidate references unknown basis index");
  } else {
    cand.resize(B.n_polys);
    for (int k = 0; k < B.n_polys; ++k) cand[k] = k;
  }
  cand.erase(std::remove_if(cand.begin(), cand.end(), [&](int32_t k) { return B.h_len[k] < 1; }), cand.end());
  KeyFmt& f = bf.f;
  f.order = c->order;
  f.n_vars = n;
  if (c->order == 2) {
    f.lane_bits = 16;
  } else {
    int b = 1;
    while ((1ll << b) <= D) ++b;
    f.lane_bits = b;
  }
  f.n_lanes = n;
  auto words_for = [&](int lane_bits) {
    int w = 1;
    while (64 * w < lane_bits * n) w *= 2;
    return w;
  };
  bf.KW = words_for(f.lane_bits);
  // never narrow the lanes of the cached basis keys when the wider format
  // needs no more words: any lane width >= bits(D) is order-isomorphic and
  // injective on the batch, and a narrower format would re-encode the whole
  // basis (k_encode_basis over every term) for nothing
  // (rank path only: the radix path sorts lane_bits * n bits)
  bf.rank_ok = rank_path_ok(c, c->order, n, D) && bf.KW <= 2;
  if (bf.rank_ok && B.ckey_lane_bits > f.lane_bits && B.ckey_lane_bits <= 16 && words_for(B.ckey_lane_bits) == bf.KW)
    f.lane_bits = B.ckey_lane_bits;
  if (bf.KW > 8) fail(F4B_ERR_PRECONDITION, "batch degree too large for the device key format");
  return bf;
}

bool rank_path_ok_pub(const Ctx* c, int order, int n, long long D) { return rank_path_ok(c, order, n, D); }

// The lane check of batch_format against the exact maximum exponents (after
// a compile that ran on the deg(LM) bounds of a pending key append).
void recheck_lanes(Ctx* c, long long r0, const int32_t* rb, const uint16_t* shift) {
  const Basis& B = c->basis;
  const int n = c->n_vars;
  for (long long i = 0; i < r0; ++i)
    for (int v = 0; v < n; ++v)
      if ((long long)shift[i * n + v] + B.h_maxe[(size_t)rb[i] * n + v] > 0xFFFF)
        fail(F4B_ERR_LANE_OVERFLOW, "shifted exponent overflows a 16-bit lane");
}

void encode_basis_kw(Ctx* c, const KeyFmt& f, int KW) {
  switch (KW) {
    case 1: encode_basis<1>(c, f); break;
    case 2: encode_basis<2>(c, f); break;
    case 4: encode_basis<4>(c, f); break;
    default: encode_basis<8>(c, f); break;
  }
}

std::vector<int32_t> reducer_preference(Ctx* c, const std::vector<int32_t>& cand) { return preference_order(c, cand); }

void compile_batch(Ctx* c, long long r0, const int32_t* rb, const uint16_t* shift, int closure, const int32_t* cands,
                   long long n_cands, long long dict_cap, f4b_plan* pl) {
  const int n = c->n_vars;
  BatchFormat bf = batch_format(c, r0, rb, shift, cands, n_cands);
  const long long D = bf.D;
  const KeyFmt& f = bf.f;
  const int KW = bf.KW;
  const std::vector<int32_t>& cand = bf.cand;
  const bool rank_ok = bf.rank_ok;
  if (rank_ok) {
    // opt_fbsp = 1: the multi-launch pipeline (the same phases as separate
    // launches; also the building blocks of the sharded compile, shard.cu)
    if (c->opt_fbsp == 1) {
      switch (KW) {
        case 1: compile_rank<1>(c, f, (int)D, r0, rb, shift, closure, cand, dict_cap, pl); break;
        case 2: compile_rank<2>(c, f, (int)D, r0, rb, shift, closure, cand, dict_cap, pl); break;
        case 4: compile_rank<4>(c, f, (int)D, r0, rb, shift, closure, cand, dict_cap, pl); break;
        default: compile_rank<8>(c, f, (int)D, r0, rb, shift, closure, cand, dict_cap, pl); break;
      }
    } else {
      // exponent vectors in registers: NV = the next of 8 / 16 / 32 >= n
      // (a 2^26 rank space keeps KW <= 2: rank_path_ok)
      const int NVs = n <= 8 ? 8 : (n <= 16 ? 16 : 32);
      if (KW == 1 && NVs == 8) compile_rank_fused<1, 8>(c, f, (int)D, r0, rb, shift, closure, cand, dict_cap, pl);
      else if (KW == 1 && NVs == 16) compile_rank_fused<1, 16>(c, f, (int)D, r0, rb, shift, closure, cand, dict_cap, pl);
      else if (KW == 1) compile_rank_fused<1, 32>(c, f, (int)D, r0, rb, shift, closure, cand, dict_cap, pl);
      else if (NVs <= 16) compile_rank_fused<2, 16>(c, f, (int)D, r0, rb, shift, closure, cand, dict_cap, pl);
      else compile_rank_fused<2, 32>(c, f, (int)D, r0, rb, shift, closure, cand, dict_cap, pl);
    }
    return;
  }
  switch (KW) {
    case 1: compile_t<1>(c, f, r0, rb, shift, closure, cand, dict_cap, pl); break;
    case 2: compile_t<2>(c, f, r0, rb, shift, closure, cand, dict_cap, pl); break;
    case 4: compile_t<4>(c, f, r0, rb, shift, closure, cand, dict_cap, pl); break;
    default: compile_t<8>(c, f, r0, rb, shift, closure, cand, dict_cap, pl); break;
  }
}

}  // namespace f4b
