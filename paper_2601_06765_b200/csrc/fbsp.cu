// FBSP symbolic preprocessing on the device — the ★★ path of the north star.
//
// Restates reference `compile_batch` (pkg/src/fpgb/symbolic.py:293-388) with
// its helpers `_materialize` (:204-225), `closure_expand` (:238-278),
// `_reducer_preference` (:228-235), `_merge_dict` (:281-290) and the
// dictionary join (bulk.py:207-241), producing a byte-identical LayoutPlan:
//
//   round 0 : rows -> per-row delta key + length (count), offsets (scan),
//             shifted keys + coefficients (fill, warp per row)
//             -> radix sort -> unique = dictionary
//   closure : mark leads done; frontier = dictionary entries not done;
//             per frontier monomial the first basis LM dividing it, in
//             (key(LM), index) order (warp ballot over 32 candidates at a
//             time, SWAR u16x2 compares); compact in ascending key order ->
//             new rows -> fill -> sort -> unique -> keys absent from the
//             dictionary become the next frontier; merge by co-rank.
//   join    : col_ind = N-1-lower_bound(dict, key) with the dictionary staged
//             in shared memory; any miss -> MissingKeyError.
//
// Device keys use the compact order-isomorphic format (common.cuh, KeyFmt),
// so the sort touches only lane_bits * n_lanes bits.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "engine.h"

namespace f4b {

static constexpr int MAXV = 32;

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

// Pass 2 (fill): one warp per row, lanes stride over the row's terms.
template <int KW>
__global__ void k_fill(long long row_lo, long long row_hi, const int* __restrict__ rb,
                       const u64* __restrict__ delta, const u32* __restrict__ rstart,
                       const u32* __restrict__ boff, const u64* __restrict__ bckey,
                       const u32* __restrict__ bcoeff, u64* __restrict__ keys, u32* __restrict__ vals) {
  long long row = row_lo + ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (row >= row_hi) return;
  const int g = rb[row];
  const Key<KW> d = key_load<KW>(delta, row);
  const u32 s = rstart[row], len = rstart[row + 1] - s, bo = boff[g];
  for (u32 j = lane; j < len; j += 32) {
    key_store<KW>(keys, (long long)s + j, key_add<KW>(key_load<KW>(bckey, (long long)bo + j), d));
    vals[s + j] = __ldg(bcoeff + bo + j);
  }
}

template <int KW>
__global__ void k_mark_leads(long long r, const u32* __restrict__ rstart, const u64* __restrict__ keys,
                             const u64* __restrict__ dict, u32 N, uint8_t* __restrict__ done) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= r) return;
  Key<KW> k = key_load<KW>(keys, rstart[i]);
  u32 pos = key_lower_bound<KW>(dict, N, k);
  if (pos < N && key_eq<KW>(key_load<KW>(dict, pos), k)) done[pos] = 1;
}

__global__ void k_not_flags(const uint8_t* __restrict__ done, long long n, uint8_t* __restrict__ flags) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flags[i] = done[i] ? 0 : 1;
}

template <int KW>
__global__ void k_compact(const u64* __restrict__ in, long long n, const uint8_t* __restrict__ flags,
                          const u32* __restrict__ pos, u64* __restrict__ out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n && flags[i]) key_store<KW>(out, pos[i], key_load<KW>(in, i));
}

// First divisor in preference order: warp per frontier monomial.
template <int KW>
__global__ void k_closure_search(KeyFmt f, const u64* __restrict__ front, long long nf,
                                 const u32* __restrict__ lmw, const int* __restrict__ cidx, int nc, int nw,
                                 int* __restrict__ red) {
  long long j = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (j >= nf) return;
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
      for (int w = 0; w < nw; ++w) ok &= (__vcmpgeu2(me[w], __ldg(lm + w)) == 0xFFFFFFFFu);
    }
    unsigned b = __ballot_sync(0xffffffffu, ok);
    if (b) {
      found = cidx[base + __ffs(b) - 1];
      break;
    }
  }
  if (lane == 0) red[j] = found;
}

__global__ void k_red_flags(const int* __restrict__ red, long long n, uint8_t* __restrict__ flags) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) flags[i] = red[i] >= 0 ? 1 : 0;
}

template <int KW>
__global__ void k_new_rows(KeyFmt f, const u64* __restrict__ front, long long nf, const int* __restrict__ red,
                           const u32* __restrict__ pos, long long row_base, long long cl_base,
                           const u32* __restrict__ boff, const u32* __restrict__ blen,
                           const u64* __restrict__ bckey, const u16* __restrict__ lmexp,
                           const u16* __restrict__ maxe, int round, int* __restrict__ rows_basis,
                           u64* __restrict__ rows_delta, u32* __restrict__ rows_len, int* __restrict__ cl_basis,
                           u16* __restrict__ cl_shift, int* __restrict__ cl_round, u32* __restrict__ err) {
  long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= nf) return;
  const int g = red[j];
  if (g < 0) return;
  const long long q = pos[j];
  const long long row = row_base + q;
  const Key<KW> m = key_load<KW>(front, j);
  const Key<KW> lmk = key_load<KW>(bckey, boff[g]);
  rows_basis[row] = g;
  key_store<KW>(rows_delta, row, key_sub<KW>(m, lmk));
  rows_len[row] = blen[g];
  u16 e[MAXV];
  key_decode<KW>(f, m, e);
  bool over = false;
  for (int v = 0; v < f.n_vars; ++v) {
    u32 s = (u32)e[v] - (u32)lmexp[(long long)g * f.n_vars + v];
    over |= (s + (u32)maxe[(long long)g * f.n_vars + v]) > 0xFFFFu;
    cl_shift[(cl_base + q) * f.n_vars + v] = (u16)s;
  }
  if (over) atomicOr(err, (u32)DEVERR_LANE_OVERFLOW);
  cl_basis[cl_base + q] = g;
  cl_round[cl_base + q] = round;
}

__global__ void k_offsets(const u32* __restrict__ scanned, long long n, u32 base, u32* __restrict__ out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= n) out[i] = base + scanned[i];
}

template <int KW>
__global__ void k_absent_flags(const u64* __restrict__ uniq, long long nu, const u64* __restrict__ dict, u32 N,
                               uint8_t* __restrict__ flags) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nu) return;
  Key<KW> k = key_load<KW>(uniq, i);
  u32 pos = key_lower_bound<KW>(dict, N, k);
  flags[i] = (pos < N && key_eq<KW>(key_load<KW>(dict, pos), k)) ? 0 : 1;
}

// Merge two disjoint ascending sets by co-rank.
template <int KW>
__global__ void k_merge_corank(const u64* __restrict__ a, u32 na, const u64* __restrict__ b, u32 nb,
                               u64* __restrict__ out) {
  long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < na) {
    Key<KW> k = key_load<KW>(a, i);
    key_store<KW>(out, i + key_lower_bound<KW>(b, nb, k), k);
  } else if (i < (long long)na + nb) {
    long long j = i - na;
    Key<KW> k = key_load<KW>(b, j);
    key_store<KW>(out, j + key_lower_bound<KW>(a, na, k), k);
  }
}

// Dictionary join: col = N-1-lower_bound(dict, key); dictionary in smem.
template <int KW>
__global__ void __launch_bounds__(512) k_join(const u64* __restrict__ keys, long long M, const u64* __restrict__ dict,
                                              u32 N, int use_smem, u32* __restrict__ col, u32* __restrict__ err) {
  extern __shared__ u64 sdict[];
  const u64* table = dict;
  if (use_smem) {
    for (long long i = threadIdx.x; i < (long long)N * KW; i += blockDim.x) sdict[i] = __ldg(dict + i);
    __syncthreads();
    table = sdict;
  }
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < M; t += (long long)gridDim.x * blockDim.x) {
    Key<KW> k = key_load<KW>(keys, t);
    u32 pos = key_lower_bound<KW>(table, N, k);
    if (pos >= N || !key_eq<KW>(key_load_rw<KW>(table, pos), k)) {
      atomicOr(err, (u32)DEVERR_MISSING_KEY);
      pos = 0;
    }
    col[t] = N - 1 - pos;
  }
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

#define LAUNCH_CHECK(name) \
  do {                     \
  } while (0)

// Term-order comparison of exponent vectors (reference monomials.py:107-128).
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
  long long t0 = B.ckey_terms, t1 = B.n_terms;
  F4B_LAUNCH(c, k_encode_basis<KW>, nblk(t1 - t0, 256), 256, 0, f, B.exps.as<u16>(), t0, t1, B.ckey.as<u64>());
  LAUNCH_CHECK("k_encode_basis");
  B.ckey_terms = t1;
}

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
  ensure(c, c->errflag, 64);
  u32* err = c->errflag.as<u32>();
  check_cuda(cudaMemsetAsync(err, 0, 4, c->stream), "memset err");

  // ---- round 0: count (host knows the lengths) / scan / fill -------------
  std::vector<uint32_t> h_start(r0 + 1);
  long long M = 0;
  for (long long i = 0; i < r0; ++i) {
    h_start[i] = (uint32_t)M;
    M += B.h_len[h_rb[i]];
  }
  h_start[r0] = (uint32_t)M;
  if (M >= (1ll << 31)) fail(F4B_ERR_SIZE_CAP, "batch has more than 2^31 terms");
  long long rcap = std::max<long long>(2 * r0 + 1024, 4096);
  ensure(c, c->rows_basis, rcap * sizeof(int));
  ensure(c, c->rows_delta, rcap * KW * sizeof(u64));
  ensure(c, c->rows_len, rcap * sizeof(u32));
  ensure(c, c->rows_start, (rcap + 1) * sizeof(u32));
  ensure(c, c->shift_in, (size_t)std::max<long long>(r0, 1) * n * sizeof(u16));
  check_cuda(cudaMemcpyAsync(c->rows_basis.p, h_rb, r0 * sizeof(int), cudaMemcpyHostToDevice, c->stream), "h2d rows");
  check_cuda(cudaMemcpyAsync(c->shift_in.p, h_shift, r0 * n * sizeof(u16), cudaMemcpyHostToDevice, c->stream), "h2d shifts");
  check_cuda(cudaMemcpyAsync(c->rows_start.p, h_start.data(), (r0 + 1) * sizeof(u32), cudaMemcpyHostToDevice, c->stream),
             "h2d starts");
  F4B_LAUNCH(c, k_rows0<KW>, nblk(r0, 256), 256, 0, f, r0, c->rows_basis.as<int>(), c->shift_in.as<u16>(),
                                                     B.len.as<u32>(), c->rows_delta.as<u64>(), c->rows_len.as<u32>());
  LAUNCH_CHECK("k_rows0");
  long long mcap = std::max<long long>(M + M / 2 + 4096, 1 << 16);
  ensure(c, c->keys_all, mcap * KW * sizeof(u64));
  ensure(c, c->vals_all, mcap * sizeof(u32));
  F4B_LAUNCH(c, k_fill<KW>, nblk(r0 * 32, 256), 256, 0, 0, r0, c->rows_basis.as<int>(), c->rows_delta.as<u64>(),
                                                         c->rows_start.as<u32>(), B.off.as<u32>(), B.ckey.as<u64>(),
                                                         B.coeff.as<u32>(), c->keys_all.as<u64>(), c->vals_all.as<u32>());
  LAUNCH_CHECK("k_fill");

  // ---- dictionary: radix sort + unique ------------------------------------
  u64* sorted = nullptr;
  radix_sort_keys(c, KW, c->keys_all.as<u64>(), M, bits, &sorted);
  pl->sort_passes += (bits + 7) / 8;
  ensure(c, c->dict_a, (size_t)(M + 1) * KW * sizeof(u64));
  long long N = unique_keys(c, KW, sorted, M, c->dict_a.as<u64>());
  u64* dict = c->dict_a.as<u64>();

  long long r = r0;
  long long rounds = 0;
  long long n_cl = 0;
  if (closure && N > 0) {
    // leads of the input rows are covered (symbolic.py:339)
    ensure(c, c->flags, (size_t)N + 16);
    ensure(c, c->front, (size_t)(N + 1) * KW * sizeof(u64));
    ensure(c, c->tmp_u32b, (size_t)(N + 2) * sizeof(u32));
    ensure(c, c->tmp_u32c, (size_t)N + 16);  // done flags (u8)
    uint8_t* done = c->tmp_u32c.as<uint8_t>();
    check_cuda(cudaMemsetAsync(done, 0, N, c->stream), "memset done");
    F4B_LAUNCH(c, k_mark_leads<KW>, nblk(r0, 256), 256, 0, r0, c->rows_start.as<u32>(), c->keys_all.as<u64>(), dict,
                                                            (u32)N, done);
    LAUNCH_CHECK("k_mark_leads");
    uint8_t* flags = c->flags.as<uint8_t>();
    F4B_LAUNCH(c, k_not_flags, nblk(N, 256), 256, 0, done, N, flags);
    LAUNCH_CHECK("k_not_flags");
    u32* pos = c->tmp_u32b.as<u32>();
    exclusive_scan_flags(c, flags, pos, N);
    F4B_LAUNCH(c, k_compact<KW>, nblk(N, 256), 256, 0, dict, N, flags, pos, c->front.as<u64>());
    LAUNCH_CHECK("k_compact");
    long long nf = read_u32(c, pos + N);

    // candidate LMs in preference order (key(LM), index) (symbolic.py:228-235)
    std::vector<int32_t> pref(cand);
    std::stable_sort(pref.begin(), pref.end(), [&](int32_t a, int32_t b) {
      int s = mon_cmp(&B.h_lm[(size_t)a * n], &B.h_lm[(size_t)b * n], n, c->order);
      return s != 0 ? s < 0 : a < b;
    });
    const int nc = (int)pref.size();
    const int nw = (n + 1) / 2;
    std::vector<uint32_t> h_lmw((size_t)std::max(nc, 1) * nw, 0u);
    for (int q = 0; q < nc; ++q)
      for (int v = 0; v < n; ++v)
        h_lmw[(size_t)q * nw + v / 2] |= (uint32_t)B.h_lm[(size_t)pref[q] * n + v] << (16 * (v & 1));
    ensure(c, c->lmpref, h_lmw.size() * sizeof(u32));
    ensure(c, c->cand_idx, (size_t)std::max(nc, 1) * sizeof(int));
    check_cuda(cudaMemcpyAsync(c->lmpref.p, h_lmw.data(), h_lmw.size() * sizeof(u32), cudaMemcpyHostToDevice, c->stream),
               "h2d lm");
    if (nc)
      check_cuda(cudaMemcpyAsync(c->cand_idx.p, pref.data(), nc * sizeof(int), cudaMemcpyHostToDevice, c->stream),
                 "h2d cand");

    long long clcap = 1024;
    ensure(c, c->cl_basis, clcap * sizeof(int));
    ensure(c, c->cl_shift, clcap * n * sizeof(u16));
    ensure(c, c->cl_round, clcap * sizeof(int));

    while (nf > 0 && nc > 0) {
      // closure search over the frontier
      ensure(c, c->red, (size_t)nf * sizeof(int));
      F4B_LAUNCH(c, k_closure_search<KW>, nblk(nf * 32, 256), 256, 0, f, c->front.as<u64>(), nf, c->lmpref.as<u32>(),
                                                                        c->cand_idx.as<int>(), nc, nw, c->red.as<int>());
      LAUNCH_CHECK("k_closure_search");
      ensure(c, c->flags, (size_t)nf + 16);
      ensure(c, c->tmp_u32b, (size_t)(nf + 2) * sizeof(u32));
      flags = c->flags.as<uint8_t>();
      pos = c->tmp_u32b.as<u32>();
      F4B_LAUNCH(c, k_red_flags, nblk(nf, 256), 256, 0, c->red.as<int>(), nf, flags);
      LAUNCH_CHECK("k_red_flags");
      exclusive_scan_flags(c, flags, pos, nf);
      long long R = read_u32(c, pos + nf);
      if (R == 0) break;
      ++rounds;
      // grow row / closure arrays (contents preserved)
      if (r + R + 1 > rcap) {
        rcap = 2 * (r + R + 1);
        ensure_keep(c, c->rows_basis, rcap * sizeof(int));
        ensure_keep(c, c->rows_delta, rcap * KW * sizeof(u64));
        ensure_keep(c, c->rows_len, rcap * sizeof(u32));
        ensure_keep(c, c->rows_start, (rcap + 1) * sizeof(u32));
      }
      if (n_cl + R > clcap) {
        clcap = 2 * (n_cl + R);
        ensure_keep(c, c->cl_basis, clcap * sizeof(int));
        ensure_keep(c, c->cl_shift, clcap * n * sizeof(u16));
        ensure_keep(c, c->cl_round, clcap * sizeof(int));
      }
      F4B_LAUNCH(c, k_new_rows<KW>, nblk(nf, 256), 256, 0, 
          f, c->front.as<u64>(), nf, c->red.as<int>(), pos, r, n_cl, B.off.as<u32>(), B.len.as<u32>(), B.ckey.as<u64>(),
          B.lmexp.as<u16>(), B.maxe.as<u16>(), (int)rounds, c->rows_basis.as<int>(), c->rows_delta.as<u64>(),
          c->rows_len.as<u32>(), c->cl_basis.as<int>(), c->cl_shift.as<u16>(), c->cl_round.as<int>(), err);
      LAUNCH_CHECK("k_new_rows");
      // offsets of the new rows continue after M
      ensure(c, c->tmp_u32a, (size_t)(R + 2) * sizeof(u32));
      exclusive_scan_u32(c, c->rows_len.as<u32>() + r, c->tmp_u32a.as<u32>(), R);
      F4B_LAUNCH(c, k_offsets, nblk(R + 1, 256), 256, 0, c->tmp_u32a.as<u32>(), R, (u32)M, c->rows_start.as<u32>() + r);
      LAUNCH_CHECK("k_offsets");
      long long Mk = read_u32(c, c->tmp_u32a.as<u32>() + R);
      if (M + Mk >= (1ll << 31)) fail(F4B_ERR_SIZE_CAP, "batch has more than 2^31 terms");
      if (M + Mk > mcap) {
        mcap = 2 * (M + Mk);
        ensure_keep(c, c->keys_all, mcap * KW * sizeof(u64));
        ensure_keep(c, c->vals_all, mcap * sizeof(u32));
      }
      F4B_LAUNCH(c, k_fill<KW>, nblk(R * 32, 256), 256, 0, r, r + R, c->rows_basis.as<int>(), c->rows_delta.as<u64>(),
                                                            c->rows_start.as<u32>(), B.off.as<u32>(), B.ckey.as<u64>(),
                                                            B.coeff.as<u32>(), c->keys_all.as<u64>(), c->vals_all.as<u32>());
      LAUNCH_CHECK("k_fill");
      u64* nk = c->keys_all.as<u64>() + (size_t)M * KW;
      radix_sort_keys(c, KW, nk, Mk, bits, &sorted);
      pl->sort_passes += (bits + 7) / 8;
      ensure(c, c->uniq, (size_t)(Mk + 1) * KW * sizeof(u64));
      long long nu = unique_keys(c, KW, sorted, Mk, c->uniq.as<u64>());
      // keys not yet in the dictionary become the next frontier
      ensure(c, c->flags, (size_t)nu + 16);
      ensure(c, c->tmp_u32b, (size_t)(nu + 2) * sizeof(u32));
      ensure(c, c->front_new, (size_t)(nu + 1) * KW * sizeof(u64));
      flags = c->flags.as<uint8_t>();
      pos = c->tmp_u32b.as<u32>();
      F4B_LAUNCH(c, k_absent_flags<KW>, nblk(nu, 256), 256, 0, c->uniq.as<u64>(), nu, dict, (u32)N, flags);
      LAUNCH_CHECK("k_absent_flags");
      exclusive_scan_flags(c, flags, pos, nu);
      F4B_LAUNCH(c, k_compact<KW>, nblk(nu, 256), 256, 0, c->uniq.as<u64>(), nu, flags, pos, c->front_new.as<u64>());
      LAUNCH_CHECK("k_compact");
      long long nnew = read_u32(c, pos + nu);
      // merged dictionary (symbolic.py:281-290)
      u64* other = (dict == c->dict_a.as<u64>()) ? nullptr : c->dict_a.as<u64>();
      DBuf& obuf = (dict == c->dict_a.as<u64>()) ? c->dict_b : c->dict_a;
      DBuf& cbuf = (dict == c->dict_a.as<u64>()) ? c->dict_a : c->dict_b;
      (void)other;
      ensure(c, obuf, (size_t)(N + nnew + 1) * KW * sizeof(u64));
      if (nnew) {
        F4B_LAUNCH(c, k_merge_corank<KW>, nblk(N + nnew, 256), 256, 0, cbuf.as<u64>(), (u32)N, c->front_new.as<u64>(),
                                                                        (u32)nnew, obuf.as<u64>());
        LAUNCH_CHECK("k_merge_corank");
        dict = obuf.as<u64>();
      }
      N += nnew;
      M += Mk;
      r += R;
      n_cl += R;
      if (N > dict_cap) fail(F4B_ERR_SIZE_CAP, "dictionary exceeded the cap after " + std::to_string(rounds) +
                                                   " closure rounds");
      // frontier <- new keys
      std::swap(c->front, c->front_new);
      nf = nnew;
    }
  }
  check_cuda(cudaEventRecord(ev1, c->stream), "event record");

  // ---- row assembly: offsets are final; join ------------------------------
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
  check_cuda(cudaMemcpyAsync(pl->row_ptr.p, c->rows_start.p, (r + 1) * sizeof(u32), cudaMemcpyDeviceToDevice, c->stream),
             "d2d row_ptr");
  if (M) {
    check_cuda(cudaMemcpyAsync(pl->val.p, c->vals_all.p, M * sizeof(u32), cudaMemcpyDeviceToDevice, c->stream), "d2d val");
  }
  if (N) {
    check_cuda(cudaMemcpyAsync(pl->dict.p, dict, N * KW * sizeof(u64), cudaMemcpyDeviceToDevice, c->stream), "d2d dict");
  }
  if (n_cl) {
    check_cuda(cudaMemcpyAsync(pl->cl_basis.p, c->cl_basis.p, n_cl * sizeof(int), cudaMemcpyDeviceToDevice, c->stream), "d2d");
    check_cuda(cudaMemcpyAsync(pl->cl_shift.p, c->cl_shift.p, n_cl * n * sizeof(u16), cudaMemcpyDeviceToDevice, c->stream),
               "d2d");
    check_cuda(cudaMemcpyAsync(pl->cl_round.p, c->cl_round.p, n_cl * sizeof(int), cudaMemcpyDeviceToDevice, c->stream), "d2d");
  }
  if (M) {
    size_t smem = (size_t)N * KW * sizeof(u64);
    int use_smem = smem <= 200 * 1024 ? 1 : 0;
    if (!use_smem) smem = 0;
    static bool attr_set[9] = {false};
    if (!attr_set[KW]) {
      check_cuda(cudaFuncSetAttribute(k_join<KW>, cudaFuncAttributeMaxDynamicSharedMemorySize, 200 * 1024 + 1024),
                 "join attr");
      attr_set[KW] = true;
    }
    int blocks = (int)std::min<long long>(nblk(M, 512), (long long)c->num_sms * (use_smem ? 1 : 4));
    F4B_LAUNCH(c, k_join<KW>, blocks, 512, smem, c->keys_all.as<u64>(), M, pl->dict.as<u64>(), (u32)N, use_smem,
                                                 pl->col_ind.as<u32>(), err);
    LAUNCH_CHECK("k_join");
  }
  if (N) {
    F4B_LAUNCH(c, k_dict_exps<KW>, nblk(N, 256), 256, 0, f, pl->dict.as<u64>(), (u32)N, pl->dict_exps.as<u16>());
    LAUNCH_CHECK("k_dict_exps");
  }
  check_cuda(cudaEventRecord(ev2, c->stream), "event record");
  u32 e = read_u32(c, err);
  float ms1 = 0, ms2 = 0;
  check_cuda(cudaEventElapsedTime(&ms1, ev0, ev1), "elapsed");
  check_cuda(cudaEventElapsedTime(&ms2, ev1, ev2), "elapsed");
  cudaEventDestroy(ev0);
  cudaEventDestroy(ev1);
  cudaEventDestroy(ev2);
  pl->dict_ns = (int64_t)(ms1 * 1e6);
  pl->asm_ns = (int64_t)(ms2 * 1e6);
  pl->launches = c->launches;
  if (e & DEVERR_LANE_OVERFLOW) fail(F4B_ERR_LANE_OVERFLOW, "shifted exponent overflows a 16-bit lane");
  if (e & DEVERR_MISSING_KEY) fail(F4B_ERR_MISSING_KEY, "row key absent from dictionary (closure defect)");
}

void compile_batch(Ctx* c, long long r0, const int32_t* rb, const uint16_t* shift, int closure, const int32_t* cands,
                   long long n_cands, long long dict_cap, f4b_plan* pl) {
  Basis& B = c->basis;
  const int n = c->n_vars;
  // validation + batch degree (host metadata only)
  long long D = 0;
  for (long long i = 0; i < r0; ++i) {
    int g = rb[i];
    if (g < 0 || g >= B.n_polys) fail(F4B_ERR_PRECONDITION, "row references unknown basis index");
    if (B.h_len[g] < 1) fail(F4B_ERR_PROPERTY, "zero polynomial referenced as a reducer");
    long long d = 0;
    for (int v = 0; v < n; ++v) {
      long long s = shift[i * n + v];
      if (s + B.h_maxe[(size_t)g * n + v] > 0xFFFF) fail(F4B_ERR_LANE_OVERFLOW, "shifted exponent overflows a 16-bit lane");
      d += s + B.h_lm[(size_t)g * n + v];
    }
    D = std::max(D, d);
  }
  std::vector<int32_t> cand;
  if (cands) {
    cand.assign(cands, cands + n_cands);
    for (int32_t k : cand)
      if (k < 0 || k >= B.n_polys) fail(F4B_ERR_PRECONDITION, "candidate references unknown basis index");
  } else {
    cand.resize(B.n_polys);
    for (int k = 0; k < B.n_polys; ++k) cand[k] = k;
  }
  // drop empty candidates (zero polynomials have no leading monomial)
  cand.erase(std::remove_if(cand.begin(), cand.end(), [&](int32_t k) { return B.h_len[k] < 1; }), cand.end());
  KeyFmt f;
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
  int bits = f.lane_bits * f.n_lanes;
  int KW = 1;
  while (64 * KW < bits) KW *= 2;
  if (KW > 8) fail(F4B_ERR_PRECONDITION, "batch degree too large for the device key format");
  switch (KW) {
    case 1: compile_t<1>(c, f, r0, rb, shift, closure, cand, dict_cap, pl); break;
    case 2: compile_t<2>(c, f, r0, rb, shift, closure, cand, dict_cap, pl); break;
    case 4: compile_t<4>(c, f, r0, rb, shift, closure, cand, dict_cap, pl); break;
    default: compile_t<8>(c, f, r0, rb, shift, closure, cand, dict_cap, pl); break;
  }
}

}  // namespace f4b
