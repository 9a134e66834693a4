// Sharded compile_batch across ranks — one rank per GPU.
//
// Restates reference compile_batch (pkg/src/fpgb/symbolic.py:293-388) as
// the stages of a multi-rank pipeline.  Every rank runs the same calls; the
// host (Python: paper_2601_06765_b200/dist.py ShardedCompiler) all-gathers the
// small per-rank outputs between them over NCCL (or gloo):
//
//   begin        every rank: all input rows' shift deltas, row table and lead
//                bits (symbolic.py:339); ITS contiguous, length-balanced row
//                range [lo, hi) materialised -> ranks -> a local presence
//                bitmap -> its sorted unique run (ascending rank = ascending
//                key, _materialize + radix_sort + unique_sorted, :204-225)
//   merge        the gathered runs -> the global dictionary (every rank the
//                same); round-1 frontier = dict & ~done (closure_expand :257)
//   round        ITS slice [f_lo, f_hi) of the frontier: first LM divisor in
//                (key(LM), index) order (:262-268), the reducer rows' terms
//                ranked against the dictionary -> its run of new monomials
//   round_merge  the gathered reducer indices (frontier order) -> the round's
//                rows appended in ascending key(m) (:270-277); the gathered
//                runs -> next frontier, dict |= new (_merge_dict :281-290)
//   finish       final dictionary (descending, column order) and the join of
//                ITS row range of the final row list (merge_join_index,
//                :366-380) -> a plan slice.
//
// Concatenating the slices of all ranks in rank order gives the single-GPU
// plan byte for byte (tests/test_gpu_shard.py).  grevlex rank path only
// (rank space <= 2^26, rank.cuh); every collective payload is a list of u32
// ranks or i32 basis indices.
#include <algorithm>
#include <chrono>
#include <cstring>
#include <vector>

#include "block.cuh"
#include "common.cuh"
#include "engine.h"
#include "fbsp_internal.cuh"
#include "rank.cuh"

namespace f4b {

static inline unsigned nbk(long long n, int t) { return (unsigned)std::max<long long>(1, (n + t - 1) / t); }

// ---------------------------------------------------------------------------
// kernels
// ---------------------------------------------------------------------------
template <int KW, int NV>
__global__ void k_sh_rows0(KeyFmt f, long long r0, const int* __restrict__ rb, const u16* __restrict__ shift,
                           const u32* __restrict__ start, const u32* __restrict__ boff, const u64* __restrict__ bckey,
                           const u32* __restrict__ bt, int st, int closure, int* __restrict__ rows_basis,
                           u64* __restrict__ rows_delta, u32* __restrict__ rows_start, u32* __restrict__ done) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i > r0) return;
  if (i == r0) {
    rows_start[r0] = start[r0];
    return;
  }
  const int n = f.n_vars;
  u16 e[NV], z[NV];
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    e[v] = v < n ? shift[i * n + v] : (u16)0;
    z[v] = 0;
  }
  const Key<KW> dl = key_sub<KW>(gl_encode<KW, NV>(f, e), gl_encode<KW, NV>(f, z));
  const int g = rb[i];
  rows_basis[i] = g;
  key_store<KW>(rows_delta, i, dl);
  rows_start[i] = start[i];
  if (closure) {
    const u32 rk = key_rank<KW>(f, bt, st, key_add<KW>(key_load<KW>(bckey, boff[g]), dl));
    atomicOr(done + (rk >> 5), 1u << (rk & 31));
  }
}

// Warp per row of [lo, hi): every term -> rank -> bit in `out` unless set in
// `known` (the dictionary) or already in `out`.
template <int KW>
__global__ void k_sh_fill(KeyFmt f, long long lo, long long hi, const int* __restrict__ rows_basis,
                          const u64* __restrict__ rows_delta, const u32* __restrict__ boff,
                          const u32* __restrict__ blen, const u64* __restrict__ bckey, const u32* __restrict__ bt_g,
                          int st, int bt_words, const u32* __restrict__ known, u32* __restrict__ out) {
  extern __shared__ u32 bt[];
  for (int i = threadIdx.x; i < bt_words; i += blockDim.x) bt[i] = bt_g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long nw = (long long)gridDim.x * (blockDim.x / 32);
  for (long long row = lo + (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); row < hi; row += nw) {
    const int g = rows_basis[row];
    const Key<KW> dl = key_load_cg<KW>(rows_delta, row);
    const u32 off = boff[g], len = blen[g];
    for (u32 t = lane; t < len; t += 32) {
      const u32 rk = key_rank<KW>(f, bt, st, key_add<KW>(key_load<KW>(bckey, (long long)off + t), dl));
      const u32 w = rk >> 5, bit = 1u << (rk & 31);
      if (known && (__ldg(known + w) & bit)) continue;
      if (!(__ldcg(out + w) & bit)) atomicOr(out + w, bit);
    }
  }
}

// cnt[w] = popc(A[w] & ~B[w])
__global__ void k_sh_wcount(const u32* __restrict__ A, const u32* __restrict__ B, u32 words, u32* __restrict__ cnt) {
  const u32 w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w < words) cnt[w] = __popc(A[w] & (B ? ~B[w] : 0xFFFFFFFFu));
}

// ranks of the set bits of A & ~B at the scanned offsets; optionally clear A
// and / or OR the emitted bits into `or_into`
__global__ void k_sh_wemit(u32* __restrict__ A, const u32* __restrict__ B, u32 words, const u32* __restrict__ pre,
                           u32* __restrict__ ranks, int clear, u32* __restrict__ or_into) {
  const u32 w = blockIdx.x * blockDim.x + threadIdx.x;
  if (w >= words) return;
  const u32 a = A[w];
  u32 x = a & (B ? ~B[w] : 0xFFFFFFFFu);
  if (clear && a) A[w] = 0;
  if (or_into && x) or_into[w] |= x;
  u32 p = pre[w];
  while (x) {
    const int b = __ffs(x) - 1;
    x &= x - 1;
    ranks[p++] = w * 32 + b;
  }
}

__global__ void k_sh_set(const u32* __restrict__ ranks, long long n, u32* __restrict__ bits) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) {
    const u32 rk = ranks[i];
    atomicOr(bits + (rk >> 5), 1u << (rk & 31));
  }
}

// ranks -> device keys (frontier) and optionally exponents in column order
template <int KW, int NV>
__global__ void k_sh_unrank(KeyFmt f, const u32* __restrict__ ranks, long long n, int D, const u32* __restrict__ bt,
                            int st, u64* __restrict__ keys, u16* __restrict__ exps_desc) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j >= n) return;
  u16 e[NV];
  gl_unrank<NV>(ranks[j], f.n_vars, D, bt, st, e);
  key_store<KW>(keys, j, gl_encode<KW, NV>(f, e));
  if (exps_desc) {
#pragma unroll
    for (int v = 0; v < NV; ++v)
      if (v < f.n_vars) exps_desc[(n - 1 - j) * f.n_vars + v] = e[v];
  }
}

// Warp per frontier monomial of [f_lo, f_hi): the first candidate LM (in
// preference order) dividing it (SWAR u16x2 compares, ballot over 32 LMs).
template <int KW, int NV>
__global__ void k_sh_search(KeyFmt f, const u64* __restrict__ front, long long f_lo, long long f_hi,
                            const u32* __restrict__ lmw, const int* __restrict__ cidx, int nc, int nw,
                            int* __restrict__ red_out) {
  const int lane = threadIdx.x & 31;
  const long long nwarps = (long long)gridDim.x * (blockDim.x / 32);
  for (long long j = f_lo + (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); j < f_hi; j += nwarps) {
    u16 e[NV];
    gl_decode<KW, NV>(f, key_load<KW>(front, j), e);
    constexpr int NW2 = (NV + 1) / 2;
    u32 me[NW2];
#pragma unroll
    for (int w = 0; w < NW2; ++w) me[w] = (u32)e[2 * w] | (2 * w + 1 < NV ? ((u32)e[2 * w + 1] << 16) : 0u);
    int found = -1;
    for (int b0 = 0; b0 < nc; b0 += 32) {
      const int cc = b0 + lane;
      bool ok = cc < nc;
      if (ok) {
        const u32* lm = lmw + (long long)cc * nw;
#pragma unroll
        for (int w = 0; w < NW2; ++w)
          if (w < nw) ok &= (__vcmpgeu2(me[w], lm[w]) == 0xFFFFFFFFu);
      }
      const unsigned bm = __ballot_sync(0xffffffffu, ok);
      if (bm) {
        found = cidx[b0 + __ffs(bm) - 1];
        break;
      }
    }
    if (lane == 0) red_out[j - f_lo] = found;
  }
}

// Warp per frontier monomial of the slice with a reducer g: the terms of
// (m / LM(g)) g ranked; monomials absent from the dictionary -> `out`.
template <int KW>
__global__ void k_sh_fill_red(KeyFmt f, const u64* __restrict__ front, const int* __restrict__ red, long long f_lo,
                              long long f_hi, const u32* __restrict__ boff, const u32* __restrict__ blen,
                              const u64* __restrict__ bckey, const u32* __restrict__ bt_g, int st, int bt_words,
                              const u32* __restrict__ dict, u32* __restrict__ out) {
  extern __shared__ u32 bt[];
  for (int i = threadIdx.x; i < bt_words; i += blockDim.x) bt[i] = bt_g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const long long nwarps = (long long)gridDim.x * (blockDim.x / 32);
  for (long long j = f_lo + (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); j < f_hi; j += nwarps) {
    const int g = red[j - f_lo];
    if (g < 0) continue;
    const u32 off = boff[g], len = blen[g];
    const Key<KW> dl = key_sub<KW>(key_load<KW>(front, j), key_load<KW>(bckey, off));
    for (u32 t = lane; t < len; t += 32) {
      const u32 rk = key_rank<KW>(f, bt, st, key_add<KW>(key_load<KW>(bckey, (long long)off + t), dl));
      const u32 w = rk >> 5, bit = 1u << (rk & 31);
      if (__ldg(dict + w) & bit) continue;
      if (!(__ldcg(out + w) & bit)) atomicOr(out + w, bit);
    }
  }
}

__global__ void k_sh_rowflags(const int* __restrict__ red, long long nf, const u32* __restrict__ blen,
                              u32* __restrict__ flag, u32* __restrict__ len) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j < nf) {
    const int g = red[j];
    flag[j] = g >= 0 ? 1u : 0u;
    len[j] = g >= 0 ? blen[g] : 0u;
  }
}

// the round's rows in frontier (= ascending key(m)) order
template <int KW, int NV>
__global__ void k_sh_write_rows(KeyFmt f, const u64* __restrict__ front, const int* __restrict__ red, long long nf,
                                const u32* __restrict__ fpre, const u32* __restrict__ lpre, long long r_base,
                                long long cl_base, u32 M_base, int round, const u32* __restrict__ boff,
                                const u64* __restrict__ bckey, const u16* __restrict__ lmexp,
                                const u16* __restrict__ maxe, int* __restrict__ rows_basis,
                                u64* __restrict__ rows_delta, u32* __restrict__ rows_start, int* __restrict__ cl_basis,
                                u16* __restrict__ cl_shift, int* __restrict__ cl_round, u32* __restrict__ err) {
  const long long j = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (j == 0) rows_start[r_base + fpre[nf]] = M_base + lpre[nf];
  if (j >= nf) return;
  const int g = red[j];
  if (g < 0) return;
  const int n = f.n_vars;
  const long long q = fpre[j], row = r_base + q;
  const Key<KW> m = key_load<KW>(front, j);
  rows_basis[row] = g;
  key_store<KW>(rows_delta, row, key_sub<KW>(m, key_load<KW>(bckey, boff[g])));
  rows_start[row] = M_base + lpre[j];
  u16 e[NV];
  gl_decode<KW, NV>(f, m, e);
  bool over = false;
#pragma unroll
  for (int v = 0; v < NV; ++v) {
    if (v < n) {
      const u32 sft = (u32)e[v] - (u32)lmexp[(long long)g * n + v];
      over |= (sft + (u32)maxe[(long long)g * n + v]) > 0xFFFFu;
      cl_shift[(cl_base + q) * n + v] = (u16)sft;
    }
  }
  if (over) atomicOr(err, (u32)DEVERR_LANE_OVERFLOW);
  cl_basis[cl_base + q] = g;
  cl_round[cl_base + q] = round;
}

// Join of rows [lo, hi): col = N-1-(prefix[word] + popc(word & below)),
// val = basis coefficient; written at term index t - start[lo].
template <int KW>
__global__ void k_sh_join(KeyFmt f, long long lo, long long hi, const int* __restrict__ rows_basis,
                          const u64* __restrict__ rows_delta, const u32* __restrict__ rows_start,
                          const u32* __restrict__ boff, const u32* __restrict__ blen, const u64* __restrict__ bckey,
                          const u32* __restrict__ bcoeff, const u32* __restrict__ bt_g, int st, int bt_words,
                          const u32* __restrict__ dict, const u32* __restrict__ wpre, u32 N, u32* __restrict__ col,
                          u32* __restrict__ val, u32* __restrict__ err) {
  extern __shared__ u32 bt[];
  for (int i = threadIdx.x; i < bt_words; i += blockDim.x) bt[i] = bt_g[i];
  __syncthreads();
  const int lane = threadIdx.x & 31;
  const u32 base = rows_start[lo];
  bool miss = false;
  const long long nwarps = (long long)gridDim.x * (blockDim.x / 32);
  for (long long row = lo + (long long)blockIdx.x * (blockDim.x / 32) + (threadIdx.x >> 5); row < hi; row += nwarps) {
    const int g = rows_basis[row];
    const Key<KW> dl = key_load<KW>(rows_delta, row);
    const u32 off = boff[g], len = blen[g], rs = rows_start[row] - base;
    for (u32 t = lane; t < len; t += 32) {
      const u32 rk = key_rank<KW>(f, bt, st, key_add<KW>(key_load<KW>(bckey, (long long)off + t), dl));
      const u32 word = __ldg(dict + (rk >> 5)), sh = rk & 31;
      if (!((word >> sh) & 1u)) miss = true;
      col[rs + t] = N - 1 - (wpre[rk >> 5] + __popc(word & ((1u << sh) - 1u)));
      val[rs + t] = __ldg(bcoeff + off + t);
    }
  }
  if (miss) atomicOr(err, (u32)DEVERR_MISSING_KEY);
}

__global__ void k_sh_rowptr(const u32* __restrict__ rows_start, long long lo, long long hi, u32* __restrict__ rp) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i <= hi - lo) rp[i] = rows_start[lo + i] - rows_start[lo];
}

}  // namespace f4b

// ---------------------------------------------------------------------------
// host side
// ---------------------------------------------------------------------------
using namespace f4b;
f4b::Ctx* f4b_ctx_of(f4b_ctx* h);  // capi.cu

struct f4b_shard {
  Ctx* c = nullptr;
  BatchFormat bf;
  int NV = 8, closure = 0, st = 0, bt_words = 0, nc = 0, nw = 0;
  long long dict_cap = 0, r0 = 0, r = 0, n_cl = 0, rounds = 0, nf = 0, N = 0;
  unsigned long long M = 0;
  u32 words = 0;
  long long rows_cap = 0, front_cap = 0;
  int64_t ns = 0;  // device time of this rank's stages (CUDA events)
  DBuf bt, stage, rows_basis, rows_delta, rows_start, cl_basis, cl_shift, cl_round;
  DBuf maps;  // dict | done | local | wcnt/pre scratch
  DBuf front, red, ranks, scan_a, scan_b, lmw, cidx;
  u32 *dict = nullptr, *done = nullptr, *local = nullptr;
  bool finished_dict = false;
};

namespace {

void ev_begin(f4b_shard* s) { check_cuda(cudaEventRecord(timing_event(s->c, 0), s->c->stream), "event"); }
void ev_end(f4b_shard* s) {
  Ctx* c = s->c;
  check_cuda(cudaEventRecord(timing_event(c, 1), c->stream), "event");
  check_cuda(cudaEventSynchronize(timing_event(c, 1)), "event sync");
  float ms = 0;
  check_cuda(cudaEventElapsedTime(&ms, timing_event(c, 0), timing_event(c, 1)), "elapsed");
  s->ns += (int64_t)(ms * 1e6);
}

// set bits of A & ~B -> s->ranks (ascending); returns the count (one read).
// count_only: the count alone (no emission, A untouched)
long long extract(f4b_shard* s, u32* A, const u32* B, int clear, u32* or_into, u32* wpre_out = nullptr,
                  bool count_only = false) {
  Ctx* c = s->c;
  const u32 words = s->words;
  ensure(c, s->scan_a, (size_t)(words + 1) * sizeof(u32));
  u32* pre = wpre_out;
  if (!pre) {
    ensure(c, s->scan_b, (size_t)(words + 1) * sizeof(u32));
    pre = s->scan_b.as<u32>();
  }
  F4B_LAUNCH(c, k_sh_wcount, nbk(words, 256), 256, 0, A, B, words, s->scan_a.as<u32>());
  exclusive_scan_u32(c, s->scan_a.as<u32>(), pre, words);
  const long long tot = read_u32(c, pre + words);
  if (count_only) return tot;
  ensure(c, s->ranks, (size_t)std::max<long long>(tot, 1) * sizeof(u32));
  F4B_LAUNCH(c, k_sh_wemit, nbk(words, 256), 256, 0, A, B, words, pre, s->ranks.as<u32>(), clear, or_into);
  return tot;
}

template <int KW, int NV>
void unrank_front(f4b_shard* s, long long n) {
  Ctx* c = s->c;
  ensure(c, s->front, (size_t)std::max<long long>(n, 1) * KW * sizeof(u64));
  if (n)
    F4B_LAUNCH(c, (k_sh_unrank<KW, NV>), nbk(n, 256), 256, 0, s->bf.f, s->ranks.as<u32>(), n, (int)s->bf.D,
               s->bt.as<u32>(), s->st, s->front.as<u64>(), (u16*)nullptr);
  s->nf = n;
}

void grow_rows(f4b_shard* s, long long need, int KW) {
  Ctx* c = s->c;
  if (need <= s->rows_cap) return;
  const long long cap = std::max(need + need / 2, 2 * s->rows_cap);
  const int n = c->n_vars;
  ensure_keep(c, s->rows_basis, (size_t)cap * sizeof(int));
  ensure_keep(c, s->rows_delta, (size_t)cap * KW * sizeof(u64));
  ensure_keep(c, s->rows_start, (size_t)(cap + 1) * sizeof(u32));
  ensure_keep(c, s->cl_basis, (size_t)cap * sizeof(int));
  ensure_keep(c, s->cl_shift, (size_t)cap * n * sizeof(u16));
  ensure_keep(c, s->cl_round, (size_t)cap * sizeof(int));
  s->rows_cap = cap;
}

template <int KW, int NV>
long long begin_t(f4b_shard* s, const int32_t* rb, const uint16_t* shift, long long lo, long long hi) {
  Ctx* c = s->c;
  Basis& B = c->basis;
  const int n = c->n_vars;
  const long long r0 = s->r0;
  encode_basis_kw(c, s->bf.f, KW);
  // binomials | rb | row starts | shifts, one page-locked upload
  std::vector<u32> hbt((size_t)s->bt_words);
  const int rows_bt = (int)s->bf.D + n + 2;
  for (int x = 0; x < rows_bt; ++x)
    for (int y = 0; y <= n; ++y)
      hbt[(size_t)x * s->st + y] = (u32)std::min<unsigned long long>(binom_ull(x, y), 0xFFFFFFFFull);
  ensure(c, s->bt, hbt.size() * sizeof(u32));
  check_cuda(cudaMemcpyAsync(s->bt.p, hbt.data(), hbt.size() * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
  std::vector<u32> hstart((size_t)r0 + 1);
  unsigned long long acc = 0;
  for (long long i = 0; i < r0; ++i) {
    hstart[i] = (u32)acc;
    acc += (unsigned long long)B.h_len[rb[i]];
  }
  if (acc >= (1ull << 30)) fail(F4B_ERR_SIZE_CAP, "batch has more than 2^30 terms");
  hstart[r0] = (u32)acc;
  s->M = acc;
  const size_t o_rb = 0, o_st = o_rb + (size_t)r0 * 4, o_sh = o_st + ((size_t)r0 + 1) * 4,
               tot = o_sh + (size_t)r0 * n * 2 + 16;
  ensure(c, s->stage, tot);
  unsigned char* ds = s->stage.as<unsigned char>();
  check_cuda(cudaMemcpyAsync(ds + o_rb, rb, (size_t)r0 * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
  check_cuda(cudaMemcpyAsync(ds + o_st, hstart.data(), ((size_t)r0 + 1) * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
  check_cuda(cudaMemcpyAsync(ds + o_sh, shift, (size_t)r0 * n * 2, cudaMemcpyHostToDevice, c->stream), "h2d");
  grow_rows(s, r0 + 1, KW);
  // presence maps
  ensure(c, s->maps, (size_t)3 * s->words * sizeof(u32) + 64);
  check_cuda(cudaMemsetAsync(s->maps.p, 0, (size_t)3 * s->words * sizeof(u32) + 64, c->stream), "memset");
  s->dict = s->maps.as<u32>();
  s->done = s->dict + s->words;
  s->local = s->done + s->words;
  F4B_LAUNCH(c, (k_sh_rows0<KW, NV>), nbk(r0 + 1, 256), 256, 0, s->bf.f, r0,
             reinterpret_cast<const int*>(ds + o_rb), reinterpret_cast<const u16*>(ds + o_sh),
             reinterpret_cast<const u32*>(ds + o_st), B.off.as<u32>(), B.ckey.as<u64>(), s->bt.as<u32>(), s->st,
             s->closure, s->rows_basis.as<int>(), s->rows_delta.as<u64>(), s->rows_start.as<u32>(), s->done);
  s->r = r0;
  if (hi > lo) {
    const size_t smem = (size_t)s->bt_words * 4;
    F4B_LAUNCH(c, k_sh_fill<KW>, (unsigned)std::min<long long>(nbk(hi - lo, 8), (long long)c->num_sms * 8), 256,
               smem, s->bf.f, lo, hi, s->rows_basis.as<int>(), s->rows_delta.as<u64>(), B.off.as<u32>(),
               B.len.as<u32>(), B.ckey.as<u64>(), s->bt.as<u32>(), s->st, s->bt_words, (const u32*)nullptr, s->local);
  }
  return extract(s, s->local, nullptr, 1, nullptr);
}

template <int KW, int NV>
long long merge_t(f4b_shard* s, const uint32_t* ranks, long long n) {
  Ctx* c = s->c;
  ensure(c, s->scan_a, (size_t)std::max<long long>(n, 1) * sizeof(u32));
  if (n) {
    check_cuda(cudaMemcpyAsync(s->scan_a.p, ranks, (size_t)n * 4, cudaMemcpyDefault, c->stream), "copy runs");
    F4B_LAUNCH(c, k_sh_set, nbk(n, 256), 256, 0, s->scan_a.as<u32>(), n, s->dict);
  }
  s->N = extract(s, s->dict, nullptr, 0, nullptr, nullptr, true);
  if (s->N > s->dict_cap) fail(F4B_ERR_SIZE_CAP, "dictionary exceeded the cap after 0 closure rounds");
  if (!s->closure) {
    s->nf = 0;
    return 0;
  }
  // round-1 frontier: dict & ~done in ascending rank (= ascending key)
  const long long nf = extract(s, s->dict, s->done, 0, nullptr);
  unrank_front<KW, NV>(s, nf);
  return nf;
}

template <int KW, int NV>
long long round_t(f4b_shard* s, long long f_lo, long long f_hi, int32_t* red_out) {
  Ctx* c = s->c;
  Basis& B = c->basis;
  const long long m = std::max<long long>(f_hi - f_lo, 0);
  ensure(c, s->red, (size_t)std::max<long long>(s->nf, 1) * sizeof(int));
  if (m) {
    const unsigned g = (unsigned)std::min<long long>(nbk(m, 8), (long long)c->num_sms * 8);
    F4B_LAUNCH(c, (k_sh_search<KW, NV>), g, 256, 0, s->bf.f, s->front.as<u64>(), f_lo, f_hi, s->lmw.as<u32>(),
               s->cidx.as<int>(), s->nc, s->nw, s->red.as<int>());
    F4B_LAUNCH(c, k_sh_fill_red<KW>, g, 256, (size_t)s->bt_words * 4, s->bf.f, s->front.as<u64>(), s->red.as<int>(),
               f_lo, f_hi, B.off.as<u32>(), B.len.as<u32>(), B.ckey.as<u64>(), s->bt.as<u32>(), s->st, s->bt_words,
               s->dict, s->local);
    check_cuda(cudaMemcpyAsync(red_out, s->red.p, (size_t)m * sizeof(int), cudaMemcpyDefault, c->stream), "red out");
  }
  return extract(s, s->local, nullptr, 1, nullptr);
}

template <int KW, int NV>
long long round_merge_t(f4b_shard* s, const int32_t* red_all, long long nf, const uint32_t* ranks, long long n) {
  Ctx* c = s->c;
  Basis& B = c->basis;
  if (nf != s->nf) fail(F4B_ERR_PRECONDITION, "shard round_merge: reducer list does not cover the frontier");
  ensure(c, s->red, (size_t)std::max<long long>(nf, 1) * sizeof(int));
  if (nf) check_cuda(cudaMemcpyAsync(s->red.p, red_all, (size_t)nf * 4, cudaMemcpyDefault, c->stream), "red in");
  // row offsets: scans of (found, length) in frontier order
  DBuf fl, ln, fpre, lpre;
  ensure(c, fl, (size_t)(nf + 1) * 4);
  ensure(c, ln, (size_t)(nf + 1) * 4);
  ensure(c, fpre, (size_t)(nf + 1) * 4);
  ensure(c, lpre, (size_t)(nf + 1) * 4);
  if (nf)
    F4B_LAUNCH(c, k_sh_rowflags, nbk(nf, 256), 256, 0, s->red.as<int>(), nf, B.len.as<u32>(), fl.as<u32>(),
               ln.as<u32>());
  exclusive_scan_u32(c, fl.as<u32>(), fpre.as<u32>(), nf);
  exclusive_scan_u32(c, ln.as<u32>(), lpre.as<u32>(), nf);
  u32* h = c->h_stat;
  check_cuda(cudaMemcpyAsync(h, fpre.as<u32>() + nf, 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
  check_cuda(cudaMemcpyAsync(h + 1, lpre.as<u32>() + nf, 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  const long long R = h[0], Mk = h[1];
  if (R == 0) {  // fixed point: no new rows, the round does not count
    release(c, fl), release(c, ln), release(c, fpre), release(c, lpre);
    s->nf = 0;
    return 0;
  }
  if (s->M + (unsigned long long)Mk >= (1ull << 30)) fail(F4B_ERR_SIZE_CAP, "batch has more than 2^30 terms");
  grow_rows(s, s->r + R + 1, KW);
  ensure(c, c->errflag, 64);
  F4B_LAUNCH(c, (k_sh_write_rows<KW, NV>), nbk(nf, 256), 256, 0, s->bf.f, s->front.as<u64>(), s->red.as<int>(), nf,
             fpre.as<u32>(), lpre.as<u32>(), s->r, s->n_cl, (u32)s->M, (int)s->rounds + 1, B.off.as<u32>(),
             B.ckey.as<u64>(), B.lmexp.as<u16>(), B.maxe.as<u16>(), s->rows_basis.as<int>(), s->rows_delta.as<u64>(),
             s->rows_start.as<u32>(), s->cl_basis.as<int>(), s->cl_shift.as<u16>(), s->cl_round.as<int>(),
             c->errflag.as<u32>());
  release(c, fl), release(c, ln), release(c, fpre), release(c, lpre);
  s->r += R;
  s->n_cl += R;
  s->M += Mk;
  s->rounds += 1;
  // next frontier: the gathered new monomials (each run excludes the
  // dictionary; duplicates across ranks merge), dict |= new
  ensure(c, s->scan_a, (size_t)std::max<long long>(n, 1) * sizeof(u32));
  if (n) {
    check_cuda(cudaMemcpyAsync(s->scan_a.p, ranks, (size_t)n * 4, cudaMemcpyDefault, c->stream), "copy runs");
    F4B_LAUNCH(c, k_sh_set, nbk(n, 256), 256, 0, s->scan_a.as<u32>(), n, s->local);
  }
  const long long nnf = extract(s, s->local, nullptr, 1, s->dict);
  s->N += nnf;
  // DICT_CAP after the merge (symbolic.py:359-363)
  if (s->N > s->dict_cap)
    fail(F4B_ERR_SIZE_CAP, "dictionary exceeded the cap after " + std::to_string(s->rounds) + " closure rounds");
  unrank_front<KW, NV>(s, nnf);
  return nnf;
}

template <int KW, int NV>
void finish_t(f4b_shard* s, long long lo, long long hi, f4b_plan* pl) {
  Ctx* c = s->c;
  Basis& B = c->basis;
  const int n = c->n_vars;
  if (lo < 0 || hi > s->r || lo > hi) fail(F4B_ERR_PRECONDITION, "shard finish: row range outside the final rows");
  // final dictionary: ascending ranks = ascending keys; word prefix for the join
  DBuf wpre;
  ensure(c, wpre, (size_t)(s->words + 1) * sizeof(u32));
  const long long N = extract(s, s->dict, nullptr, 0, nullptr, wpre.as<u32>());
  s->N = N;
  ensure(c, pl->dict, (size_t)std::max<long long>(N, 1) * KW * sizeof(u64));
  ensure(c, pl->dict_exps, (size_t)std::max<long long>(N, 1) * n * sizeof(u16));
  if (N)
    F4B_LAUNCH(c, (k_sh_unrank<KW, NV>), nbk(N, 256), 256, 0, s->bf.f, s->ranks.as<u32>(), N, (int)s->bf.D,
               s->bt.as<u32>(), s->st, pl->dict.as<u64>(), pl->dict_exps.as<u16>());
  // this rank's rows: row_ptr relative to its first term, then the join
  u32* h = c->h_stat;
  check_cuda(cudaMemcpyAsync(h, s->rows_start.as<u32>() + lo, 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
  check_cuda(cudaMemcpyAsync(h + 1, s->rows_start.as<u32>() + hi, 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  const long long Ml = (long long)h[1] - (long long)h[0];
  ensure(c, pl->row_ptr, (size_t)(hi - lo + 1) * sizeof(u32));
  ensure(c, pl->col_ind, (size_t)std::max<long long>(Ml, 1) * sizeof(u32));
  ensure(c, pl->val, (size_t)std::max<long long>(Ml, 1) * sizeof(u32));
  F4B_LAUNCH(c, k_sh_rowptr, nbk(hi - lo + 1, 256), 256, 0, s->rows_start.as<u32>(), lo, hi, pl->row_ptr.as<u32>());
  ensure(c, c->errflag, 64);
  check_cuda(cudaMemsetAsync(c->errflag.p, 0, 4, c->stream), "memset");
  if (hi > lo)
    F4B_LAUNCH(c, k_sh_join<KW>, (unsigned)std::min<long long>(nbk(hi - lo, 8), (long long)c->num_sms * 8), 256,
               (size_t)s->bt_words * 4, s->bf.f, lo, hi, s->rows_basis.as<int>(), s->rows_delta.as<u64>(),
               s->rows_start.as<u32>(), B.off.as<u32>(), B.len.as<u32>(), B.ckey.as<u64>(), B.coeff.as<u32>(),
               s->bt.as<u32>(), s->st, s->bt_words, s->dict, wpre.as<u32>(), (u32)N, pl->col_ind.as<u32>(),
               pl->val.as<u32>(), c->errflag.as<u32>());
  // closure-row metadata: all rounds (identical on every rank)
  const long long ncl = s->n_cl;
  ensure(c, pl->cl_basis, (size_t)std::max<long long>(ncl, 1) * sizeof(int));
  ensure(c, pl->cl_shift, (size_t)std::max<long long>(ncl, 1) * n * sizeof(u16));
  ensure(c, pl->cl_round, (size_t)std::max<long long>(ncl, 1) * sizeof(int));
  if (ncl) {
    check_cuda(cudaMemcpyAsync(pl->cl_basis.p, s->cl_basis.p, ncl * sizeof(int), cudaMemcpyDeviceToDevice, c->stream), "d2d");
    check_cuda(cudaMemcpyAsync(pl->cl_shift.p, s->cl_shift.p, ncl * n * sizeof(u16), cudaMemcpyDeviceToDevice, c->stream),
               "d2d");
    check_cuda(cudaMemcpyAsync(pl->cl_round.p, s->cl_round.p, ncl * sizeof(int), cudaMemcpyDeviceToDevice, c->stream), "d2d");
  }
  const u32 e = read_u32(c, c->errflag.as<u32>());
  if (e & DEVERR_LANE_OVERFLOW) fail(F4B_ERR_LANE_OVERFLOW, "shifted exponent overflows a 16-bit lane");
  if (e & DEVERR_MISSING_KEY) fail(F4B_ERR_MISSING_KEY, "row key absent from dictionary (closure defect)");
  release(c, wpre);
  pl->KW = KW;
  pl->lane_bits = s->bf.f.lane_bits;
  pl->r = hi - lo;
  pl->r0 = 0;
  pl->ncl_all = ncl;
  pl->row_lo = lo;
  pl->r_total = s->r;
  pl->N = N;
  pl->M = Ml;
  pl->closure_rounds = s->rounds;
  pl->dict_ns = s->ns;
  pl->asm_ns = 0;
}

// dispatch on (KW, NV) like compile_batch's fused path
template <class F>
auto dispatch(f4b_shard* s, F&& fn) {
  const int n = s->c->n_vars;
  const int KW = s->bf.KW;
  if (KW == 1 && n <= 8) return fn(std::integral_constant<int, 1>{}, std::integral_constant<int, 8>{});
  if (KW == 1 && n <= 16) return fn(std::integral_constant<int, 1>{}, std::integral_constant<int, 16>{});
  if (KW == 1) return fn(std::integral_constant<int, 1>{}, std::integral_constant<int, 32>{});
  if (n <= 16) return fn(std::integral_constant<int, 2>{}, std::integral_constant<int, 16>{});
  return fn(std::integral_constant<int, 2>{}, std::integral_constant<int, 32>{});
}

}  // namespace

// C ABI (include/f4b200.h) — bodies wrapped like the rest of capi.cu
#define SH_BEGIN(sh)                        \
  if (!(sh)) return F4B_ERR_PRECONDITION;   \
  Ctx* _c = (sh)->c;                        \
  try {
#define SH_END                              \
  }                                         \
  catch (const Error& e) {                  \
    _c->last_error = e.msg;                 \
    return e.code;                          \
  }                                         \
  return F4B_OK;

extern "C" {

int f4b_shard_begin(f4b_ctx* ctx, int64_t n_rows, const int32_t* row_basis, const uint16_t* row_shift, int closure,
                    const int32_t* candidates, int64_t n_candidates, int64_t dict_cap, int64_t row_lo, int64_t row_hi,
                    f4b_shard** out, int64_t* n_run) {
  if (!ctx || !out || !n_run || n_rows < 1 || row_lo < 0 || row_hi > n_rows || row_lo > row_hi)
    return F4B_ERR_PRECONDITION;
  Ctx* c = f4b_ctx_of(ctx);
  f4b_shard* s = new f4b_shard();
  s->c = c;
  try {
    basis_finish(c);
    check_cuda(cudaSetDevice(c->device), "cudaSetDevice");
    s->bf = batch_format(c, n_rows, row_basis, row_shift, candidates, n_candidates);
    if (!s->bf.rank_ok) fail(F4B_ERR_PRECONDITION, "sharded compile needs the grevlex rank path (rank space <= 2^26)");
    const int n = c->n_vars;
    s->closure = closure;
    s->dict_cap = dict_cap;
    s->r0 = n_rows;
    s->st = n + 1;
    s->bt_words = ((int)s->bf.D + n + 2) * s->st;
    s->words = (u32)((binom_ull(n + (int)s->bf.D, n) + 31) / 32);
    // LM table of the candidates in preference order (u16x2 per word)
    if (closure) {
      Basis& B = c->basis;
      std::vector<int32_t> pref = reducer_preference(c, s->bf.cand);
      s->nc = (int)pref.size();
      s->nw = (n + 1) / 2;
      std::vector<u32> h((size_t)std::max(s->nc, 1) * s->nw, 0u);
      for (int q = 0; q < s->nc; ++q)
        for (int v = 0; v < n; ++v) h[(size_t)q * s->nw + v / 2] |= (u32)B.h_lm[(size_t)pref[q] * n + v] << (16 * (v & 1));
      ensure(c, s->lmw, h.size() * 4);
      ensure(c, s->cidx, (size_t)std::max(s->nc, 1) * 4);
      check_cuda(cudaMemcpyAsync(s->lmw.p, h.data(), h.size() * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
      if (s->nc)
        check_cuda(cudaMemcpyAsync(s->cidx.p, pref.data(), (size_t)s->nc * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
    }
    ev_begin(s);
    *n_run = dispatch(s, [&](auto kw, auto nv) {
      return begin_t<decltype(kw)::value, decltype(nv)::value>(s, row_basis, row_shift, row_lo, row_hi);
    });
    ev_end(s);
  } catch (const Error& e) {
    c->last_error = e.msg;
    delete s;
    return e.code;
  }
  *out = s;
  return F4B_OK;
}

int f4b_shard_take_run(f4b_shard* sh, uint32_t* out, int64_t n) {
  SH_BEGIN(sh)
  if (n > 0) {
    check_cuda(cudaMemcpyAsync(out, sh->ranks.p, (size_t)n * 4, cudaMemcpyDefault, _c->stream), "run out");
    check_cuda(cudaStreamSynchronize(_c->stream), "sync");
  }
  SH_END
}

int f4b_shard_merge(f4b_shard* sh, const uint32_t* ranks, int64_t n, int64_t* n_frontier) {
  SH_BEGIN(sh)
  ev_begin(sh);
  *n_frontier = dispatch(sh, [&](auto kw, auto nv) { return merge_t<decltype(kw)::value, decltype(nv)::value>(sh, ranks, n); });
  ev_end(sh);
  SH_END
}

int f4b_shard_round(f4b_shard* sh, int64_t f_lo, int64_t f_hi, int32_t* red_out, int64_t* n_run) {
  SH_BEGIN(sh)
  if (f_lo < 0 || f_hi > sh->nf || f_lo > f_hi) fail(F4B_ERR_PRECONDITION, "shard round: slice outside the frontier");
  ev_begin(sh);
  *n_run = dispatch(sh, [&](auto kw, auto nv) {
    return round_t<decltype(kw)::value, decltype(nv)::value>(sh, f_lo, f_hi, red_out);
  });
  ev_end(sh);
  SH_END
}

int f4b_shard_round_merge(f4b_shard* sh, const int32_t* red_all, int64_t nf, const uint32_t* ranks, int64_t n,
                          int64_t* n_frontier) {
  SH_BEGIN(sh)
  ev_begin(sh);
  *n_frontier = dispatch(sh, [&](auto kw, auto nv) {
    return round_merge_t<decltype(kw)::value, decltype(nv)::value>(sh, red_all, nf, ranks, n);
  });
  ev_end(sh);
  SH_END
}

int f4b_shard_rows(f4b_shard* sh, int64_t* r_total, uint32_t* row_start) {
  SH_BEGIN(sh)
  *r_total = sh->r;
  if (row_start) {
    check_cuda(cudaMemcpyAsync(row_start, sh->rows_start.p, (size_t)(sh->r + 1) * 4, cudaMemcpyDefault, _c->stream),
               "rows out");
    check_cuda(cudaStreamSynchronize(_c->stream), "sync");
  }
  SH_END
}

int f4b_shard_finish(f4b_shard* sh, int64_t row_lo, int64_t row_hi, f4b_plan** out) {
  SH_BEGIN(sh)
  f4b_plan* pl = new f4b_plan();
  pl->ctx = _c;
  try {
    ev_begin(sh);
    dispatch(sh, [&](auto kw, auto nv) {
      finish_t<decltype(kw)::value, decltype(nv)::value>(sh, row_lo, row_hi, pl);
      return 0;
    });
    ev_end(sh);
    pl->dict_ns = sh->ns;
  } catch (...) {
    plan_release(pl);
    throw;
  }
  *out = pl;
  SH_END
}

int f4b_shard_info(const f4b_shard* sh, int64_t* rounds, int64_t* n_dict, int64_t* device_ns) {
  if (!sh) return F4B_ERR_PRECONDITION;
  if (rounds) *rounds = sh->rounds;
  if (n_dict) *n_dict = sh->N;
  if (device_ns) *device_ns = sh->ns;
  return F4B_OK;
}

int f4b_shard_free(f4b_shard* sh) {
  if (!sh) return F4B_OK;
  Ctx* c = sh->c;
  for (DBuf* b : {&sh->bt, &sh->stage, &sh->rows_basis, &sh->rows_delta, &sh->rows_start, &sh->cl_basis, &sh->cl_shift,
                  &sh->cl_round, &sh->maps, &sh->front, &sh->red, &sh->ranks, &sh->scan_a, &sh->scan_b, &sh->lmw,
                  &sh->cidx})
    release(c, *b);
  delete sh;
  return F4B_OK;
}

}  // extern "C"
