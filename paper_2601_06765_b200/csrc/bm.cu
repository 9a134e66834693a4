// Berlekamp–Massey on the device (reference sparselin.py:377-413, SURVEY.md
// §8a row a24): the minimal recurrence of each Krylov projection sequence of
// Block Wiedemann.  The reference runs the scalar recurrence in pure Python,
// O(len²) per sequence; at MQ-16 / F_31 sizes (len = 2·dim up to ~41k) that
// is the whole cost of a Wiedemann F4 step.  Here one CTA per sequence runs
// the same recurrence — same connection / previous polynomials, same gap and
// length updates, so the output polynomial is identical — with the
// discrepancy as a block-wide dot product and the update as a block-wide
// axpy; the b sequences of a round run side by side.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "engine.h"

f4b::Ctx* f4b_ctx_of(f4b_ctx* h);

namespace f4b {

Fp make_fp_pub(Ctx* c);

static constexpr int BM_THREADS = 1024;

// seqs [b][len] (standard residues), work [b][3][len + 2], out_conn [b][len + 1],
// out_L [b].  SMALLP: p < 2^16, products < 2^32 summed lazily in u64.
template <bool SMALLP>
__global__ void __launch_bounds__(BM_THREADS) k_bm(Fp fp, const u32* __restrict__ seqs, long long len,
                                                   u32* __restrict__ work, u32* __restrict__ out_conn,
                                                   long long* __restrict__ out_L) {
  const u32 p = fp.p;
  const u32* s = seqs + (size_t)blockIdx.x * len;
  u32* buf0 = work + (size_t)blockIdx.x * 3 * (len + 2);
  u32* conn = buf0;
  u32* prev = buf0 + (len + 2);
  u32* tmp = buf0 + 2 * (len + 2);
  __shared__ unsigned long long red[BM_THREADS / 32];
  const int tid = threadIdx.x, lane = tid & 31, warp = tid >> 5;
  if (tid == 0) {
    conn[0] = 1;
    prev[0] = 1;
  }
  long long L = 0, gap = 1, lenc = 1, lenp = 1;
  u32 inv_last = 1;  // inverse of the last nonzero discrepancy (initially 1)
  __syncthreads();
  for (long long n = 0; n < len; ++n) {
    // discrepancy d = s[n] + sum_{i=1..L} conn[i] s[n-i]
    unsigned long long part = 0;
    u32 partm = 0;
    for (long long i = 1 + tid; i <= L; i += BM_THREADS) {
      if (SMALLP)
        part += (unsigned long long)conn[i] * s[n - i];
      else
        partm = fp.add(partm, fp.mul(conn[i], s[n - i]));
    }
    if (!SMALLP) part = partm;
#pragma unroll
    for (int o = 16; o; o >>= 1) part += __shfl_xor_sync(0xffffffffu, part, o);
    if (lane == 0) red[warp] = SMALLP ? part : part % p;
    __syncthreads();
    unsigned long long tot = s[n];
    for (int w = 0; w < BM_THREADS / 32; ++w) tot += red[w];
    const u32 d = (u32)(tot % p);
    __syncthreads();  // red[] reused next iteration
    if (d == 0) {
      ++gap;
      continue;
    }
    const u32 scale = fp.mul(d, inv_last);
    const long long need = lenp + gap, newlen = std::max(lenc, need);
    if (2 * L <= n) {
      // conn' = conn - scale x^gap prev into tmp; prev <- conn; conn <- tmp
      for (long long i = tid; i < newlen; i += BM_THREADS) {
        u32 v = i < lenc ? conn[i] : 0u;
        const long long j = i - gap;
        if (j >= 0 && j < lenp) v = fp.sub(v, fp.mul(scale, prev[j]));
        tmp[i] = v;
      }
      u32* t = prev;
      prev = conn;
      conn = tmp;
      tmp = t;
      lenp = lenc;
      lenc = newlen;
      L = n + 1 - L;
      inv_last = fp.inv(d);
      gap = 1;
    } else {
      for (long long i = lenc + tid; i < newlen; i += BM_THREADS) conn[i] = 0;
      __syncthreads();
      for (long long j = tid; j < lenp; j += BM_THREADS) conn[j + gap] = fp.sub(conn[j + gap], fp.mul(scale, prev[j]));
      lenc = newlen;
      ++gap;
    }
    __syncthreads();
  }
  // conn[0..L] (zero padded when shorter)
  u32* o = out_conn + (size_t)blockIdx.x * (len + 1);
  for (long long i = tid; i <= L; i += BM_THREADS) o[i] = i < lenc ? conn[i] : 0u;
  if (tid == 0) out_L[blockIdx.x] = L;
}

}  // namespace f4b

using namespace f4b;

extern "C" {

int f4b_bm(f4b_ctx* h, const uint64_t* seqs, int64_t len, int64_t b, uint64_t* polys, int64_t* degrees) {
  if (!h || len < 1 || b < 1 || !seqs || !polys || !degrees) return F4B_ERR_PRECONDITION;
  Ctx* c = f4b_ctx_of(h);
  try {
    const size_t nseq = (size_t)b * len;
    std::vector<u32> hs(nseq);
    for (size_t i = 0; i < nseq; ++i) hs[i] = (u32)(seqs[i] % c->p);
    DBuf ds, work, oc, ol;
    ensure(c, ds, nseq * 4);
    ensure(c, work, (size_t)b * 3 * (len + 2) * 4);
    ensure(c, oc, (size_t)b * (len + 1) * 4);
    ensure(c, ol, (size_t)b * 8);
    check_cuda(cudaMemcpyAsync(ds.p, hs.data(), nseq * 4, cudaMemcpyHostToDevice, c->stream), "h2d seqs");
    Fp fp = make_fp_pub(c);
    if (c->p < 65536u)
      F4B_LAUNCH(c, k_bm<true>, (int)b, BM_THREADS, 0, fp, ds.as<u32>(), (long long)len, work.as<u32>(), oc.as<u32>(),
                 ol.as<long long>());
    else
      F4B_LAUNCH(c, k_bm<false>, (int)b, BM_THREADS, 0, fp, ds.as<u32>(), (long long)len, work.as<u32>(), oc.as<u32>(),
                 ol.as<long long>());
    std::vector<u32> hc((size_t)b * (len + 1));
    check_cuda(cudaMemcpyAsync(hc.data(), oc.p, hc.size() * 4, cudaMemcpyDeviceToHost, c->stream), "d2h conn");
    check_cuda(cudaMemcpyAsync(degrees, ol.p, (size_t)b * 8, cudaMemcpyDeviceToHost, c->stream), "d2h L");
    check_cuda(cudaStreamSynchronize(c->stream), "sync");
    // reference output: [c % p for c in reversed(conn[:L + 1])] (ascending,
    // monic), written as polys[j][0..L]
    for (int64_t j = 0; j < b; ++j) {
      const int64_t L = degrees[j];
      const u32* cj = hc.data() + (size_t)j * (len + 1);
      for (int64_t i = 0; i <= L; ++i) polys[(size_t)j * (len + 1) + i] = cj[L - i];
    }
    release(c, ds);
    release(c, work);
    release(c, oc);
    release(c, ol);
  } catch (const Error& e) {
    c->last_error = e.msg;
    return e.code;
  }
  return F4B_OK;
}

}  // extern "C"
