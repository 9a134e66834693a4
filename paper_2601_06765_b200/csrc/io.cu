// Wire / disk formats streamed from device buffers and the
// device transpose of the public csr_transpose (§8a a23).
//
//   f4b_plan_text      the number lists of plan_to_text (reference
//                      symbolic.py:438-460: row_ptr, col_ind, val, dict_keys as
//                      decimal text, one space between numbers) formatted on
//                      the device: digit counts -> exclusive scan -> digits.
//                      One D2H of the text; the host adds the header lines.
//   f4b_csr_transpose  stable counting-sort transpose (reference
//                      sparselin.py:108-121): keys (col << 32 | row) sorted by
//                      the one-sweep radix sort (radix.cu; the pairs are
//                      unique, so sort == stable order), column counts ->
//                      scan -> row_ptr of the transpose, values found by a
//                      binary search in the source row.
//   f4b_plan_validate  LayoutPlan.validate (reference symbolic.py:125-163) on
//                      the device buffers: one pass over rows, terms and
//                      dictionary entries; the first violation in the
//                      reference's check order wins (atomicMin of
//                      reason << 40 | index), so the message names the same
//                      row the host check would.
#include <algorithm>
#include <cstring>
#include <string>

#include "common.cuh"
#include "engine.h"

f4b::Ctx* f4b_ctx_of(f4b_ctx* h);  // capi.cu

namespace f4b {

static inline unsigned nbi(long long n, int t) { return (unsigned)std::max<long long>(1, (n + t - 1) / t); }

F4B_DEV int ndigits(unsigned long long v) {
  int d = 1;
  while (v >= 10ull) {
    v /= 10ull;
    ++d;
  }
  return d;
}

template <typename T>
__global__ void k_txt_len(const T* __restrict__ v, long long n, u32* __restrict__ len) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) len[i] = (u32)ndigits((unsigned long long)v[i]) + (i > 0 ? 1u : 0u);
}

template <typename T>
__global__ void k_txt_write(const T* __restrict__ v, long long n, const u32* __restrict__ off, char* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= n) return;
  unsigned long long x = (unsigned long long)v[i];
  u32 o = off[i];
  if (i > 0) out[o++] = ' ';
  const int d = ndigits(x);
  for (int k = d - 1; k >= 0; --k) {
    out[o + k] = (char)('0' + (int)(x % 10ull));
    x /= 10ull;
  }
}

template <typename T>
static long long format_list(Ctx* c, const T* dv, long long n, char* host_out, long long cap) {
  if (n == 0) return 0;
  if (n >= (1ll << 31)) fail(F4B_ERR_SIZE_CAP, "plan_text: list longer than 2^31");
  DBuf len, off, txt;
  ensure(c, len, (size_t)(n + 1) * 4);
  ensure(c, off, (size_t)(n + 1) * 4);
  F4B_LAUNCH(c, k_txt_len<T>, nbi(n, 256), 256, 0, dv, n, len.as<u32>());
  exclusive_scan_u32(c, len.as<u32>(), off.as<u32>(), n);  // 21 bytes per number at most: < 2^32 for n < 2^27
  const long long tot = read_u32(c, off.as<u32>() + n);
  if (host_out && tot <= cap) {
    ensure(c, txt, (size_t)tot);
    F4B_LAUNCH(c, k_txt_write<T>, nbi(n, 256), 256, 0, dv, n, off.as<u32>(), txt.as<char>());
    check_cuda(cudaMemcpyAsync(host_out, txt.p, (size_t)tot, cudaMemcpyDeviceToHost, c->stream), "d2h text");
    check_cuda(cudaStreamSynchronize(c->stream), "sync");
  }
  release(c, len);
  release(c, off);
  release(c, txt);
  return tot;
}

__global__ void k_tr_keys(const long long* __restrict__ rp, const long long* __restrict__ col, long long r,
                          unsigned long long* __restrict__ keys, u32* __restrict__ ccount) {
  const long long row = ((long long)blockIdx.x * blockDim.x + threadIdx.x) >> 5;
  const int lane = threadIdx.x & 31;
  if (row >= r) return;
  for (long long k = rp[row] + lane; k < rp[row + 1]; k += 32) {
    keys[k] = ((unsigned long long)col[k] << 32) | (unsigned long long)row;
    atomicAdd(ccount + col[k], 1u);
  }
}

__global__ void k_tr_fill(const unsigned long long* __restrict__ keys, long long nnz, const long long* __restrict__ rp,
                          const long long* __restrict__ col, const unsigned long long* __restrict__ val,
                          long long* __restrict__ tcol, unsigned long long* __restrict__ tval) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= nnz) return;
  const unsigned long long k = keys[i];
  const long long c = (long long)(k >> 32), row = (long long)(k & 0xFFFFFFFFull);
  long long lo = rp[row], hi = rp[row + 1];  // columns ascending within the row
  while (lo + 1 < hi) {
    const long long mid = (lo + hi) >> 1;
    if (col[mid] <= c) lo = mid; else hi = mid;
  }
  tcol[i] = row;
  tval[i] = val[lo];
}

__global__ void k_u32_to_i64(const u32* __restrict__ in, long long n, long long* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i < n) out[i] = in[i];
}


// violation keys, ordered like the reference's checks (symbolic.py:133-154):
// tiling, negative segment, then per row (empty, ascending, range), zero
// value, dictionary order; an unreduced value (>= p, never produced by a
// compile) is reported last
enum : unsigned long long {
  V_TILE = 1ull << 40,
  V_NEG = 2ull << 40,
  V_ROW = 3ull << 40,  // | row * 4 + {0 empty, 1 ascending, 2 range}
  V_ZERO = 4ull << 40,
  V_DICT = 5ull << 40,
  V_UNRED = 6ull << 40,
};

F4B_DEV long long row_of(const u32* __restrict__ rp, long long r, long long t) {
  long long lo = 0, hi = r;  // rp[lo] <= t < rp[hi]
  while (lo + 1 < hi) {
    const long long mid = (lo + hi) >> 1;
    if ((long long)rp[mid] <= t) lo = mid; else hi = mid;
  }
  return lo;
}

// key(a) > key(b) in the ring order (monomials.py:131-148 key layout):
// grevlex (0) / deglex (1) by degree first; then grevlex by the reversed
// complemented exponents, deglex and lex (2) by the exponents
F4B_DEV bool mono_gt(const uint16_t* a, const uint16_t* b, int n, int order) {
  if (order != 2) {
    u32 da = 0, db = 0;
    for (int v = 0; v < n; ++v) {
      da += a[v];
      db += b[v];
    }
    if (da != db) return da > db;
  }
  for (int l = 0; l < n; ++l) {
    const u32 x = order == 0 ? 0xFFFFu - a[n - 1 - l] : a[l];
    const u32 y = order == 0 ? 0xFFFFu - b[n - 1 - l] : b[l];
    if (x != y) return x > y;
  }
  return false;
}

F4B_DEV void validate_body(const u32* __restrict__ rp, long long r, const u32* __restrict__ col,
                           const u32* __restrict__ val, long long M, long long N, u32 p,
                           const uint16_t* __restrict__ dex, int n, int order, unsigned long long* __restrict__ flag) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long t0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  unsigned long long f = ~0ull;
  if (t0 == 0 && (rp[0] != 0 || (long long)rp[r] != M)) f = V_TILE;
  for (long long i = t0; i < r; i += stride) {
    const u32 a = rp[i], b = rp[i + 1];
    if (b < a) f = min(f, V_NEG | (unsigned long long)i);
    else if (b == a) f = min(f, V_ROW | (unsigned long long)(i * 4));
  }
  for (long long t = t0; t < M; t += stride) {
    const u32 c = col[t], v = val[t];
    if (v == 0) f = min(f, V_ZERO | (unsigned long long)t);
    else if (v >= p) f = min(f, V_UNRED | (unsigned long long)t);
    const bool range = (long long)c >= N;
    const bool desc = t + 1 < M && col[t + 1] <= c;
    if (range || desc) {
      const long long i = row_of(rp, r, t);
      if (range) f = min(f, V_ROW | (unsigned long long)(i * 4 + 2));
      if (desc && (long long)rp[i + 1] != t + 1) f = min(f, V_ROW | (unsigned long long)(i * 4 + 1));
    }
  }
  for (long long k = t0; k + 1 < N; k += stride)
    if (!mono_gt(dex + k * n, dex + (k + 1) * n, n, order)) f = min(f, V_DICT | (unsigned long long)k);
  if (f != ~0ull) atomicMin(flag, f);
}

__global__ void k_validate(const u32* __restrict__ rp, long long r, const u32* __restrict__ col,
                           const u32* __restrict__ val, long long M, long long N, u32 p,
                           const uint16_t* __restrict__ dex, int n, int order, unsigned long long* __restrict__ flag) {
  validate_body(rp, r, col, val, M, N, p, dex, n, order, flag);
}

// sizes on the device (behind the compile kernel, no host round trip)
__global__ void k_validate_dev(const u32* __restrict__ rp, const u32* __restrict__ col, const u32* __restrict__ val,
                               const u32* __restrict__ sz, u32 p, const uint16_t* __restrict__ dex, int n, int order,
                               unsigned long long* __restrict__ flag) {
  if (sz[6]) return;  // LoopOut.flags: an aborted (re-run) compile, sizes not final
  validate_body(rp, sz[0], col, val, sz[2], sz[3], p, dex, n, order, flag);
}

void validate_launch_dev(Ctx* c, const f4b_plan* pl, const uint32_t* sz, unsigned long long* flag) {
  check_cuda(cudaMemsetAsync(flag, 0xFF, 8, c->stream), "memset");
  F4B_LAUNCH(c, k_validate_dev, (unsigned)(c->num_sms * 4), 256, 0, pl->row_ptr.as<u32>(), pl->col_ind.as<u32>(),
             pl->val.as<u32>(), sz, c->p, pl->dict_exps.as<uint16_t>(), c->n_vars, c->order, flag);
}

std::string validate_message(unsigned long long f, long long row_lo) {
  const unsigned long long kind = f >> 40, idx = f & ((1ull << 40) - 1);
  const long long row = row_lo + (long long)(idx >> 2);
  switch (kind) {
    case 1: return "row_ptr does not tile the value stream";
    case 2: return "negative row segment length";
    case 3:
      return (idx & 3) == 0 ? "empty row " + std::to_string(row) + " (basis members are nonzero)"
             : (idx & 3) == 1 ? "row " + std::to_string(row) + " columns not strictly ascending"
                              : "row " + std::to_string(row) + " column out of range";
    case 4: return "zero value stored in plan";
    case 5: return "dictionary keys not strictly descending";
    default: return "value not reduced mod p at term " + std::to_string(idx);
  }
}

}  // namespace f4b

using namespace f4b;

extern "C" {

int f4b_plan_text(const f4b_plan* pl, int which, char* out, int64_t cap, int64_t* length) {
  if (!pl || !length || which < 0 || which > 3) return F4B_ERR_PRECONDITION;
  Ctx* c = pl->ctx;
  try {
    long long tot = 0;
    switch (which) {
      case 0: tot = format_list<u32>(c, pl->row_ptr.as<u32>(), pl->r + 1, out, cap); break;
      case 1: tot = format_list<u32>(c, pl->col_ind.as<u32>(), pl->M, out, cap); break;
      case 2: tot = format_list<u32>(c, pl->val.as<u32>(), pl->M, out, cap); break;
      default: {
        const int W = ((c->order == 2 ? 0 : 32) + 16 * c->n_vars + 63) / 64;
        DBuf kb;
        ensure(c, kb, (size_t)std::max<long long>(pl->N, 1) * W * 8);
        ref_keys_device(c, pl, kb.as<unsigned long long>(), W);
        tot = format_list<unsigned long long>(c, kb.as<unsigned long long>(), pl->N * W, out, cap);
        release(c, kb);
      }
    }
    *length = tot;
  } catch (const Error& e) {
    c->last_error = e.msg;
    return e.code;
  }
  return F4B_OK;
}

int f4b_plan_validate(const f4b_plan* pl, int64_t* violation) {
  if (!pl) return F4B_ERR_PRECONDITION;
  Ctx* c = pl->ctx;
  try {
    DBuf fl;
    ensure(c, fl, 8);
    check_cuda(cudaMemsetAsync(fl.p, 0xFF, 8, c->stream), "memset");
    const long long work = std::max({pl->r, pl->M, pl->N, 1ll});
    const unsigned g = (unsigned)std::min<long long>(nbi(work, 256), 148ll * 8);
    F4B_LAUNCH(c, k_validate, g, 256, 0, pl->row_ptr.as<u32>(), pl->r, pl->col_ind.as<u32>(), pl->val.as<u32>(),
               pl->M, pl->N, c->p, pl->dict_exps.as<uint16_t>(), c->n_vars, c->order, fl.as<unsigned long long>());
    unsigned long long f = 0;
    check_cuda(cudaMemcpyAsync(&f, fl.p, 8, cudaMemcpyDeviceToHost, c->stream), "d2h");
    check_cuda(cudaStreamSynchronize(c->stream), "sync");
    release(c, fl);
    if (violation) *violation = f == ~0ull ? -1 : (int64_t)f;
    if (f != ~0ull) fail(F4B_ERR_PROPERTY, validate_message(f, pl->row_lo));
  } catch (const Error& e) {
    c->last_error = e.msg;
    return e.code;
  }
  return F4B_OK;
}

// fault injection for the validation tests: overwrite one u32 entry of the
// plan's row_ptr (0), col_ind (1) or val (2) on the device
int f4b_plan_poke(f4b_plan* pl, int which, int64_t index, uint32_t value) {
  if (!pl || which < 0 || which > 2 || index < 0) return F4B_ERR_PRECONDITION;
  const long long len = which == 0 ? pl->r + 1 : pl->M;
  if (index >= len) return F4B_ERR_PRECONDITION;
  Ctx* c = pl->ctx;
  u32* base = (which == 0 ? pl->row_ptr : which == 1 ? pl->col_ind : pl->val).as<u32>();
  try {
    check_cuda(cudaMemcpyAsync(base + index, &value, 4, cudaMemcpyHostToDevice, c->stream), "h2d");
    check_cuda(cudaStreamSynchronize(c->stream), "sync");
  } catch (const Error& e) {
    c->last_error = e.msg;
    return e.code;
  }
  return F4B_OK;
}

int f4b_csr_transpose(f4b_ctx* ctx, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col_ind,
                      const uint64_t* val, int64_t* t_row_ptr, int64_t* t_col_ind, uint64_t* t_val) {
  if (!ctx || n_rows < 0 || n_cols < 0) return F4B_ERR_PRECONDITION;
  Ctx* c = f4b_ctx_of(ctx);
  try {
    const long long nnz = row_ptr[n_rows];
    if (n_rows >= (1ll << 32) - 1 || n_cols >= (1ll << 31) || nnz >= (1ll << 32) - 2)
      fail(F4B_ERR_SIZE_CAP, "csr_transpose: rows < 2^32 - 1, columns < 2^31, nnz < 2^32 - 2");
    for (long long i = 0; i < n_rows; ++i)
      if (row_ptr[i + 1] < row_ptr[i]) fail(F4B_ERR_PROPERTY, "row_ptr not monotone");
    DBuf drp, dcol, dval, keys, sk, cnt, tcp, tc, tv, d_count;
    ensure(c, drp, (size_t)(n_rows + 1) * 8);
    ensure(c, dcol, (size_t)std::max<long long>(nnz, 1) * 8);
    ensure(c, dval, (size_t)std::max<long long>(nnz, 1) * 8);
    ensure(c, cnt, (size_t)(n_cols + 1) * 4);
    ensure(c, tcp, (size_t)(n_cols + 1) * 4);
    check_cuda(cudaMemcpyAsync(drp.p, row_ptr, (size_t)(n_rows + 1) * 8, cudaMemcpyHostToDevice, c->stream), "h2d");
    if (nnz) {
      check_cuda(cudaMemcpyAsync(dcol.p, col_ind, (size_t)nnz * 8, cudaMemcpyHostToDevice, c->stream), "h2d");
      check_cuda(cudaMemcpyAsync(dval.p, val, (size_t)nnz * 8, cudaMemcpyHostToDevice, c->stream), "h2d");
    }
    check_cuda(cudaMemsetAsync(cnt.p, 0, (size_t)(n_cols + 1) * 4, c->stream), "memset");
    if (nnz) {
      ensure(c, keys, (size_t)nnz * 8);
      ensure(c, sk, (size_t)nnz * 8);
      ensure(c, d_count, 16);
      F4B_LAUNCH(c, k_tr_keys, nbi(n_rows * 32, 256), 256, 0, drp.as<long long>(), dcol.as<long long>(), n_rows,
                 keys.as<unsigned long long>(), cnt.as<u32>());
      int bits = 32;
      while (bits < 64 && (1ll << (bits - 32)) < n_cols) ++bits;
      sort_unique(c, 1, keys.as<uint64_t>(), nullptr, (uint32_t)nnz, bits, nullptr, nullptr, sk.as<uint64_t>(),
                  d_count.as<uint32_t>());
      if ((long long)read_u32(c, d_count.as<uint32_t>()) != nnz)
        fail(F4B_ERR_PROPERTY, "csr_transpose: duplicate (row, column) entries");
      ensure(c, tc, (size_t)nnz * 8);
      ensure(c, tv, (size_t)nnz * 8);
      F4B_LAUNCH(c, k_tr_fill, nbi(nnz, 256), 256, 0, sk.as<unsigned long long>(), nnz, drp.as<long long>(),
                 dcol.as<long long>(), dval.as<unsigned long long>(), tc.as<long long>(), tv.as<unsigned long long>());
      check_cuda(cudaMemcpyAsync(t_col_ind, tc.p, (size_t)nnz * 8, cudaMemcpyDeviceToHost, c->stream), "d2h");
      check_cuda(cudaMemcpyAsync(t_val, tv.p, (size_t)nnz * 8, cudaMemcpyDeviceToHost, c->stream), "d2h");
    }
    exclusive_scan_u32(c, cnt.as<u32>(), tcp.as<u32>(), n_cols);
    DBuf trp64;
    ensure(c, trp64, (size_t)(n_cols + 1) * 8);
    F4B_LAUNCH(c, k_u32_to_i64, nbi(n_cols + 1, 256), 256, 0, tcp.as<u32>(), n_cols + 1, trp64.as<long long>());
    check_cuda(cudaMemcpyAsync(t_row_ptr, trp64.p, (size_t)(n_cols + 1) * 8, cudaMemcpyDeviceToHost, c->stream), "d2h");
    check_cuda(cudaStreamSynchronize(c->stream), "sync");
    for (DBuf* b : {&drp, &dcol, &dval, &keys, &sk, &cnt, &tcp, &tc, &tv, &d_count, &trp64}) release(c, *b);
  } catch (const Error& e) {
    c->last_error = e.msg;
    return e.code;
  }
  return F4B_OK;
}

}  // extern "C"
