// Device-resident black-box operator for Block Wiedemann (reference
// sparselin.py:450-548).
//
// The reference applies B = A (square) or B = AᵀA (rectangular) 2·dim times
// per round through `spmm`, each call a fresh host round trip.  Here the CSR
// of A (and Aᵀ, built once by a counting sort on the host) stays in HBM and
// the Krylov sequence  seq[k][j] = Σ_i U[i][j] · (B^k V)[i][j]  is produced by
// one fused launch per application (warp per output row: the row of B·W and,
// from the W it reads, the projection U·W of step k), with the projections
// accumulated on the device and read back once.  The generator evaluation
// acc = g[L-1] v;  acc = B acc + g[i] v  (Horner, reference :425-429) is the
// same kernel with an axpy term.  Arithmetic is exact mod p, so the sequences
// and vectors are bit-identical to the reference's NumPy loop.
#include <algorithm>
#include <cstring>
#include <vector>

#include "common.cuh"
#include "engine.h"

struct f4b_op {
  f4b::Ctx* ctx = nullptr;
  long long n_rows = 0, n_cols = 0, dim = 0;
  int normal = 0;  // 1: B = AᵀA (A is n_rows x n_cols, dim = n_cols)
  f4b::DBuf rp, col, val;     // A   (u32 CSR)
  f4b::DBuf trp, tcol, tval;  // Aᵀ  (normal only)
  f4b::DBuf w0, w1, t, v, u, acc;  // work vectors [dim or n_rows][b]; acc u64 [steps][b]
};

namespace f4b {

// Y[row][j] = Σ_k val[k] X[col[k]][j] (+ c · Z[row][j]); optionally the step
// projection acc[j] += Σ_row U[row][j] · X[row][j] (X square: same index space).
__global__ void k_op_apply(Fp fp, const u32* __restrict__ rp, const u32* __restrict__ col, const u32* __restrict__ val,
                           long long r, const u32* __restrict__ X, int b, u32* __restrict__ Y, u32 cmul,
                           const u32* __restrict__ Z, const u32* __restrict__ U, unsigned long long* __restrict__ proj) {
  const long long row = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (row >= r) return;
  const u32 s = rp[row], e = rp[row + 1];
  for (int j = 0; j < b; ++j) {
    unsigned long long a = 0;  // < 32 reduced products per lane between reductions
    for (u32 k = s + lane; k < e; k += 32) {
      a += fp.mul(__ldg(val + k), __ldg(X + (size_t)__ldg(col + k) * b + j));
      if (a >= (1ull << 62)) a %= fp.p;
    }
    a %= fp.p;
#pragma unroll
    for (int o = 16; o; o >>= 1) a = (a + __shfl_xor_sync(0xffffffffu, a, o)) % fp.p;
    if (lane == 0) {
      u32 y = (u32)a;
      if (Z) y = fp.add(y, fp.mul(cmul, Z[(size_t)row * b + j]));
      Y[(size_t)row * b + j] = y;
      if (proj) atomicAdd(proj + j, (unsigned long long)fp.mul(U[(size_t)row * b + j], X[(size_t)row * b + j]));
    }
  }
}

// b = 4 (the reference's block width): one pass over the row's nonzeros for
// all four columns (one 16-byte gather of X per nonzero), products summed
// lazily in u64 (SMALLP: p < 2^16, raw products < 2^32; else exact residues
// < 2^31) with a single reduction mod p per output after the warp sum.
template <bool SMALLP>
__global__ void k_op_apply4(Fp fp, const u32* __restrict__ rp, const u32* __restrict__ col,
                            const u32* __restrict__ val, long long r, const uint4* __restrict__ X,
                            uint4* __restrict__ Y, u32 cmul, const uint4* __restrict__ Z,
                            const uint4* __restrict__ U, unsigned long long* __restrict__ proj) {
  const long long row = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (row >= r) return;
  const u32 s = rp[row], e = rp[row + 1];
  unsigned long long a0 = 0, a1 = 0, a2 = 0, a3 = 0;
  auto term = [&](u32 v, const uint4& x) {
    if (SMALLP) {
      a0 += (unsigned long long)v * x.x;
      a1 += (unsigned long long)v * x.y;
      a2 += (unsigned long long)v * x.z;
      a3 += (unsigned long long)v * x.w;
    } else {
      const u32 vm = fp.to_mont(v);
      a0 += fp.mont_mul(vm, x.x);
      a1 += fp.mont_mul(vm, x.y);
      a2 += fp.mont_mul(vm, x.z);
      a3 += fp.mont_mul(vm, x.w);
    }
  };
  u32 k = s + lane;
  for (; k + 32 < e; k += 64) {
    const u32 c0 = __ldg(col + k), c1 = __ldg(col + k + 32);
    const u32 v0 = __ldg(val + k), v1 = __ldg(val + k + 32);
    const uint4 x0 = __ldg(X + c0), x1 = __ldg(X + c1);
    term(v0, x0);
    term(v1, x1);
  }
  if (k < e) term(__ldg(val + k), __ldg(X + __ldg(col + k)));
#pragma unroll
  for (int o = 16; o; o >>= 1) {
    a0 += __shfl_xor_sync(0xffffffffu, a0, o);
    a1 += __shfl_xor_sync(0xffffffffu, a1, o);
    a2 += __shfl_xor_sync(0xffffffffu, a2, o);
    a3 += __shfl_xor_sync(0xffffffffu, a3, o);
  }
  if (lane == 0) {
    const u32 p = fp.p;
    uint4 y = make_uint4((u32)(a0 % p), (u32)(a1 % p), (u32)(a2 % p), (u32)(a3 % p));
    if (Z) {
      const uint4 z = Z[row];
      y.x = fp.add(y.x, fp.mul(cmul, z.x));
      y.y = fp.add(y.y, fp.mul(cmul, z.y));
      y.z = fp.add(y.z, fp.mul(cmul, z.z));
      y.w = fp.add(y.w, fp.mul(cmul, z.w));
    }
    Y[row] = y;
    if (proj) {
      const uint4 u = U[row], x = X[row];
      atomicAdd(proj + 0, (unsigned long long)fp.mul(u.x, x.x));
      atomicAdd(proj + 1, (unsigned long long)fp.mul(u.y, x.y));
      atomicAdd(proj + 2, (unsigned long long)fp.mul(u.z, x.z));
      atomicAdd(proj + 3, (unsigned long long)fp.mul(u.w, x.w));
    }
  }
}

// acc[j] += Σ_i U[i][j] X[i][j] (when the projection cannot ride on the apply)
__global__ void k_op_proj(Fp fp, const u32* __restrict__ U, const u32* __restrict__ X, long long n, int b,
                          unsigned long long* __restrict__ proj) {
  for (int j = 0; j < b; ++j) {
    unsigned long long a = 0;
    for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
      a += fp.mul(U[(size_t)i * b + j], X[(size_t)i * b + j]);
#pragma unroll
    for (int o = 16; o; o >>= 1) a += __shfl_xor_sync(0xffffffffu, a, o);
    if ((threadIdx.x & 31) == 0 && a) atomicAdd(proj + j, a % fp.p);
  }
}

__global__ void k_any_nonzero(const u32* __restrict__ X, long long n, u32* __restrict__ flag) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    if (X[i]) {
      *flag = 1;
      return;
    }
}

Fp make_fp_pub(Ctx* c);

static void upload_csr(Ctx* c, long long r, const int64_t* rp, const int64_t* col, const uint64_t* val, DBuf& drp,
                       DBuf& dcol, DBuf& dval) {
  const long long M = rp[r];
  if (M >= (1ll << 32)) fail(F4B_ERR_SIZE_CAP, "operator has more than 2^32 nonzeros");
  std::vector<u32> hrp(r + 1), hcol(std::max<long long>(M, 1)), hval(std::max<long long>(M, 1));
  for (long long i = 0; i <= r; ++i) hrp[i] = (u32)rp[i];
  for (long long k = 0; k < M; ++k) {
    hcol[k] = (u32)col[k];
    hval[k] = (u32)(val[k] % c->p);
  }
  ensure(c, drp, (r + 1) * 4);
  ensure(c, dcol, hcol.size() * 4);
  ensure(c, dval, hval.size() * 4);
  check_cuda(cudaMemcpyAsync(drp.p, hrp.data(), (r + 1) * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
  check_cuda(cudaMemcpyAsync(dcol.p, hcol.data(), hcol.size() * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
  check_cuda(cudaMemcpyAsync(dval.p, hval.data(), hval.size() * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
}

// W_out = B W_in (+ cmul * Z); proj (optional) += U · W_in
static void apply_rows(Ctx* c, const Fp& fp, const u32* rp, const u32* col, const u32* val, long long r,
                       const u32* X, int b, u32* Y, u32 cmul, const u32* Z, const u32* U, unsigned long long* proj) {
  const int grid = (int)((r * 32 + 255) / 256);
  if (b == 4) {
    const uint4 *X4 = reinterpret_cast<const uint4*>(X), *Z4 = reinterpret_cast<const uint4*>(Z),
                *U4 = reinterpret_cast<const uint4*>(U);
    uint4* Y4 = reinterpret_cast<uint4*>(Y);
    if (c->p < 65536u)
      F4B_LAUNCH(c, k_op_apply4<true>, grid, 256, 0, fp, rp, col, val, r, X4, Y4, cmul, Z4, U4, proj);
    else
      F4B_LAUNCH(c, k_op_apply4<false>, grid, 256, 0, fp, rp, col, val, r, X4, Y4, cmul, Z4, U4, proj);
  } else {
    F4B_LAUNCH(c, k_op_apply, grid, 256, 0, fp, rp, col, val, r, X, b, Y, cmul, Z, U, proj);
  }
}

static void op_apply_dev(f4b_op* op, const u32* Win, u32* Wout, int b, u32 cmul, const u32* Z, const u32* U,
                         unsigned long long* proj) {
  Ctx* c = op->ctx;
  Fp fp = make_fp_pub(c);
  if (!op->normal) {
    const long long r = op->n_rows;
    apply_rows(c, fp, op->rp.as<u32>(), op->col.as<u32>(), op->val.as<u32>(), r, Win, b, Wout, cmul, Z, U, proj);
  } else {
    // T = A W (n_rows), W' = Aᵀ T (dim); the projection of W rides on the second pass
    const long long r = op->n_rows, d = op->dim;
    apply_rows(c, fp, op->rp.as<u32>(), op->col.as<u32>(), op->val.as<u32>(), r, Win, b, op->t.as<u32>(), 0u,
               nullptr, nullptr, nullptr);
    if (proj)
      F4B_LAUNCH(c, k_op_proj, (int)std::min<long long>((d + 255) / 256, c->num_sms * 4), 256, 0, fp, U, Win, d, b, proj);
    apply_rows(c, fp, op->trp.as<u32>(), op->tcol.as<u32>(), op->tval.as<u32>(), d, op->t.as<u32>(), b, Wout, cmul, Z,
               nullptr, nullptr);
  }
}

static void to_dev_u32(Ctx* c, DBuf& d, const uint64_t* h, long long n) {
  std::vector<u32> t((size_t)std::max<long long>(n, 1));
  for (long long i = 0; i < n; ++i) t[i] = (u32)(h[i] % c->p);
  ensure(c, d, t.size() * 4);
  check_cuda(cudaMemcpyAsync(d.p, t.data(), (size_t)n * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
}

static void from_dev_u32(Ctx* c, const DBuf& d, uint64_t* h, long long n) {
  std::vector<u32> t((size_t)std::max<long long>(n, 1));
  check_cuda(cudaMemcpyAsync(t.data(), d.p, (size_t)n * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  for (long long i = 0; i < n; ++i) h[i] = t[i];
}

}  // namespace f4b

using namespace f4b;

#define OP_BEGIN(op)      \
  Ctx* _c = (op)->ctx;    \
  try {
#define OP_END                                   \
  }                                              \
  catch (const Error& e) {                       \
    if (_c) _c->last_error = e.msg;              \
    return e.code;                               \
  }                                              \
  catch (const std::bad_alloc&) {                \
    if (_c) _c->last_error = "host allocation failed"; \
    return F4B_ERR_OOM;                          \
  }                                              \
  return F4B_OK;


f4b::Ctx* f4b_ctx_of(f4b_ctx* h);

int f4b_op_create(f4b_ctx* h, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col_ind,
                  const uint64_t* val, int normal, f4b_op** out) {
  if (!h || !out || n_rows < 0 || n_cols < 0) return F4B_ERR_PRECONDITION;
  *out = nullptr;
  f4b_op* op = new f4b_op();
  op->ctx = f4b_ctx_of(h);
  Ctx* c = op->ctx;
  try {
    op->n_rows = n_rows;
    op->n_cols = n_cols;
    op->normal = normal ? 1 : 0;
    op->dim = n_cols;
    if (!normal && n_rows != n_cols) fail(F4B_ERR_PRECONDITION, "a non-normal operator must be square");
    upload_csr(c, n_rows, row_ptr, col_ind, val, op->rp, op->col, op->val);
    if (normal) {
      // Aᵀ by a counting sort over the columns (rows ascending inside a
      // column, as csr_transpose produces it)
      const long long M = row_ptr[n_rows];
      std::vector<int64_t> trp(n_cols + 1, 0), tcol(std::max<long long>(M, 1));
      std::vector<uint64_t> tval(std::max<long long>(M, 1));
      for (long long k = 0; k < M; ++k) ++trp[col_ind[k] + 1];
      for (long long j = 0; j < n_cols; ++j) trp[j + 1] += trp[j];
      std::vector<int64_t> pos(trp.begin(), trp.end() - 1);
      for (long long i = 0; i < n_rows; ++i)
        for (long long k = row_ptr[i]; k < row_ptr[i + 1]; ++k) {
          const long long q = pos[col_ind[k]]++;
          tcol[q] = i;
          tval[q] = val[k];
        }
      upload_csr(c, n_cols, trp.data(), tcol.data(), tval.data(), op->trp, op->tcol, op->tval);
    }
  } catch (const Error& e) {
    c->last_error = e.msg;
    f4b_op_free(op);
    return e.code;
  } catch (const std::bad_alloc&) {
    f4b_op_free(op);
    return F4B_ERR_OOM;
  }
  *out = op;
  return F4B_OK;
}

int f4b_op_free(f4b_op* op) {
  if (!op) return F4B_OK;
  Ctx* c = op->ctx;
  cudaStreamSynchronize(c->stream);
  DBuf* bufs[] = {&op->rp, &op->col, &op->val, &op->trp, &op->tcol, &op->tval,
                  &op->w0, &op->w1, &op->t, &op->v, &op->u, &op->acc};
  for (DBuf* b : bufs) release(c, *b);
  delete op;
  return F4B_OK;
}

int f4b_op_apply(f4b_op* op, const uint64_t* X, int64_t b, uint64_t* Y) {
  if (!op || b < 1) return F4B_ERR_PRECONDITION;
  OP_BEGIN(op)
  Ctx* c = op->ctx;
  const long long d = op->dim;
  to_dev_u32(c, op->w0, X, d * b);
  ensure(c, op->w1, (size_t)std::max<long long>(d * b, 1) * 4);
  if (op->normal) ensure(c, op->t, (size_t)std::max<long long>(op->n_rows * b, 1) * 4);
  op_apply_dev(op, op->w0.as<u32>(), op->w1.as<u32>(), (int)b, 0u, nullptr, nullptr, nullptr);
  from_dev_u32(c, op->w1, Y, d * b);
  OP_END
}

// seqs[k][j] = Σ_i U[i][j] (B^k V)[i][j] mod p, k < steps (reference :408-412)
int f4b_op_krylov(f4b_op* op, const uint64_t* U, const uint64_t* V, int64_t b, int64_t steps, uint64_t* seqs) {
  if (!op || b < 1 || steps < 0) return F4B_ERR_PRECONDITION;
  OP_BEGIN(op)
  Ctx* c = op->ctx;
  const long long d = op->dim;
  to_dev_u32(c, op->u, U, d * b);
  to_dev_u32(c, op->w0, V, d * b);
  ensure(c, op->w1, (size_t)std::max<long long>(d * b, 1) * 4);
  if (op->normal) ensure(c, op->t, (size_t)std::max<long long>(op->n_rows * b, 1) * 4);
  ensure(c, op->acc, (size_t)std::max<long long>(steps * b, 1) * 8);
  check_cuda(cudaMemsetAsync(op->acc.p, 0, (size_t)std::max<long long>(steps * b, 1) * 8, c->stream), "memset");
  u32* a = op->w0.as<u32>();
  u32* bb = op->w1.as<u32>();
  unsigned long long* acc = op->acc.as<unsigned long long>();
  for (long long k = 0; k < steps; ++k) {
    // the last step only needs the projection of B^(steps-1) V
    if (k + 1 < steps) {
      op_apply_dev(op, a, bb, (int)b, 0u, nullptr, op->u.as<u32>(), acc + k * b);
      std::swap(a, bb);
    } else {
      Fp fp = make_fp_pub(c);
      F4B_LAUNCH(c, k_op_proj, (int)std::min<long long>((d + 255) / 256, c->num_sms * 4), 256, 0, fp, op->u.as<u32>(),
                 a, d, (int)b, acc + k * b);
    }
  }
  std::vector<unsigned long long> h((size_t)std::max<long long>(steps * b, 1));
  check_cuda(cudaMemcpyAsync(h.data(), op->acc.p, (size_t)steps * b * 8, cudaMemcpyDeviceToHost, c->stream), "d2h");
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  for (long long q = 0; q < steps * b; ++q) seqs[q] = h[q] % c->p;
  OP_END
}

// out = Σ_i g[i] B^i v (Horner from the top coefficient, reference :425-429)
int f4b_op_horner(f4b_op* op, const uint64_t* g, int64_t len, const uint64_t* v, uint64_t* out) {
  if (!op || len < 1) return F4B_ERR_PRECONDITION;
  OP_BEGIN(op)
  Ctx* c = op->ctx;
  const long long d = op->dim;
  to_dev_u32(c, op->v, v, d);
  std::vector<uint64_t> init((size_t)std::max<long long>(d, 1));
  const unsigned long long top = g[len - 1] % c->p;
  for (long long i = 0; i < d; ++i) init[i] = (unsigned long long)((unsigned __int128)top * (v[i] % c->p) % c->p);
  to_dev_u32(c, op->w0, init.data(), d);
  ensure(c, op->w1, (size_t)std::max<long long>(d, 1) * 4);
  if (op->normal) ensure(c, op->t, (size_t)std::max<long long>(op->n_rows, 1) * 4);
  u32* a = op->w0.as<u32>();
  u32* bb = op->w1.as<u32>();
  for (long long i = len - 2; i >= 0; --i) {
    op_apply_dev(op, a, bb, 1, (u32)(g[i] % c->p), op->v.as<u32>(), nullptr, nullptr);
    std::swap(a, bb);
  }
  std::vector<u32> t((size_t)std::max<long long>(d, 1));
  check_cuda(cudaMemcpyAsync(t.data(), a, (size_t)d * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  for (long long i = 0; i < d; ++i) out[i] = t[i];
  OP_END
}

// acc = v; up to max_steps times: nxt = B acc; stop before nxt == 0
// (reference :430-434).  *taken = applications kept.
int f4b_op_power_until_zero(f4b_op* op, const uint64_t* v, int64_t max_steps, uint64_t* out, int64_t* taken) {
  if (!op || max_steps < 0) return F4B_ERR_PRECONDITION;
  OP_BEGIN(op)
  Ctx* c = op->ctx;
  const long long d = op->dim;
  to_dev_u32(c, op->w0, v, d);
  ensure(c, op->w1, (size_t)std::max<long long>(d, 1) * 4 + 16);
  if (op->normal) ensure(c, op->t, (size_t)std::max<long long>(op->n_rows, 1) * 4);
  ensure(c, op->acc, 16);
  u32* a = op->w0.as<u32>();
  u32* bb = op->w1.as<u32>();
  u32* flag = reinterpret_cast<u32*>(op->acc.p);
  long long k = 0;
  for (; k < max_steps; ++k) {
    op_apply_dev(op, a, bb, 1, 0u, nullptr, nullptr, nullptr);
    check_cuda(cudaMemsetAsync(flag, 0, 4, c->stream), "memset");
    F4B_LAUNCH(c, k_any_nonzero, (int)std::min<long long>((d + 255) / 256, c->num_sms * 4), 256, 0, bb, d, flag);
    u32 hf = 0;
    check_cuda(cudaMemcpyAsync(&hf, flag, 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
    check_cuda(cudaStreamSynchronize(c->stream), "sync");
    if (!hf) break;
    std::swap(a, bb);
  }
  std::vector<u32> t((size_t)std::max<long long>(d, 1));
  check_cuda(cudaMemcpyAsync(t.data(), a, (size_t)d * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  for (long long i = 0; i < d; ++i) out[i] = t[i];
  *taken = k;
  OP_END
}
