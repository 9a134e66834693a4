// C ABI of libf4b200.so (include/f4b200.h): context, device memory through
// the registered allocator, the device-resident basis, and the thin wrappers
// that translate C++ exceptions into f4b_status codes.
#include <algorithm>
#include <chrono>
#include <cstdint>
#include <cstdio>
#include <cstring>
#include <new>
#include <vector>

#include "common.cuh"
#include "engine.h"

struct f4b_ctx {
  f4b::Ctx c;
};

f4b::Ctx* f4b_ctx_of(f4b_ctx* h) { return &h->c; }

namespace f4b {

[[noreturn]] void fail(int code, const std::string& msg) { throw Error{code, msg}; }

void check_cuda(cudaError_t e, const char* what) {
  if (e != cudaSuccess) {
    cudaGetLastError();
    fail(e == cudaErrorMemoryAllocation ? F4B_ERR_OOM : F4B_ERR_CUDA,
         std::string(what) + ": " + cudaGetErrorString(e));
  }
}

static void* raw_alloc(Ctx* c, size_t bytes) {
  if (bytes == 0) bytes = 16;
  void* p = nullptr;
  ++c->raw_allocs;
  const auto t0 = std::chrono::steady_clock::now();
  struct Tm {
    Ctx* c;
    std::chrono::steady_clock::time_point t0;
    ~Tm() { c->raw_alloc_us += std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count(); }
  } tm{c, t0};
  if (c->alloc) {
    p = c->alloc(bytes, c->user);
    if (!p) fail(F4B_ERR_OOM, "device allocation of " + std::to_string(bytes) + " bytes failed");
  } else if (c->mempool) {
    check_cuda(cudaMallocFromPoolAsync(&p, bytes, c->mempool, c->stream), "cudaMallocFromPoolAsync");
  } else {
    check_cuda(cudaMalloc(&p, bytes), "cudaMalloc");
  }
  return p;
}

static void raw_free(Ctx* c, void* p) {
  if (!p) return;
  ++c->raw_frees;
  if (c->dfree) c->dfree(p, c->user);
  else if (c->mempool) cudaFreeAsync(p, c->stream);
  else cudaFree(p);
}

static constexpr size_t POOL_MAX_BUFS = 96;
static constexpr size_t POOL_MAX_BYTES = (size_t)8 << 30;

void release(Ctx* c, DBuf& b) {
  if (b.p && c->pool.size() < POOL_MAX_BUFS && c->pool_bytes + b.cap <= POOL_MAX_BYTES) {
    c->pool.push_back({b.p, b.cap});
    c->pool_bytes += b.cap;
  } else {
    raw_free(c, b.p);
  }
  b.p = nullptr;
  b.cap = 0;
}

void pool_flush(Ctx* c) {
  for (auto& e : c->pool) raw_free(c, e.first);
  c->pool.clear();
  c->pool_bytes = 0;
}

// smallest pooled buffer in [bytes, 2 * bytes + 1 MiB]
static bool pool_take(Ctx* c, DBuf& b, size_t bytes) {
  size_t best = SIZE_MAX, bi = 0;
  for (size_t i = 0; i < c->pool.size(); ++i) {
    const size_t cp = c->pool[i].second;
    if (cp >= bytes && cp <= 2 * bytes + (1u << 20) && cp < best) {
      best = cp;
      bi = i;
    }
  }
  if (best == SIZE_MAX) return false;
  b.p = c->pool[bi].first;
  b.cap = best;
  c->pool_bytes -= best;
  c->pool[bi] = c->pool.back();
  c->pool.pop_back();
  return true;
}

void ensure(Ctx* c, DBuf& b, size_t bytes) {
  if (bytes <= b.cap && b.p) return;
  release(c, b);
  if (pool_take(c, b, bytes)) return;
  size_t cap = std::max<size_t>(bytes + bytes / 4, 256);
  cap = (cap + 255) & ~(size_t)255;
  b.p = raw_alloc(c, cap);
  b.cap = cap;
}

void ensure_keep(Ctx* c, DBuf& b, size_t bytes) {
  if (bytes <= b.cap && b.p) return;
  size_t cap = std::max<size_t>(bytes + bytes / 2, 256);
  cap = (cap + 255) & ~(size_t)255;
  void* np = raw_alloc(c, cap);
  if (b.p && b.cap) check_cuda(cudaMemcpyAsync(np, b.p, b.cap, cudaMemcpyDeviceToDevice, c->stream), "grow copy");
  raw_free(c, b.p);
  b.p = np;
  b.cap = cap;
}

uint32_t read_u32(Ctx* c, const uint32_t* dptr) {
  check_cuda(cudaMemcpyAsync(c->h_stat, dptr, sizeof(uint32_t), cudaMemcpyDeviceToHost, c->stream), "d2h u32");
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  return c->h_stat[0];
}

cudaEvent_t timing_event(Ctx* c, int i) {
  if (!c->tev[i]) check_cuda(cudaEventCreate(&c->tev[i]), "event");
  return c->tev[i];
}

void memset_async(Ctx* c, void* p, int v, size_t bytes) { check_cuda(cudaMemsetAsync(p, v, bytes, c->stream), "memset"); }

ProfScope::ProfScope(Ctx* c_, const char* n) : c(c_), name(n) {
  ++c->launches;
  ++c->total_launches;
  if (!c->prof) return;
  if (c->ev_used + 2 > c->ev_pool.size()) {
    size_t grow = std::max<size_t>(256, c->ev_pool.size());
    for (size_t i = 0; i < grow; ++i) {
      cudaEvent_t e;
      check_cuda(cudaEventCreate(&e), "event pool");
      c->ev_pool.push_back(e);
    }
  }
  e0 = c->ev_used++;
  check_cuda(cudaEventRecord(c->ev_pool[e0], c->stream), "event record");
}

ProfScope::~ProfScope() {
  if (!c->prof) return;
  size_t e1 = c->ev_used++;
  cudaEventRecord(c->ev_pool[e1], c->stream);
  c->pending.push_back({name, e0, e1});
}

static void prof_resolve(Ctx* c) {
  if (c->pending.empty()) return;
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  for (const auto& p : c->pending) {
    float ms = 0;
    cudaEventElapsedTime(&ms, c->ev_pool[p.e0], c->ev_pool[p.e1]);
    auto it = std::find_if(c->prof_acc.begin(), c->prof_acc.end(), [&](const auto& kv) { return kv.first == p.name; });
    if (it == c->prof_acc.end()) {
      c->prof_acc.push_back({p.name, {0.0, 0}});
      it = c->prof_acc.end() - 1;
    }
    it->second.first += ms;
    it->second.second += 1;
  }
  c->pending.clear();
  c->ev_used = 0;
}

void plan_release(f4b_plan* pl) {
  if (!pl) return;
  Ctx* c = pl->ctx;
  if (pl->pf_done) {  // a prefetch still reading the buffers (or writing the host block)
    cudaEventSynchronize(pl->pf_done);
    cudaEventDestroy(pl->pf_done);
  }
  DBuf* bufs[] = {&pl->row_ptr, &pl->col_ind, &pl->val, &pl->dict, &pl->dict_exps, &pl->cl_basis, &pl->cl_shift,
                  &pl->cl_round, &pl->pf_wide};
  for (DBuf* b : bufs) release(c, *b);
  delete pl;
}

// ---------------------------------------------------------------------------
// SpMM (reference sparselin.py:142-173): Y = A X mod p, one warp per row.
// ---------------------------------------------------------------------------
__global__ void k_spmm(Fp fp, const u32* __restrict__ rp, const u32* __restrict__ col, const u32* __restrict__ val,
                       long long r, const u32* __restrict__ X, int b, u32* __restrict__ Y) {
  long long row = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (row >= r) return;
  const u32 s = rp[row], e = rp[row + 1];
  for (int j = 0; j < b; ++j) {
    unsigned long long acc = 0;  // sum of < 32 reduced products per lane fits 64 bits
    for (u32 k = s + lane; k < e; k += 32) {
      acc += fp.mul(__ldg(val + k), __ldg(X + (size_t)col[k] * b + j));
      if (acc >= (1ull << 62)) acc %= fp.p;
    }
    acc %= fp.p;
#pragma unroll
    for (int o = 16; o; o >>= 1) {
      unsigned long long y = __shfl_xor_sync(0xffffffffu, acc, o);
      acc = (acc + y) % fp.p;
    }
    if (lane == 0) Y[(size_t)row * b + j] = (u32)acc;
  }
}

void spmm(Ctx* c, long long r, long long N, const int64_t* rp, const int64_t* col, const uint64_t* val,
          const uint64_t* X, long long b, uint64_t* Y) {
  const long long M = rp[r];
  // the device CSR holds u32 offsets / columns (row_ptr, col_ind)
  if (M < 0 || M >= (1ll << 32) - 1 || N >= (1ll << 32) - 1 || r >= (1ll << 32) - 1)
    fail(F4B_ERR_SIZE_CAP, "spmm: nnz, rows and columns must stay below 2^32 - 1");
  std::vector<u32> hrp(r + 1), hcol(std::max<long long>(M, 1)), hval(std::max<long long>(M, 1));
  std::vector<u32> hx(std::max<long long>(N * b, 1)), hy(std::max<long long>(r * b, 1));
  for (long long i = 0; i <= r; ++i) hrp[i] = (u32)rp[i];
  for (long long k = 0; k < M; ++k) {
    hcol[k] = (u32)col[k];
    hval[k] = (u32)(val[k] % c->p);
  }
  for (long long k = 0; k < N * b; ++k) hx[k] = (u32)(X[k] % c->p);
  DBuf drp, dcol, dval, dx, dy;
  ensure(c, drp, hrp.size() * 4);
  ensure(c, dcol, hcol.size() * 4);
  ensure(c, dval, hval.size() * 4);
  ensure(c, dx, hx.size() * 4);
  ensure(c, dy, hy.size() * 4);
  check_cuda(cudaMemcpyAsync(drp.p, hrp.data(), hrp.size() * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
  check_cuda(cudaMemcpyAsync(dcol.p, hcol.data(), hcol.size() * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
  check_cuda(cudaMemcpyAsync(dval.p, hval.data(), hval.size() * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
  check_cuda(cudaMemcpyAsync(dx.p, hx.data(), hx.size() * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
  Fp fp{c->p, c->pprime, c->r2};
  if (r > 0 && b > 0) {
    unsigned blocks = (unsigned)std::max<long long>(1, (r * 32 + 255) / 256);
    F4B_LAUNCH(c, k_spmm, blocks, 256, 0, fp, drp.as<u32>(), dcol.as<u32>(), dval.as<u32>(), r, dx.as<u32>(), (int)b,
                                          dy.as<u32>());
    check_cuda(cudaGetLastError(), "k_spmm");
  }
  check_cuda(cudaMemcpyAsync(hy.data(), dy.p, hy.size() * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  for (long long k = 0; k < r * b; ++k) Y[k] = hy[k];
  release(c, drp);
  release(c, dcol);
  release(c, dval);
  release(c, dx);
  release(c, dy);
}

}  // namespace f4b

using namespace f4b;

#define API_BEGIN(ctxp) \
  Ctx* _c = (ctxp);     \
  try {
#define API_END                                  \
  }                                              \
  catch (const Error& e) {                       \
    if (_c) _c->last_error = e.msg;              \
    return e.code;                               \
  }                                              \
  catch (const std::bad_alloc&) {                \
    if (_c) _c->last_error = "host allocation";  \
    return F4B_ERR_OOM;                          \
  }                                              \
  catch (...) {                                  \
    if (_c) _c->last_error = "unknown failure";  \
    return F4B_ERR_CUDA;                         \
  }                                              \
  return F4B_OK;

extern "C" {

int f4b_abi_version(void) { return 2; }

int f4b_ctx_create(int device, uint32_t p, int n_vars, int order, f4b_alloc_fn alloc, f4b_free_fn dfree, void* user,
                   f4b_ctx** out) {
  if (!out) return F4B_ERR_PRECONDITION;
  *out = nullptr;
  if (p < 3 || p >= (1u << 31) || (p & 1u) == 0 || n_vars < 1 || n_vars > 32 || order < 0 || order > 2)
    return F4B_ERR_PRECONDITION;
  f4b_ctx* h = new (std::nothrow) f4b_ctx();
  if (!h) return F4B_ERR_OOM;
  Ctx* c = &h->c;
  try {
    check_cuda(cudaSetDevice(device), "cudaSetDevice");
    c->device = device;
    c->p = p;
    c->n_vars = n_vars;
    c->order = order;
    c->alloc = alloc;
    c->dfree = dfree;
    c->user = user;
    int sms = 0;
    check_cuda(cudaDeviceGetAttribute(&sms, cudaDevAttrMultiProcessorCount, device), "sm count");
    c->num_sms = sms;
    if (const char* e = getenv("F4B_DICT")) c->opt_dict_sort = !strcmp(e, "sort");
    if (const char* e = getenv("F4B_FBSP")) c->opt_fbsp = !strcmp(e, "multi");
    if (getenv("F4B_DICT_LSD")) c->opt_dict_lsd = 1;
    // Montgomery constants: p * p' = -1 mod 2^32, R^2 mod p
    uint32_t x = 1;
    for (int i = 0; i < 6; ++i) x = x * (2u - p * x);
    c->pprime = (uint32_t)(0u - x);
    c->r2 = (uint32_t)(((unsigned __int128)1 << 64) % p);
    check_cuda(cudaMallocHost((void**)&c->h_stat, 4096), "pinned");
    if (!alloc) {
      cudaMemPoolProps props = {};
      props.allocType = cudaMemAllocationTypePinned;
      props.location.type = cudaMemLocationTypeDevice;
      props.location.id = device;
      check_cuda(cudaMemPoolCreate(&c->mempool, &props), "cudaMemPoolCreate");
      uint64_t keep = UINT64_MAX;
      check_cuda(cudaMemPoolSetAttribute(c->mempool, cudaMemPoolAttrReleaseThreshold, &keep), "mempool attr");
      // reserve physical memory up front: growing the pool inside a call was
      // measured to stall it for tens of ms (a 65 ms cudaMallocFromPoolAsync
      // in the middle of an elimination); freed blocks stay with the pool
      size_t free_b = 0, total_b = 0;
      cudaMemGetInfo(&free_b, &total_b);
      const size_t reserve = std::min<size_t>((size_t)2 << 30, free_b / 8);
      if (reserve) {
        void* warm = nullptr;
        if (cudaMallocFromPoolAsync(&warm, reserve, c->mempool, c->stream) == cudaSuccess) {
          cudaFreeAsync(warm, c->stream);
          cudaStreamSynchronize(c->stream);
        }
        cudaGetLastError();
      }
    }
    c->basis.h_off.push_back(0);
  } catch (const Error& e) {
    delete h;
    return e.code;
  }
  *out = h;
  return F4B_OK;
}

int f4b_ctx_destroy(f4b_ctx* h) {
  if (!h) return F4B_OK;
  Ctx* c = &h->c;
  cudaStreamSynchronize(c->stream);
  DBuf* bufs[] = {&c->basis.exps, &c->basis.coeff, &c->basis.off, &c->basis.len, &c->basis.lmexp, &c->basis.ckey,
                  &c->basis.maxe, &c->scan_tmp, &c->sort_a, &c->sort_b, &c->sort_hist, &c->flags, &c->errflag,
                  &c->tmp_u32a, &c->tmp_u32b, &c->tmp_u32c, &c->rows_basis, &c->rows_delta, &c->rows_len,
                  &c->rows_start, &c->keys_all, &c->vals_all, &c->dict_a, &c->dict_b, &c->front, &c->front_new,
                  &c->uniq, &c->red, &c->lmpref, &c->cand_idx, &c->shift_in, &c->cl_basis, &c->cl_shift,
                  &c->cl_round, &c->loop_scratch, &c->dstage, &c->maps, &c->dwp, &c->fcnt};
  for (DBuf* b : bufs) release(c, *b);
  pool_flush(c);
  if (c->h_stage) cudaFreeHost(c->h_stage);
  if (c->h_stat) cudaFreeHost(c->h_stat);
  if (c->copy_stream) cudaStreamDestroy(c->copy_stream);
  if (c->h_app) cudaFreeHost(c->h_app);
  for (cudaEvent_t e : c->ev_pool) cudaEventDestroy(e);
  for (cudaEvent_t& e : c->tev)
    if (e) cudaEventDestroy(e);
  if (c->mempool) {
    cudaStreamSynchronize(c->stream);
    cudaMemPoolDestroy(c->mempool);
  }
  delete h;
  return F4B_OK;
}

int f4b_ctx_set_stream(f4b_ctx* h, void* stream) {
  if (!h) return F4B_ERR_PRECONDITION;
  if (h->c.stream != (cudaStream_t)stream) {
    // pooled buffers were last used on the old stream
    cudaStreamSynchronize(h->c.stream);
    try {
      pool_flush(&h->c);
    } catch (const Error& e) {
      return e.code;
    }
  }
  h->c.stream = (cudaStream_t)stream;
  return F4B_OK;
}

int f4b_ctx_set_option(f4b_ctx* h, const char* name, int64_t value) {
  if (!h || !name) return F4B_ERR_PRECONDITION;
  Ctx* c = &h->c;
  struct {
    const char* n;
    int* p;
    int64_t hi;
  } opts[] = {{"sweep", &c->opt_sweep, 2},
              {"dense", &c->opt_dense, 1},
              {"dense_rows", &c->opt_dense_rows, 1},
              {"fbsp", &c->opt_fbsp, 1},
              {"dict_sort", &c->opt_dict_sort, 1},
              {"dict_lsd", &c->opt_dict_lsd, 1}};
  for (auto& o : opts)
    if (!strcmp(o.n, name)) {
      if (value < 0 || value > o.hi) {
        c->last_error = std::string("option value out of range: ") + name;
        return F4B_ERR_PRECONDITION;
      }
      *o.p = (int)value;
      return F4B_OK;
    }
  c->last_error = std::string("unknown option: ") + name;
  return F4B_ERR_PRECONDITION;
}

int f4b_ctx_profile(f4b_ctx* h, int enable) {
  if (!h) return F4B_ERR_PRECONDITION;
  Ctx* _c = &h->c;
  try {
    prof_resolve(_c);
  } catch (const Error& e) {
    return e.code;
  }
  _c->prof_acc.clear();
  _c->prof = enable != 0;
  return F4B_OK;
}

int f4b_ctx_profile_read(f4b_ctx* h, char* buf, int64_t buflen, int64_t* total_launches) {
  if (!h) return F4B_ERR_PRECONDITION;
  Ctx* _c = &h->c;
  try {
    prof_resolve(_c);
  } catch (const Error& e) {
    return e.code;
  }
  if (total_launches) *total_launches = _c->total_launches;
  std::string out;
  for (const auto& kv : _c->prof_acc) {
    char line[256];
    snprintf(line, sizeof line, "%s %lld %.0f\n", kv.first.c_str(), kv.second.second, kv.second.first * 1e6);
    out += line;
  }
  if (buf && buflen > 0) {
    size_t n = std::min<size_t>(out.size(), (size_t)buflen - 1);
    memcpy(buf, out.data(), n);
    buf[n] = 0;
  }
  return F4B_OK;
}

const char* f4b_ctx_last_error(const f4b_ctx* h) { return h ? h->c.last_error.c_str() : "null context"; }

int f4b_basis_clear(f4b_ctx* h) {
  if (!h) return F4B_ERR_PRECONDITION;
  if (h->c.pend.active) {  // a pending append is discarded with the basis
    h->c.pend.active = false;
    h->c.pend.applied = false;
    cudaStreamSynchronize(h->c.stream);
    release(&h->c, h->c.pend.raw);
  }
  Basis& B = h->c.basis;
  B.n_polys = 0;
  B.n_terms = 0;
  B.h_len.clear();
  B.h_off.assign(1, 0);
  B.h_lm.clear();
  B.h_maxe.clear();
  B.ckey_terms = 0;
  B.ckey_lane_bits = -1;
  B.lm_order.clear();
  B.lm_sorted = 0;
  B.h_lmw.clear();
  B.lmw_polys = 0;
  return F4B_OK;
}

int f4b_basis_append(f4b_ctx* h, int64_t n_polys, const int64_t* lengths, const uint16_t* exps, const uint32_t* coeffs) {
  if (!h) return F4B_ERR_PRECONDITION;
  API_BEGIN(&h->c)
  Ctx* c = _c;
  basis_finish(c);
  Basis& B = c->basis;
  const int n = c->n_vars;
  if (n_polys < 0) fail(F4B_ERR_PRECONDITION, "negative polynomial count");
  long long T = 0;
  for (long long i = 0; i < n_polys; ++i) {
    if (lengths[i] < 0) fail(F4B_ERR_PRECONDITION, "negative polynomial length");
    T += lengths[i];
  }
  for (long long t = 0; t < T; ++t)
    if (coeffs[t] == 0 || coeffs[t] >= c->p) fail(F4B_ERR_PROPERTY, "basis coefficient outside [1, p)");
  const long long T0 = B.n_terms, P0 = B.n_polys, T1 = T0 + T, P1 = P0 + n_polys;
  if (T1 >= (1ll << 31)) fail(F4B_ERR_SIZE_CAP, "basis has more than 2^31 terms");
  // host mirrors
  long long at = 0;
  for (long long i = 0; i < n_polys; ++i) {
    const long long L = lengths[i];
    B.h_len.push_back(L);
    B.h_off.push_back(B.h_off.back() + L);
    for (int v = 0; v < n; ++v) {
      uint16_t lm = L ? exps[(at)*n + v] : 0, mx = 0;
      for (long long j = 0; j < L; ++j) mx = std::max<uint16_t>(mx, exps[(at + j) * n + v]);
      B.h_lm.push_back(lm);
      B.h_maxe.push_back(mx);
    }
    at += L;
  }
  // device streams (grow, preserving the existing basis)
  ensure_keep(c, B.exps, (size_t)(T1 + 1) * n * sizeof(u16));
  ensure_keep(c, B.coeff, (size_t)(T1 + 1) * sizeof(u32));
  ensure_keep(c, B.off, (size_t)(P1 + 1) * sizeof(u32));
  ensure_keep(c, B.len, (size_t)(P1 + 1) * sizeof(u32));
  ensure_keep(c, B.lmexp, (size_t)(P1 + 1) * n * sizeof(u16));
  ensure_keep(c, B.maxe, (size_t)(P1 + 1) * n * sizeof(u16));
  std::vector<u32> hoff(n_polys + 1), hlen(std::max<long long>(n_polys, 1));
  for (long long i = 0; i <= n_polys; ++i) hoff[i] = (u32)B.h_off[P0 + i];
  for (long long i = 0; i < n_polys; ++i) hlen[i] = (u32)lengths[i];
  if (T) {
    check_cuda(cudaMemcpyAsync(B.exps.as<u16>() + T0 * n, exps, T * n * sizeof(u16), cudaMemcpyHostToDevice, c->stream),
               "h2d exps");
    check_cuda(cudaMemcpyAsync(B.coeff.as<u32>() + T0, coeffs, T * sizeof(u32), cudaMemcpyHostToDevice, c->stream),
               "h2d coeff");
  }
  check_cuda(cudaMemcpyAsync(B.off.as<u32>() + P0, hoff.data(), (n_polys + 1) * sizeof(u32), cudaMemcpyHostToDevice,
                             c->stream), "h2d off");
  if (n_polys) {
    check_cuda(cudaMemcpyAsync(B.len.as<u32>() + P0, hlen.data(), n_polys * sizeof(u32), cudaMemcpyHostToDevice, c->stream),
               "h2d len");
    check_cuda(cudaMemcpyAsync(B.lmexp.as<u16>() + P0 * n, B.h_lm.data() + P0 * n, n_polys * n * sizeof(u16),
                               cudaMemcpyHostToDevice, c->stream), "h2d lm");
    check_cuda(cudaMemcpyAsync(B.maxe.as<u16>() + P0 * n, B.h_maxe.data() + P0 * n, n_polys * n * sizeof(u16),
                               cudaMemcpyHostToDevice, c->stream), "h2d maxe");
  }
  // the staging vectors die here: make the copies complete first
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  B.n_terms = T1;
  B.n_polys = (int)P1;
  API_END
}

__global__ void k_narrow_terms(const int64_t* __restrict__ e64, const uint64_t* __restrict__ c64, long long T, int n,
                               uint32_t p, uint16_t* __restrict__ e16, uint32_t* __restrict__ c32,
                               uint32_t* __restrict__ bad) {
  uint32_t flags = 0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (long long)gridDim.x * blockDim.x) {
    for (int v = 0; v < n; ++v) {
      const int64_t x = e64[t * n + v];
      if (x < 0 || x > 0xFFFF) flags |= 1u;
      e16[t * n + v] = (uint16_t)x;
    }
    const uint64_t cc = c64[t];
    if (cc == 0 || cc >= p) flags |= 2u;
    c32[t] = (uint32_t)cc;
  }
  if (flags) atomicOr(bad, flags);
}

// The same from the reference keys (monomials.py mon_key_pack: MSB first,
// [32-bit degree if graded] then one 16-bit lane per variable, grevlex lanes
// 0xFFFF - e in reversed variable order; W words per key): exponents
// recovered from the lanes, the degree lane checked against their sum
// (flag 4: corrupt key) and the padding bits against zero.
__global__ void k_narrow_keys(const uint64_t* __restrict__ keys, int W, int order, const uint64_t* __restrict__ c64,
                              long long T, int n, uint32_t p, uint16_t* __restrict__ e16, uint32_t* __restrict__ c32,
                              uint32_t* __restrict__ bad) {
  uint32_t flags = 0;
  const bool graded = order != 2, grevlex = order == 0;
  const int head = graded ? 32 : 0;
  for (long long t = (long long)blockIdx.x * blockDim.x + threadIdx.x; t < T; t += (long long)gridDim.x * blockDim.x) {
    const uint64_t* k = keys + t * W;
    uint64_t deg = 0;
    for (int i = 0; i < n; ++i) {
      const int off = head + 16 * i;
      const uint32_t lane = (uint32_t)(k[off >> 6] >> (48 - (off & 63))) & 0xFFFFu;
      const uint32_t e = grevlex ? 0xFFFFu - lane : lane;
      e16[t * n + (grevlex ? n - 1 - i : i)] = (uint16_t)e;
      deg += e;
    }
    if (graded && (k[0] >> 32) != deg) flags |= 4u;
    const int used = head + 16 * n;  // padding bits below the last lane
    if (used < 64 * W) {
      const int w = used >> 6, b = used & 63;
      if (b && (k[w] << b) != 0) flags |= 4u;
      for (int x = w + (b ? 1 : 0); x < W; ++x)
        if (k[x]) flags |= 4u;
    }
    const uint64_t cc = c64[t];
    if (cc == 0 || cc >= p) flags |= 2u;
    c32[t] = (uint32_t)cc;
  }
  if (flags) atomicOr(bad, flags);
}

// per polynomial (warp each): offset, length, LM exponents, max exponent per variable
__global__ void k_poly_meta(const uint16_t* __restrict__ e16, const int64_t* __restrict__ lens, long long P,
                            long long T0, int n, uint32_t* __restrict__ off, uint32_t* __restrict__ len,
                            uint16_t* __restrict__ lmexp, uint16_t* __restrict__ maxe,
                            const long long* __restrict__ pre) {
  const long long i = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (i >= P) return;
  const long long s = pre[i], L = lens[i];
  if (lane == 0) {
    off[i] = (uint32_t)(T0 + s);
    len[i] = (uint32_t)L;
  }
  for (int v = 0; v < n; ++v) {
    uint32_t mx = 0;
    for (long long j = lane; j < L; j += 32) mx = max(mx, (uint32_t)e16[(s + j) * n + v]);
#pragma unroll
    for (int o = 16; o; o >>= 1) mx = max(mx, __shfl_xor_sync(0xffffffffu, mx, o));
    if (lane == 0) {
      maxe[i * n + v] = (uint16_t)mx;
      lmexp[i * n + v] = L ? e16[s * n + v] : (uint16_t)0;
    }
  }
}

// Issue an append of the reference's int64 / uint64 streams (narrowing,
// range checks, LM / max exponents on the device) without waiting: the host
// mirrors and the error flag are completed by basis_finish.
// keys != nullptr: the terms come as reference keys (W words each) instead of
// int64 exponent rows (exps unused).
static void basis_append_wide_issue(Ctx* c, int64_t n_polys, const int64_t* lengths, const int64_t* exps,
                                    const uint64_t* coeffs, const uint64_t* keys = nullptr, int W = 0) {
  basis_finish(c);  // the staging block is reused
  Basis& B = c->basis;
  const int n = c->n_vars;
  if (n_polys < 0) fail(F4B_ERR_PRECONDITION, "negative polynomial count");
  std::vector<long long> pre((size_t)n_polys + 1, 0);
  for (long long i = 0; i < n_polys; ++i) {
    if (lengths[i] < 0) fail(F4B_ERR_PRECONDITION, "negative polynomial length");
    pre[i + 1] = pre[i] + lengths[i];
  }
  const long long T = pre[n_polys];
  const long long T0 = B.n_terms, P0 = B.n_polys, T1 = T0 + T, P1 = P0 + n_polys;
  if (T1 >= (1ll << 31)) fail(F4B_ERR_SIZE_CAP, "basis has more than 2^31 terms");
  ensure_keep(c, B.exps, (size_t)(T1 + 1) * n * sizeof(u16));
  ensure_keep(c, B.coeff, (size_t)(T1 + 1) * sizeof(u32));
  ensure_keep(c, B.off, (size_t)(P1 + 1) * sizeof(u32));
  ensure_keep(c, B.len, (size_t)(P1 + 1) * sizeof(u32));
  ensure_keep(c, B.lmexp, (size_t)(P1 + 1) * n * sizeof(u16));
  ensure_keep(c, B.maxe, (size_t)(P1 + 1) * n * sizeof(u16));
  // raw streams -> device staging -> narrowed basis streams
  Ctx::PendingAppend& pa = c->pend;
  DBuf& raw = pa.raw;
  if (keys && (W < 1 || W > 8 || (c->order != 2 ? 32 : 0) + 16 * n > 64 * W))
    fail(F4B_ERR_PRECONDITION, "key words do not match the ring");
  const size_t b_e = keys ? (size_t)T * W * 8 : (size_t)T * n * 8, b_c = (size_t)T * 8, b_l = (size_t)std::max<long long>(n_polys, 1) * 8,
               b_p = (size_t)(n_polys + 1) * 8;
  ensure(c, raw, b_e + b_c + b_l + b_p + 64);
  unsigned char* rp = raw.as<unsigned char>();
  int64_t* d_e = reinterpret_cast<int64_t*>(rp);
  uint64_t* d_c = reinterpret_cast<uint64_t*>(rp + b_e);
  int64_t* d_l = reinterpret_cast<int64_t*>(rp + b_e + b_c);
  long long* d_p = reinterpret_cast<long long*>(rp + b_e + b_c + b_l);
  uint32_t* d_bad = reinterpret_cast<uint32_t*>(rp + b_e + b_c + b_l + b_p);
  // page-locked staging: [lengths | prefix | tail offset] up, [LM | max exps | flag] down
  const size_t np1 = (size_t)std::max<long long>(n_polys, 1);
  const size_t o_len = 0, o_pre = o_len + np1 * 8, o_tail = o_pre + (size_t)(n_polys + 1) * 8,
               o_lm = o_tail + 16, o_mx = o_lm + ((np1 * n * 2 + 15) & ~(size_t)15),
               o_bad = o_mx + ((np1 * n * 2 + 15) & ~(size_t)15), app_bytes = o_bad + 16;
  if (c->h_app_cap < app_bytes) {
    if (c->h_app) cudaFreeHost(c->h_app);
    c->h_app = nullptr;
    c->h_app_cap = 0;
    const size_t cap = std::max<size_t>(app_bytes + app_bytes / 2, 1 << 16);
    check_cuda(cudaHostAlloc(&c->h_app, cap, cudaHostAllocDefault), "cudaHostAlloc app");
    c->h_app_cap = cap;
  }
  unsigned char* ha = static_cast<unsigned char*>(c->h_app);
  if (n_polys) {
    memcpy(ha + o_len, lengths, (size_t)n_polys * 8);
    memcpy(ha + o_pre, pre.data(), (size_t)(n_polys + 1) * 8);
  }
  *reinterpret_cast<u32*>(ha + o_tail) = (u32)T1;  // the basis end offset off[P1]
  check_cuda(cudaMemsetAsync(d_bad, 0, 4, c->stream), "memset");
  if (T) {
    check_cuda(cudaMemcpyAsync(d_e, keys ? (const void*)keys : (const void*)exps, b_e, cudaMemcpyHostToDevice,
                               c->stream), "h2d exps");
    check_cuda(cudaMemcpyAsync(d_c, coeffs, b_c, cudaMemcpyHostToDevice, c->stream), "h2d coeffs");
  }
  if (n_polys)
    check_cuda(cudaMemcpyAsync(d_l, ha + o_len, o_tail - o_len, cudaMemcpyHostToDevice, c->stream), "h2d lens+pre");
  if (T) {
    const int g = (int)std::min<long long>((T + 255) / 256, (long long)c->num_sms * 8);
    if (keys)
      F4B_LAUNCH(c, k_narrow_keys, g, 256, 0, reinterpret_cast<const uint64_t*>(d_e), W, c->order, d_c, T, n, c->p,
                 B.exps.as<u16>() + T0 * n, B.coeff.as<u32>() + T0, d_bad);
    else
      F4B_LAUNCH(c, k_narrow_terms, g, 256, 0, d_e, d_c, T, n, c->p, B.exps.as<u16>() + T0 * n,
                 B.coeff.as<u32>() + T0, d_bad);
  }
  if (n_polys) {
    F4B_LAUNCH(c, k_poly_meta, (int)((n_polys * 32 + 255) / 256), 256, 0, B.exps.as<u16>() + T0 * n, d_l, n_polys, T0,
               n, B.off.as<u32>() + P0, B.len.as<u32>() + P0, B.lmexp.as<u16>() + P0 * n,
               B.maxe.as<u16>() + P0 * n, d_p);
    check_cuda(cudaMemcpyAsync(ha + o_lm, B.lmexp.as<u16>() + P0 * n, (size_t)n_polys * n * 2, cudaMemcpyDeviceToHost,
                               c->stream), "d2h lm");
    check_cuda(cudaMemcpyAsync(ha + o_mx, B.maxe.as<u16>() + P0 * n, (size_t)n_polys * n * 2, cudaMemcpyDeviceToHost,
                               c->stream), "d2h maxe");
  }
  check_cuda(cudaMemcpyAsync(B.off.as<u32>() + P1, ha + o_tail, 4, cudaMemcpyHostToDevice, c->stream), "h2d off");
  check_cuda(cudaMemcpyAsync(ha + o_bad, d_bad, 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
  pa.active = true;
  pa.n_polys = n_polys;
  pa.T0 = T0;
  pa.P0 = P0;
  pa.T1 = T1;
  pa.P1 = P1;
  pa.applied = false;
  pa.lazy_ok = keys != nullptr && c->order != 2;
  if (pa.lazy_ok) {
    // LMs from the host keys (same lanes as k_narrow_keys), bound deg(LM)
    pa.lm_host.assign((size_t)n_polys * n, 0);
    pa.bound_host.assign((size_t)n_polys * n, 0);
    const bool grevlex = c->order == 0;
    for (long long i = 0; i < n_polys; ++i) {
      if (!lengths[i]) continue;
      const uint64_t* k = keys + (size_t)pre[i] * W;
      const uint64_t deg = k[0] >> 32;
      for (int q = 0; q < n; ++q) {
        const int off = 32 + 16 * q;
        const uint32_t lane = (uint32_t)(k[off >> 6] >> (48 - (off & 63))) & 0xFFFFu;
        pa.lm_host[(size_t)i * n + (grevlex ? n - 1 - q : q)] = (uint16_t)(grevlex ? 0xFFFFu - lane : lane);
      }
      for (int v = 0; v < n; ++v) pa.bound_host[(size_t)i * n + v] = (uint16_t)std::min<uint64_t>(deg, 0xFFFFu);
    }
  }
  pa.o_lm = o_lm;
  pa.o_mx = o_mx;
  pa.o_bad = o_bad;
  pa.lengths.assign(lengths, lengths + n_polys);
}

static bool basis_apply_lazy_impl(Ctx* c) {
  Ctx::PendingAppend& pa = c->pend;
  if (!pa.active) return false;
  if (!pa.lazy_ok) {
    basis_finish(c);
    return false;
  }
  if (pa.applied) return true;
  Basis& B = c->basis;
  for (long long i = 0; i < pa.n_polys; ++i) {
    B.h_len.push_back(pa.lengths[i]);
    B.h_off.push_back(B.h_off.back() + pa.lengths[i]);
  }
  B.h_lm.insert(B.h_lm.end(), pa.lm_host.begin(), pa.lm_host.end());
  B.h_maxe.insert(B.h_maxe.end(), pa.bound_host.begin(), pa.bound_host.end());
  B.n_terms = pa.T1;
  B.n_polys = (int)pa.P1;
  pa.applied = true;
  return true;
}

static void basis_finish_impl(Ctx* c) {
  Ctx::PendingAppend& pa = c->pend;
  if (!pa.active) return;
  pa.active = false;
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  Basis& B = c->basis;
  const int n = c->n_vars;
  const unsigned char* ha = static_cast<const unsigned char*>(c->h_app);
  const uint32_t bad = *reinterpret_cast<const u32*>(ha + pa.o_bad);
  release(c, pa.raw);
  if (pa.applied) {
    pa.applied = false;
    if (bad) {
      // roll the mirrors back to the basis before this append
      B.h_len.resize((size_t)pa.P0);
      B.h_off.resize((size_t)pa.P0 + 1);
      B.h_lm.resize((size_t)pa.P0 * n);
      B.h_maxe.resize((size_t)pa.P0 * n);
      B.n_terms = pa.T0;
      B.n_polys = (int)pa.P0;
      if (B.lm_sorted > pa.P0) {
        B.lm_order.clear();
        B.lm_sorted = 0;
      }
      B.lmw_polys = std::min<int>(B.lmw_polys, (int)pa.P0);
      B.ckey_terms = std::min<long long>(B.ckey_terms, pa.T0);
    } else {
      const uint16_t* hmx = reinterpret_cast<const uint16_t*>(ha + pa.o_mx);
      std::copy(hmx, hmx + (size_t)pa.n_polys * n, B.h_maxe.begin() + (size_t)pa.P0 * n);
      return;
    }
  }
  // a rejected append leaves the basis as it was (n_terms / n_polys not advanced)
  if (bad & 1u) fail(F4B_ERR_LANE_OVERFLOW, "exponent does not fit a 16-bit lane");
  if (bad & 2u) fail(F4B_ERR_PROPERTY, "basis coefficient outside [1, p)");
  if (bad & 4u) fail(F4B_ERR_PROPERTY, "basis key lanes are internally inconsistent");
  for (long long i = 0; i < pa.n_polys; ++i) {
    B.h_len.push_back(pa.lengths[i]);
    B.h_off.push_back(B.h_off.back() + pa.lengths[i]);
  }
  const uint16_t* hlm = reinterpret_cast<const uint16_t*>(ha + pa.o_lm);
  const uint16_t* hmx = reinterpret_cast<const uint16_t*>(ha + pa.o_mx);
  B.h_lm.insert(B.h_lm.end(), hlm, hlm + (size_t)pa.n_polys * n);
  B.h_maxe.insert(B.h_maxe.end(), hmx, hmx + (size_t)pa.n_polys * n);
  B.n_terms = pa.T1;
  B.n_polys = (int)pa.P1;
}

int f4b_basis_append_wide(f4b_ctx* h, int64_t n_polys, const int64_t* lengths, const int64_t* exps,
                          const uint64_t* coeffs) {
  if (!h) return F4B_ERR_PRECONDITION;
  API_BEGIN(&h->c)
  basis_append_wide_issue(_c, n_polys, lengths, exps, coeffs);
  basis_finish(_c);
  API_END
}

int f4b_basis_append_wide_async(f4b_ctx* h, int64_t n_polys, const int64_t* lengths, const int64_t* exps,
                                const uint64_t* coeffs) {
  if (!h) return F4B_ERR_PRECONDITION;
  API_BEGIN(&h->c)
  basis_append_wide_issue(_c, n_polys, lengths, exps, coeffs);
  API_END
}

int f4b_basis_append_keys_async(f4b_ctx* h, int64_t n_polys, const int64_t* lengths, const uint64_t* keys,
                                int key_words, const uint64_t* coeffs) {
  if (!h) return F4B_ERR_PRECONDITION;
  API_BEGIN(&h->c)
  basis_append_wide_issue(_c, n_polys, lengths, nullptr, coeffs, keys, key_words);
  API_END
}

int f4b_basis_sync(f4b_ctx* h) {
  if (!h) return F4B_ERR_PRECONDITION;
  API_BEGIN(&h->c)
  basis_finish(_c);
  API_END
}

int f4b_basis_size(const f4b_ctx* h, int64_t* n_polys, int64_t* n_terms) {
  if (!h) return F4B_ERR_PRECONDITION;
  if (h->c.pend.active) {
    const int code = f4b_basis_sync(const_cast<f4b_ctx*>(h));
    if (code) return code;
  }
  if (n_polys) *n_polys = h->c.basis.n_polys;
  if (n_terms) *n_terms = h->c.basis.n_terms;
  return F4B_OK;
}

int f4b_compile_batch(f4b_ctx* h, int64_t n_rows, const int32_t* row_basis, const uint16_t* row_shift, int closure,
                      const int32_t* candidates, int64_t n_candidates, int64_t dict_cap, f4b_plan** out) {
  if (!h || !out) return F4B_ERR_PRECONDITION;
  *out = nullptr;
  f4b_plan* pl = new (std::nothrow) f4b_plan();
  if (!pl) return F4B_ERR_OOM;
  pl->ctx = &h->c;
  API_BEGIN(&h->c)
  try {
    static const bool htrace = getenv("F4B_HOST_TRACE") != nullptr;
    const auto t0 = std::chrono::steady_clock::now();
    // a pending key append is not waited for: the compile is queued behind
    // it on the stream, its check completes after the compile (below)
    const bool lazy = basis_apply_lazy_impl(_c);
    if (htrace)
      fprintf(stderr, "[host] basis_finish %.1f us\n",
              std::chrono::duration<double, std::micro>(std::chrono::steady_clock::now() - t0).count());
    compile_batch(_c, n_rows, row_basis, row_shift, closure, candidates, n_candidates, dict_cap, pl);
    if (lazy) {
      basis_finish_impl(_c);  // the append's flag (fails with its error) and the exact maximum exponents
      recheck_lanes(_c, n_rows, row_basis, row_shift);
    }
  } catch (...) {
    plan_release(pl);
    throw;
  }
  *out = pl;
  API_END
}

int f4b_plan_get_info(const f4b_plan* pl, f4b_plan_info* info) {
  if (!pl || !info) return F4B_ERR_PRECONDITION;
  info->r = pl->r;
  info->N = pl->N;
  info->M = pl->M;
  info->closure_rounds = pl->closure_rounds;
  info->n_closure_rows = pl->n_closure();
  info->row_lo = pl->row_lo;
  info->r_total = pl->r_total >= 0 ? pl->r_total : pl->r;
  info->key_words = pl->KW;
  info->lane_bits = pl->lane_bits;
  info->dict_build_ns = pl->dict_ns;
  info->row_assemble_ns = pl->asm_ns;
  info->sort_passes = pl->sort_passes;
  info->kernel_launches = pl->launches;
  info->validated = pl->validated ? 1 : 0;
  return F4B_OK;
}

__global__ void k_widen_u32(const u32* __restrict__ in, long long n, unsigned long long* __restrict__ out) {
  for (long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x; i < n; i += (long long)gridDim.x * blockDim.x)
    out[i] = in[i];
}

int f4b_plan_download(const f4b_plan* pl, int64_t* row_ptr, int64_t* col_ind, uint64_t* val, uint16_t* dict_exps,
                      int32_t* closure_basis, uint16_t* closure_shift, int32_t* closure_round) {
  if (!pl) return F4B_ERR_PRECONDITION;
  API_BEGIN(pl->ctx)
  Ctx* c = _c;
  const int n = c->n_vars;
  const long long r = pl->r, M = pl->M, N = pl->N, ncl = pl->n_closure();
  // widen u32 -> 64-bit on the device, then one D2H per array straight into
  // the caller's buffers (page-locked ones copy at full link rate)
  const long long w_row = row_ptr ? r + 1 : 0, w_col = col_ind ? M : 0, w_val = val ? M : 0;
  DBuf wide;
  if (w_row + w_col + w_val) {
    ensure(c, wide, (size_t)(w_row + w_col + w_val) * 8);
    unsigned long long* wp = wide.as<unsigned long long>();
    const int g = c->num_sms * 4;
    if (w_row) F4B_LAUNCH(c, k_widen_u32, g, 256, 0, pl->row_ptr.as<u32>(), w_row, wp);
    if (w_col) F4B_LAUNCH(c, k_widen_u32, g, 256, 0, pl->col_ind.as<u32>(), w_col, wp + w_row);
    if (w_val) F4B_LAUNCH(c, k_widen_u32, g, 256, 0, pl->val.as<u32>(), w_val, wp + w_row + w_col);
    const bool contiguous = w_row && w_col && w_val && col_ind == row_ptr + w_row &&
                            reinterpret_cast<int64_t*>(val) == col_ind + w_col;
    if (contiguous) {  // one host block (the Python host allocates it so): one copy
      check_cuda(cudaMemcpyAsync(row_ptr, wp, (w_row + w_col + w_val) * 8, cudaMemcpyDeviceToHost, c->stream), "d2h");
    } else {
      if (w_row) check_cuda(cudaMemcpyAsync(row_ptr, wp, w_row * 8, cudaMemcpyDeviceToHost, c->stream), "d2h");
      if (w_col) check_cuda(cudaMemcpyAsync(col_ind, wp + w_row, w_col * 8, cudaMemcpyDeviceToHost, c->stream), "d2h");
      if (w_val)
        check_cuda(cudaMemcpyAsync(val, wp + w_row + w_col, w_val * 8, cudaMemcpyDeviceToHost, c->stream), "d2h");
    }
  }
  if (dict_exps && N)
    check_cuda(cudaMemcpyAsync(dict_exps, pl->dict_exps.p, N * n * sizeof(u16), cudaMemcpyDeviceToHost, c->stream), "d2h");
  if (ncl) {
    if (closure_basis)
      check_cuda(cudaMemcpyAsync(closure_basis, pl->cl_basis.p, ncl * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
    if (closure_shift)
      check_cuda(cudaMemcpyAsync(closure_shift, pl->cl_shift.p, ncl * n * 2, cudaMemcpyDeviceToHost, c->stream), "d2h");
    if (closure_round)
      check_cuda(cudaMemcpyAsync(closure_round, pl->cl_round.p, ncl * 4, cudaMemcpyDeviceToHost, c->stream), "d2h");
  }
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  release(c, wide);
  API_END
}

// reference keys (monomials.py:131-148) from the plan's column-order exponents
__global__ void k_ref_keys(const uint16_t* __restrict__ ex, long long N, int n, int order, int W,
                           unsigned long long* __restrict__ out) {
  const long long i = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  if (i >= N) return;
  const uint16_t* e = ex + i * n;
  const int head = order == 2 ? 0 : 32;
  unsigned long long w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
  if (order != 2) {
    unsigned long long d = 0;
    for (int v = 0; v < n; ++v) d += e[v];
    w[0] |= d << 32;
  }
  for (int l = 0; l < n; ++l) {
    const unsigned long long lane = order == 0 ? (unsigned long long)(0xFFFFu - e[n - 1 - l]) : (unsigned long long)e[l];
    const int off = head + 16 * l;
    w[off / 64] |= lane << (64 - (off % 64) - 16);
  }
  for (int q = 0; q < W; ++q) out[i * W + q] = w[q];
}

extern "C++" {
namespace f4b {
// reference keys of the plan dictionary (column order) into a device buffer
void ref_keys_device(Ctx* c, const f4b_plan* pl, unsigned long long* out, int W) {
  if (pl->N)
    F4B_LAUNCH(c, k_ref_keys, (int)((pl->N + 255) / 256), 256, 0, pl->dict_exps.as<uint16_t>(), pl->N, c->n_vars,
               c->order, W, out);
}
}  // namespace f4b
}

int f4b_plan_download_ref_keys(const f4b_plan* pl, uint64_t* keys) {
  if (!pl) return F4B_ERR_PRECONDITION;
  API_BEGIN(pl->ctx)
  Ctx* c = _c;
  const int n = c->n_vars;
  const int W = ((c->order == 2 ? 0 : 32) + 16 * n + 63) / 64;
  if (W > 8) fail(F4B_ERR_PRECONDITION, "reference key wider than 8 words");
  const long long N = pl->N;
  if (N) {
    DBuf kb;
    ensure(c, kb, (size_t)N * W * 8);
    F4B_LAUNCH(c, k_ref_keys, (int)((N + 255) / 256), 256, 0, pl->dict_exps.as<uint16_t>(), N, n, c->order, W,
               kb.as<unsigned long long>());
    check_cuda(cudaMemcpyAsync(keys, kb.p, (size_t)N * W * 8, cudaMemcpyDeviceToHost, c->stream), "d2h keys");
    check_cuda(cudaStreamSynchronize(c->stream), "sync");
    release(c, kb);
  }
  API_END
}

// Y[col][j] += v[row][j] * a[row][col]: warp per row, u64 atomics of
// reduced products (< 2^31 each, so 2^32 of them fit before the final mod)
__global__ void k_left_apply(Fp fp, const u32* __restrict__ rp, const u32* __restrict__ col,
                             const u32* __restrict__ val, long long r, const u32* __restrict__ V, int b,
                             unsigned long long* __restrict__ Y) {
  const long long row = ((long long)blockIdx.x * blockDim.x + threadIdx.x) / 32;
  const int lane = threadIdx.x & 31;
  if (row >= r) return;
  const u32 s = rp[row], e = rp[row + 1];
  for (int j = 0; j < b; ++j) {
    const u32 vj = V[(size_t)row * b + j];
    if (!vj) continue;
    for (u32 k = s + lane; k < e; k += 32) atomicAdd(Y + (size_t)col[k] * b + j, (unsigned long long)fp.mul(vj, val[k]));
  }
}

// Asynchronous host download: ONE staging block [r+1 | M | M | N*W] of
// 64-bit words (row_ptr, col_ind, val widened; the reference dictionary keys)
// built by one kernel on the context's copy stream behind the plan's
// completion and copied in one D2H — the next compile_batch runs on the
// main stream while the copy engine drains this one.  f4b_plan_wait blocks
// until the host block is complete.
__global__ void k_prefetch_pack(const u32* __restrict__ rp, long long r1, const u32* __restrict__ col,
                                const u32* __restrict__ val, long long M, const uint16_t* __restrict__ ex,
                                long long N, int n, int order, int W, unsigned long long* __restrict__ out) {
  const long long stride = (long long)gridDim.x * blockDim.x;
  const long long i0 = (long long)blockIdx.x * blockDim.x + threadIdx.x;
  for (long long i = i0; i < r1; i += stride) out[i] = rp[i];
  for (long long i = i0; i < M; i += stride) {
    out[r1 + i] = col[i];
    out[r1 + M + i] = val[i];
  }
  unsigned long long* kout = out + r1 + 2 * M;
  const int head = order == 2 ? 0 : 32;
  for (long long i = i0; i < N; i += stride) {  // k_ref_keys, reference monomials.py:131-148
    const uint16_t* e = ex + i * n;
    unsigned long long w[8] = {0, 0, 0, 0, 0, 0, 0, 0};
    if (order != 2) {
      unsigned long long d = 0;
      for (int v = 0; v < n; ++v) d += e[v];
      w[0] |= d << 32;
    }
    for (int l = 0; l < n; ++l) {
      const unsigned long long lane = order == 0 ? (unsigned long long)(0xFFFFu - e[n - 1 - l]) : (unsigned long long)e[l];
      const int off = head + 16 * l;
      w[off / 64] |= lane << (64 - (off % 64) - 16);
    }
    for (int q = 0; q < W; ++q) kout[i * W + q] = w[q];
  }
}

int f4b_plan_prefetch(f4b_plan* pl, uint64_t* block, int W) {
  if (!pl || !block || W < 1 || W > 8) return F4B_ERR_PRECONDITION;
  API_BEGIN(pl->ctx)
  Ctx* c = _c;
  if (pl->pf_pending) fail(F4B_ERR_PRECONDITION, "plan prefetch already pending");
  if (!c->copy_stream) check_cuda(cudaStreamCreateWithFlags(&c->copy_stream, cudaStreamNonBlocking), "stream");
  if (!pl->pf_done) check_cuda(cudaEventCreateWithFlags(&pl->pf_done, cudaEventDisableTiming), "event");
  const long long r1 = pl->r + 1, M = pl->M, N = pl->N;
  const long long words = r1 + 2 * M + N * W;
  ensure(c, pl->pf_wide, (size_t)words * 8);
  cudaEvent_t ready = timing_event(c, 1);  // the plan and the staging allocation complete on the main stream
  check_cuda(cudaEventRecord(ready, c->stream), "event");
  check_cuda(cudaStreamWaitEvent(c->copy_stream, ready, 0), "wait");
  const long long most = std::max({r1, M, N, 1ll});
  const int g = (int)std::min<long long>((most + 255) / 256, (long long)c->num_sms * 4);
  k_prefetch_pack<<<g, 256, 0, c->copy_stream>>>(pl->row_ptr.as<u32>(), r1, pl->col_ind.as<u32>(), pl->val.as<u32>(),
                                                 M, pl->dict_exps.as<uint16_t>(), N, c->n_vars, c->order, W,
                                                 pl->pf_wide.as<unsigned long long>());
  check_cuda(cudaGetLastError(), "k_prefetch_pack");
  check_cuda(cudaMemcpyAsync(block, pl->pf_wide.p, (size_t)words * 8, cudaMemcpyDeviceToHost, c->copy_stream), "d2h");
  check_cuda(cudaEventRecord(pl->pf_done, c->copy_stream), "event");
  pl->pf_pending = true;
  API_END
}

int f4b_plan_wait(f4b_plan* pl) {
  if (!pl) return F4B_ERR_PRECONDITION;
  API_BEGIN(pl->ctx)
  if (pl->pf_pending) {
    check_cuda(cudaEventSynchronize(pl->pf_done), "prefetch wait");
    pl->pf_pending = false;
  }
  API_END
}

int f4b_plan_left_apply(const f4b_plan* pl, const uint64_t* V, int64_t b, uint64_t* Y) {
  if (!pl || b < 1) return F4B_ERR_PRECONDITION;
  API_BEGIN(pl->ctx)
  Ctx* c = _c;
  const long long r = pl->r, N = pl->N;
  Fp fp;
  fp.p = c->p;
  fp.pprime = c->pprime;
  fp.r2 = c->r2;
  std::vector<u32> hv((size_t)std::max<long long>(r * b, 1));
  for (long long i = 0; i < r * b; ++i) hv[i] = (u32)(V[i] % c->p);
  DBuf dv, dy;
  ensure(c, dv, hv.size() * 4);
  ensure(c, dy, (size_t)std::max<long long>(N * b, 1) * 8);
  check_cuda(cudaMemcpyAsync(dv.p, hv.data(), (size_t)r * b * 4, cudaMemcpyHostToDevice, c->stream), "h2d");
  check_cuda(cudaMemsetAsync(dy.p, 0, (size_t)std::max<long long>(N * b, 1) * 8, c->stream), "memset");
  if (r) F4B_LAUNCH(c, k_left_apply, (int)((r * 32 + 255) / 256), 256, 0, fp, pl->row_ptr.as<u32>(), pl->col_ind.as<u32>(),
                    pl->val.as<u32>(), r, dv.as<u32>(), (int)b, dy.as<unsigned long long>());
  std::vector<unsigned long long> hy((size_t)std::max<long long>(N * b, 1));
  check_cuda(cudaMemcpyAsync(hy.data(), dy.p, (size_t)N * b * 8, cudaMemcpyDeviceToHost, c->stream), "d2h");
  check_cuda(cudaStreamSynchronize(c->stream), "sync");
  for (long long i = 0; i < N * b; ++i) Y[i] = hy[i] % c->p;
  release(c, dv);
  release(c, dy);
  API_END
}

int f4b_plan_free(f4b_plan* pl) {
  plan_release(pl);
  return F4B_OK;
}

int f4b_psge_plan(f4b_ctx* h, const f4b_plan* pl, int mode, f4b_echelon** out) {
  if (!h || !pl || !out) return F4B_ERR_PRECONDITION;
  *out = nullptr;
  API_BEGIN(&h->c)
  *out = psge_plan(_c, pl, mode);
  API_END
}

int f4b_psge_csr(f4b_ctx* h, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col_ind,
                 const uint64_t* val, int mode, f4b_echelon** out) {
  if (!h || !out) return F4B_ERR_PRECONDITION;
  *out = nullptr;
  API_BEGIN(&h->c)
  *out = psge_csr(_c, n_rows, n_cols, row_ptr, col_ind, val, mode);
  API_END
}

int f4b_echelon_complete(f4b_ctx* h, f4b_echelon* e) {
  if (!h || !e) return F4B_ERR_PRECONDITION;
  API_BEGIN(&h->c)
  echelon_complete(_c, e);
  API_END
}

int f4b_echelon_complete_rows(f4b_ctx* h, f4b_echelon* e, const int64_t* lead_cols, int64_t n) {
  if (!h || !e || n < 0 || (n && !lead_cols)) return F4B_ERR_PRECONDITION;
  API_BEGIN(&h->c)
  echelon_complete_rows(_c, e, lead_cols, n);
  API_END
}

int f4b_echelon_get_info(const f4b_echelon* e, f4b_echelon_info* info) {
  if (!e || !info) return F4B_ERR_PRECONDITION;
  echelon_info(e, info);
  return F4B_OK;
}

int f4b_echelon_download(const f4b_echelon* e, int which, int64_t* leads, int64_t* row_ptr, int64_t* cols,
                         uint64_t* vals) {
  if (!e) return F4B_ERR_PRECONDITION;
  try {
    echelon_download(e, which, leads, row_ptr, cols, vals);
  } catch (const Error& er) {
    return er.code;
  }
  return F4B_OK;
}

int f4b_echelon_pivot_cols(const f4b_echelon* e, int64_t* cols) {
  if (!e) return F4B_ERR_PRECONDITION;
  try {
    echelon_pivot_cols(e, cols);
  } catch (const Error& er) {
    return er.code;
  }
  return F4B_OK;
}

int f4b_basis_append_echelon(f4b_ctx* h, const f4b_plan* plan, const f4b_echelon* ech) {
  if (!h || !plan || !ech) return F4B_ERR_PRECONDITION;
  API_BEGIN(&h->c)
  basis_finish(_c);
  basis_append_echelon(_c, plan, ech);
  API_END
}

int f4b_echelon_free(f4b_echelon* e) {
  echelon_release(e);
  return F4B_OK;
}

int f4b_spmm(f4b_ctx* h, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr, const int64_t* col_ind,
             const uint64_t* val, const uint64_t* X, int64_t b, uint64_t* Y) {
  if (!h) return F4B_ERR_PRECONDITION;
  API_BEGIN(&h->c)
  spmm(_c, n_rows, n_cols, row_ptr, col_ind, val, X, b, Y);
  API_END
}

int f4b_dict_build(f4b_ctx* h, const uint64_t* keys, int64_t n, int words, int key_bits, uint64_t* out,
                   int64_t* n_unique) {
  if (!h || !n_unique) return F4B_ERR_PRECONDITION;
  API_BEGIN(&h->c)
  *n_unique = dict_build(_c, keys, n, words, key_bits, out);
  API_END
}

int f4b_join_index(f4b_ctx* h, const uint64_t* dict, int64_t n_dict, const uint64_t* keys, int64_t n, int words,
                   int64_t* pos) {
  if (!h) return F4B_ERR_PRECONDITION;
  API_BEGIN(&h->c)
  join_index(_c, dict, n_dict, keys, n, words, pos);
  API_END
}

int f4b_mod_fma(f4b_ctx* h, uint32_t p, const uint64_t* a, const uint64_t* b, const uint64_t* acc, int64_t n,
                uint64_t* out) {
  if (!h) return F4B_ERR_PRECONDITION;
  API_BEGIN(&h->c)
  mod_fma(_c, p, a, b, acc, n, out);
  API_END
}

}  // extern "C"

void f4b::basis_finish(Ctx* c) { basis_finish_impl(c); }
bool f4b::basis_apply_lazy(Ctx* c) { return basis_apply_lazy_impl(c); }
