// Internal (C++) interface between the translation units of libf4b200.so.
// The public C ABI is include/f4b200.h.
#pragma once
#include <cstddef>
#include <cstdint>
#include <string>
#include <vector>
#include <cuda_runtime.h>

#include "../../include/f4b200.h"

namespace f4b {

struct Ctx;

// A device buffer obtained through the context allocator (torch caching
// allocator when the Python host registers it, cudaMalloc otherwise).
struct DBuf {
  void* p = nullptr;
  size_t cap = 0;
  template <class T> T* as() const { return reinterpret_cast<T*>(p); }
};

// Per-status error carrying a C-ABI code.
struct Error {
  int code;
  std::string msg;
};

void ensure(Ctx* c, DBuf& b, size_t bytes);  // grow-only; contents not preserved
void ensure_keep(Ctx* c, DBuf& b, size_t bytes);  // grow-only; contents preserved
void release(Ctx* c, DBuf& b);
void basis_finish(Ctx* c);  // completes a pending asynchronous basis append
bool basis_apply_lazy(Ctx* c);
void recheck_lanes(Ctx* c, long long r0, const int32_t* rb, const uint16_t* shift);  // advances the host mirrors of a pending key append without waiting (true if pending)
void pool_flush(Ctx* c);
void check_cuda(cudaError_t e, const char* what);  // throws Error{F4B_ERR_CUDA}
[[noreturn]] void fail(int code, const std::string& msg);

// Timing helper: CUDA events recorded on the context stream.
struct EventPair {
  cudaEvent_t a = nullptr, b = nullptr;
};

struct Basis {
  int n_polys = 0;
  long long n_terms = 0;
  // host mirrors (small): lengths, offsets, LM exps, LM degrees, per-poly max exps
  std::vector<int64_t> h_len, h_off;
  std::vector<uint16_t> h_lm;    // n_polys * n_vars
  std::vector<uint16_t> h_maxe;  // n_polys * n_vars
  // device streams
  DBuf exps;    // u16 [T * n]
  DBuf coeff;   // u32 [T]
  DBuf off;     // u32 [n_polys + 1]
  DBuf len;     // u32 [n_polys]
  DBuf lmexp;   // u16 [n_polys * n]
  // cached device keys for the current key format
  DBuf ckey;    // u64 [T * KW]
  DBuf maxe;    // u16 [n_polys * n] per-polynomial max exponent per variable
  int ckey_lane_bits = -1, ckey_words = 0;
  long long ckey_terms = 0;  // terms already encoded in this format
  // nonzero polynomials sorted by (key(LM), index): the closure preference
  // order (symbolic.py:228-235), extended incrementally on append
  std::vector<int32_t> lm_order;
  int lm_sorted = 0;  // polynomials [0, lm_sorted) are merged into lm_order
  // LMs packed two 16-bit lanes per word (the closure kernels' LM table
  // format), polynomials [0, lmw_polys) done
  std::vector<uint32_t> h_lmw;
  int lmw_polys = 0;
};

struct Ctx {
  int device = 0;
  uint32_t p = 0;
  int n_vars = 0;
  int order = 0;
  f4b_alloc_fn alloc = nullptr;
  f4b_free_fn dfree = nullptr;
  void* user = nullptr;
  // without a registered allocator: a per-context stream-ordered pool
  // (cudaMallocFromPoolAsync, memory retained by the pool: no device
  // synchronisation and no host callback per buffer)
  cudaMemPool_t mempool = nullptr;
  // page-locked staging of f4b_basis_append* (lengths / prefix up, LM and
  // max-exponent rows + error flag down: async copies, one sync per call)
  void* h_app = nullptr;
  size_t h_app_cap = 0;
  // an f4b_basis_append_wide_async whose host side (range-check flag, LM and
  // max-exponent mirrors) is completed by the next call that needs it
  struct PendingAppend {
    bool active = false;
    long long n_polys = 0, T0 = 0, P0 = 0, T1 = 0, P1 = 0;
    size_t o_lm = 0, o_mx = 0, o_bad = 0;
    std::vector<int64_t> lengths;
    DBuf raw;
    // key appends of a graded ring: the host mirrors can be advanced before
    // the device finishes (basis_apply_lazy) from the LMs read off the host
    // keys, with deg(LM) as the bound of every exponent (terms descend in a
    // graded order); basis_finish then checks the flag and installs the
    // exact maximum exponents, or rolls the mirrors back
    bool lazy_ok = false, applied = false;
    std::vector<uint16_t> lm_host, bound_host;
  } pend;
  cudaStream_t stream = 0;
  cudaStream_t copy_stream = nullptr;  // plan prefetches (created on first use)
  int num_sms = 148;
  // path selection (f4b_ctx_set_option); the defaults are the measured best
  // paths, the others are the fallbacks the automatic choice takes when a
  // shape does not fit, forced here so the parity tests reach every kernel
  int opt_sweep = 0;        // "sweep": 0 auto, 1 blocked sweep, 2 k_sweep only
  int opt_dense_rows = 0;   // "dense_rows": 0 auto (D' rows in shared memory when they fit), 1 always in HBM
  int opt_dense = 0;        // "dense": 0 pivot blocks (k_dense_blk), 1 k_dense_forward
  int opt_fbsp = 0;         // "fbsp": 0 one cooperative k_fbsp, 1 multi-launch rank path
  int opt_dict_sort = 0;    // "dict_sort": 1 = radix-sort dictionary even for grevlex
  int opt_dict_lsd = 0;  // "dict_lsd": 1 = f4b_dict_build sorts every key (LSD), no MSD bucket pass
  std::string last_error;
  Basis basis;
  // pinned host scratch for round counters
  uint32_t* h_stat = nullptr;
  // reusable device scratch
  DBuf scan_tmp, sort_a, sort_b, sort_hist, flags, errflag, tmp_u32a, tmp_u32b, tmp_u32c;
  // FBSP scratch (grow-only, reused across compile_batch calls)
  DBuf rows_basis, rows_delta, rows_len, rows_start, keys_all, vals_all;
  DBuf dict_a, dict_b, front, front_new, uniq, red, lmpref, cand_idx, shift_in;
  DBuf cl_basis, cl_shift, cl_round, loop_scratch;
  long long closure_cap_hint = 0;  // frontier / closure-row capacity of the persistent loop
  long long m_cap_hint = 0, n_cap_hint = 0;  // plan capacities of the fused FBSP kernel
  void* h_stage = nullptr;                   // page-locked H2D staging (grow-only)
  size_t h_stage_cap = 0;
  std::vector<uint32_t> h_binom;  // binomial table of the rank path, cached per (rows, n)
  int h_binom_rows = -1, h_binom_n = -1;
  DBuf dstage;
  // k_fbsp presence maps + chunk counters: zero between calls; the first
  // maps_clean bytes of `maps` are known to be zero
  DBuf maps, dwp;
  size_t maps_clean = 0;
  DBuf fcnt;          // two sets of 4G chunk counters (alternating per call)
  int fcnt_G = 0, fcnt_parity = 0;
  int fbsp_bps = -1;
  size_t fbsp_bps_smem = 0;
  // released buffers kept for reuse on the context stream (stream-ordered,
  // like the caching allocator itself, without a host callback per buffer)
  std::vector<std::pair<void*, size_t>> pool;
  size_t pool_bytes = 0;
  uint32_t pprime = 0, r2 = 0;
  long long launches = 0;        // kernel launches issued (reset per compile call)
  long long total_launches = 0;  // monotonically increasing
  long long raw_allocs = 0, raw_frees = 0;  // device allocations / frees past the buffer cache
  double raw_alloc_us = 0;                  // host time inside them
  // optional per-kernel CUDA-event timing (f4b_ctx_profile)
  bool prof = false;
  std::vector<cudaEvent_t> ev_pool;
  cudaEvent_t tev[4] = {};  // per-call timing events (created once, reused)
  size_t ev_used = 0;
  struct Pending {
    const char* name;
    size_t e0, e1;
  };
  std::vector<Pending> pending;
  std::vector<std::pair<std::string, std::pair<double, long long>>> prof_acc;
};

// RAII scope: records CUDA events around one launch when profiling is on.
struct ProfScope {
  Ctx* c;
  const char* name;
  size_t e0 = 0;
  ProfScope(Ctx* c_, const char* n);
  ~ProfScope();
};

#define F4B_LAUNCH(c, kern, grid, block, smem, ...)                   \
  do {                                                                \
    ::f4b::ProfScope _f4b_ps((c), #kern);                             \
    kern<<<(grid), (block), (smem), (c)->stream>>>(__VA_ARGS__);      \
    ::f4b::check_cuda(cudaGetLastError(), #kern);                     \
  } while (0)

// scan.cu: exclusive scan of n u32 values into out (n+1 entries; out[n] = total).
void exclusive_scan_u32(Ctx* c, const uint32_t* in, uint32_t* out, long long n);
// exclusive scan where in[i] = (flags[i] != 0)
void exclusive_scan_flags(Ctx* c, const uint8_t* flags, uint32_t* out, long long n);

// radix.cu: ascending unique keys of in[0, n) (n = *d_n if d_n, else n_max),
// dropping keys present in the ascending dictionary `dict` (size *d_ndict)
// when dict != nullptr; result compacted into out, count into *d_count.
// Only the low `bits` bits of the keys vary.  No host synchronisation.
void sort_unique(Ctx* c, int KW, const uint64_t* in, const uint32_t* d_n, uint32_t n_max, int bits,
                 const uint64_t* dict, const uint32_t* d_ndict, uint64_t* out, uint32_t* d_count);

uint32_t read_u32(Ctx* c, const uint32_t* dptr);  // synchronous small D2H
cudaEvent_t timing_event(Ctx* c, int i);           // reusable event i < 4 of the context
void memset_async(Ctx* c, void* p, int v, size_t bytes);

}  // namespace f4b

// ---------------------------------------------------------------------------
// Opaque objects of the C ABI
// ---------------------------------------------------------------------------
struct f4b_plan {
  f4b::Ctx* ctx = nullptr;
  int KW = 1, lane_bits = 1;
  long long r = 0, r0 = 0, N = 0, M = 0, closure_rounds = 0;
  long long sort_passes = 0, launches = 0;
  int64_t dict_ns = 0, asm_ns = 0;
  f4b::DBuf row_ptr;    // u32 [r+1]
  f4b::DBuf col_ind;    // u32 [M]
  f4b::DBuf val;        // u32 [M]
  f4b::DBuf dict;       // u64 [N*KW] ascending device keys
  f4b::DBuf dict_exps;  // u16 [N*n] descending (column order)
  f4b::DBuf cl_basis;   // i32 [r-r0]
  f4b::DBuf cl_shift;   // u16 [(r-r0)*n]
  f4b::DBuf cl_round;   // i32 [r-r0]
  // slice of a sharded compile (shard.cu): rows [row_lo, row_lo + r) of the
  // r_total final rows; the closure metadata covers all ncl_all closure rows
  long long row_lo = 0, r_total = -1, ncl_all = -1;
  long long n_closure() const { return ncl_all >= 0 ? ncl_all : r - r0; }
  // asynchronous host download (f4b_plan_prefetch): staging and completion
  f4b::DBuf pf_wide;
  cudaEvent_t pf_done = nullptr;
  bool pf_pending = false;
  bool validated = false;  // the compile ran f4b_plan_validate's checks (fused, io.cu)
};

struct f4b_echelon;

namespace f4b {
void plan_release(f4b_plan* pl);
void ref_keys_device(Ctx* c, const f4b_plan* pl, unsigned long long* out, int W);  // capi.cu
// io.cu: LayoutPlan.validate on the device with the sizes read on the device
// (sz[0] = r, sz[2] = M, sz[3] = N: the LoopOut layout), result in *flag
// (~0 = valid); validate_message turns a flag into the reference's message
void validate_launch_dev(Ctx* c, const f4b_plan* pl, const uint32_t* sz, unsigned long long* flag);
std::string validate_message(unsigned long long f, long long row_lo);
}

namespace f4b {
void compile_batch(Ctx* c, long long r0, const int32_t* rb, const uint16_t* shift, int closure, const int32_t* cands,
                   long long n_cands, long long dict_cap, f4b_plan* pl);
f4b_echelon* psge_plan(Ctx* c, const f4b_plan* pl, int mode);
f4b_echelon* psge_csr(Ctx* c, long long r, long long N, const int64_t* rp, const int64_t* col, const uint64_t* val,
                      int mode);
void echelon_complete(Ctx* c, f4b_echelon* E);
void echelon_complete_rows(Ctx* c, f4b_echelon* E, const int64_t* lead_cols, long long n);
void echelon_info(const f4b_echelon* E, f4b_echelon_info* info);
void echelon_download(const f4b_echelon* E, int which, int64_t* leads, int64_t* row_ptr, int64_t* cols, uint64_t* vals);
void echelon_release(f4b_echelon* E);
void basis_append_echelon(Ctx* c, const f4b_plan* pl, const f4b_echelon* E);
void echelon_pivot_cols(const f4b_echelon* E, int64_t* cols);
void spmm(Ctx* c, long long r, long long N, const int64_t* rp, const int64_t* col, const uint64_t* val,
          const uint64_t* X, long long b, uint64_t* Y);
// micro.cu: the reference microbenchmark primitives on device buffers
long long dict_build(Ctx* c, const uint64_t* keys, long long n, int words, int key_bits, uint64_t* out);
void join_index(Ctx* c, const uint64_t* dict, long long nd, const uint64_t* keys, long long n, int words,
                int64_t* pos);
void mod_fma(Ctx* c, uint32_t p, const uint64_t* a, const uint64_t* b, const uint64_t* acc, long long n,
             uint64_t* out);
}  // namespace f4b
