/*
 * f4b200.h — C ABI of the B200-native F4 hot path (libf4b200.so).
 *
 * The reference (arXiv 2601.06765, package `fpgb`) has no FFI: its boundary
 * is the set of module-level Python functions that the F4 driver calls
 * (pkg/src/fpgb/groebner.py:32-50, call site f4_step :253-311).  These entry
 * points are what a binding of that boundary needs; the Python shim
 * (paper_2601_06765_b200/_capi.py) binds them with ctypes and keeps the
 * reference signatures.  Each function cites the reference interface it
 * replaces.
 *
 * Conventions
 *  - Every call returns F4B_OK (0) or an f4b_status code; the message of the
 *    last failure is available from f4b_ctx_last_error().  Codes map 1:1 onto
 *    the reference exception classes (pkg/src/fpgb/errors.py).
 *  - Arrays named h_* / passed as `const T*` without "device" in the comment
 *    are HOST pointers.  Device memory is owned by the context and obtained
 *    through the registered allocator when one is given; with a NULL
 *    allocator (the Python host's default) from a per-context stream-ordered
 *    cudaMemPool (cudaMallocFromPoolAsync / cudaFreeAsync on the context
 *    stream, memory retained by the pool).
 *  - All work is issued on the stream set with f4b_ctx_set_stream (default
 *    stream 0).  One context per (device, ring); calls on one context are not
 *    thread-safe.
 *  - Inputs are never modified; every plan / echelon is a fresh object that
 *    stays valid until freed (reference ownership rule).
 */
#ifndef F4B200_H
#define F4B200_H

#include <stddef.h>
#include <stdint.h>

#ifdef __cplusplus
extern "C" {
#endif

enum f4b_status {
  F4B_OK = 0,
  F4B_ERR_MISSING_KEY = 1,     /* MissingKeyError  (bulk.py:235-240)          */
  F4B_ERR_SIZE_CAP = 2,        /* SizeCapError     (symbolic.py:359-363)      */
  F4B_ERR_LANE_OVERFLOW = 3,   /* LaneOverflowError (monomials.py:142-147)    */
  F4B_ERR_PROPERTY = 4,        /* PropertyViolationError (symbolic.py:214-215)*/
  F4B_ERR_PRECONDITION = 5,    /* PreconditionError (sparselin.py:288-289)    */
  F4B_ERR_CUDA = 6,            /* CUDA runtime / launch failure               */
  F4B_ERR_OOM = 7,             /* device allocation failed                    */
  F4B_ERR_PROBABILISTIC = 8    /* ProbabilisticFailureError                   */
};

enum f4b_order { F4B_GREVLEX = 0, F4B_DEGLEX = 1, F4B_LEX = 2 };
enum f4b_closure { F4B_SUPPORT_ONLY = 0, F4B_ONE_STEP_REDUCTION = 1 };
enum f4b_psge_mode { F4B_NEW_ONLY = 0, F4B_FULL_RREF = 1 };

typedef void* (*f4b_alloc_fn)(size_t bytes, void* user);
typedef void (*f4b_free_fn)(void* device_ptr, void* user);

typedef struct f4b_ctx f4b_ctx;
typedef struct f4b_plan f4b_plan;
typedef struct f4b_echelon f4b_echelon;

int f4b_abi_version(void);

/* Context = FieldModulus + Ring on one device (fp.py:80-128, monomials.py:40-95). */
int f4b_ctx_create(int device, uint32_t p, int n_vars, int order, f4b_alloc_fn alloc,
                   f4b_free_fn dfree, void* user, f4b_ctx** out);
int f4b_ctx_destroy(f4b_ctx* ctx);
int f4b_ctx_set_stream(f4b_ctx* ctx, void* cuda_stream);
const char* f4b_ctx_last_error(const f4b_ctx* ctx);
/* Path selection (no reference counterpart: the reference has one path per
 * function).  Every setting computes the same bytes; the non-default ones
 * force the fallback kernels the automatic choice takes for shapes the
 * default path does not fit, so tests can reach them:
 *   "sweep"       0 auto | 1 blocked C-row sweep | 2 generic k_sweep
 *   "dense"       0 pivot-block RREF(D') | 1 per-pivot k_dense_forward
 *   "dense_rows"  0 auto (a CTA's D' rows in shared memory when they fit) | 1 in HBM
 *   "fbsp"        0 one cooperative k_fbsp | 1 multi-launch rank pipeline
 *   "dict_sort"   1 = radix-sort dictionary for grevlex too
 *   "dict_lsd"    1 = f4b_dict_build sorts every key (LSD), no MSD buckets */
int f4b_ctx_set_option(f4b_ctx* ctx, const char* name, int64_t value);
/* Instrumentation: when enabled, every kernel launch is bracketed by CUDA
 * events on the context stream; profile_read resolves them into lines
 * "kernel launches total_ns" and reports the total launch count. */
int f4b_ctx_profile(f4b_ctx* ctx, int enable);
int f4b_ctx_profile_read(f4b_ctx* ctx, char* buf, int64_t buflen, int64_t* total_launches);

/* Device-resident basis — replaces soa_pack / SoaPolySet
 * (polynomials.py:243-299, groebner.py:143-146).  `exps` is [T][n_vars] u16,
 * `coeffs` [T] standard residues, `lengths` [n_polys]; each polynomial's terms
 * strictly descending in the term order, leading term first. */
int f4b_basis_clear(f4b_ctx* ctx);
int f4b_basis_append(f4b_ctx* ctx, int64_t n_polys, const int64_t* lengths,
                     const uint16_t* exps, const uint32_t* coeffs);
/* Same, for the reference's own SoaPolySet streams (soa_pack,
 * polynomials.py:248-262): exps [T][n_vars] int64, coeffs [T] uint64.  The
 * narrowing, the range checks (0 <= e <= 0xFFFF -> F4B_ERR_LANE_OVERFLOW,
 * 1 <= c < p -> F4B_ERR_PROPERTY) and the per-polynomial LM / maximum
 * exponents run on the device; page-locked host buffers copy at full rate. */
int f4b_basis_append_wide(f4b_ctx* ctx, int64_t n_polys, const int64_t* lengths,
                          const int64_t* exps, const uint64_t* coeffs);
/* Same, without waiting for the device: the host-side completion (range-check
 * result, LM / max-exponent mirrors) happens in the next call that needs the
 * basis (f4b_compile_batch, f4b_basis_*), which then reports a range error of
 * this append (the basis is left as it was).  The caller's host buffers must
 * stay valid until that call.  f4b_basis_sync completes it explicitly. */
int f4b_basis_append_wide_async(f4b_ctx* ctx, int64_t n_polys, const int64_t* lengths,
                                const int64_t* exps, const uint64_t* coeffs);
/* Same as f4b_basis_append_wide_async with the terms given by the reference
 * keys of the SoaPolySet (mon_key [T][key_words] uint64, monomials.py
 * mon_key_pack / key_pack_vec) instead of the int64 exponent rows: 8 W bytes
 * per term up instead of 8 n (cyclic-8: 24 instead of 64).  The exponents are
 * recovered from the 16-bit lanes on the device; a degree lane that differs
 * from the lanes' sum, or nonzero padding bits, is F4B_ERR_PROPERTY (the
 * reference's CorruptKeyError condition, key_unpack_vec). */
int f4b_basis_append_keys_async(f4b_ctx* ctx, int64_t n_polys, const int64_t* lengths,
                                const uint64_t* keys, int key_words, const uint64_t* coeffs);
int f4b_basis_sync(f4b_ctx* ctx);
int f4b_basis_size(const f4b_ctx* ctx, int64_t* n_polys, int64_t* n_terms);

typedef struct {
  int64_t r, N, M, closure_rounds, n_closure_rows;
  int64_t key_words, lane_bits;
  int64_t dict_build_ns, row_assemble_ns; /* device time (CUDA events) */
  int64_t sort_passes, kernel_launches;
  int64_t row_lo, r_total; /* a sharded-compile slice: rows [row_lo, row_lo + r) of r_total */
  int64_t validated;       /* 1: f4b_plan_validate's checks already ran inside the compile */
} f4b_plan_info;

/* compile_batch (symbolic.py:293-388): rows in select_rows order
 * (symbolic.py:166-201): row_basis[r], row_shift[r][n_vars].  closure is an
 * f4b_closure; candidates (may be NULL = all basis polys) restricts the
 * closure reducers (symbolic.py:228-235).  dict_cap mirrors DICT_CAP. */
int f4b_compile_batch(f4b_ctx* ctx, int64_t n_rows, const int32_t* row_basis,
                      const uint16_t* row_shift, int closure, const int32_t* candidates,
                      int64_t n_candidates, int64_t dict_cap, f4b_plan** out);
int f4b_plan_get_info(const f4b_plan* plan, f4b_plan_info* info);
/* LayoutPlan arrays (symbolic.py:99-163) to host memory; any pointer may be NULL.
 * dict_exps is [N][n_vars], columns in DESCENDING term order (column 0 is the
 * greatest monomial); closure rows (appended after the input rows) report
 * their basis index, shift and discovery round. */
int f4b_plan_download(const f4b_plan* plan, int64_t* row_ptr, int64_t* col_ind, uint64_t* val,
                      uint16_t* dict_exps, int32_t* closure_basis, uint16_t* closure_shift,
                      int32_t* closure_round);
/* LayoutPlan.dict_keys (symbolic.py:99-163): reference keys
 * (monomials.py:131-148; big-endian u64 words, W = ceil((32 [graded] +
 * 16 n_vars) / 64)) in column order (descending), [N][W], built on the device. */
int f4b_plan_download_ref_keys(const f4b_plan* plan, uint64_t* keys);
/* Y = Aᵀ V over the plan's matrix (A = r x N, V [r][b], Y [N][b], u64
 * residues): the left-kernel check vᵀA = 0 of verify_kernel_syzygy
 * (groebner.py:409-428) — row i of the plan is exactly t_i g_{k_i} over the
 * dictionary, so Y = 0 is the exact recombination Σ v_i t_i g_{k_i} = 0. */
int f4b_plan_left_apply(const f4b_plan* plan, const uint64_t* V, int64_t b, uint64_t* Y);
int f4b_plan_free(f4b_plan* plan);
/* plan_to_text (symbolic.py:438-460) number lists formatted on the device:
 * which = 0 row_ptr, 1 col_ind, 2 val, 3 dict_keys (reference key words, row
 * major); decimal numbers separated by one space, no label, no newline.
 * *length receives the byte count; the text is written when cap >= length
 * (call with out = NULL to size the buffer). */
int f4b_plan_text(const f4b_plan* plan, int which, char* out, int64_t cap, int64_t* length);

/* Asynchronous host download on the context's copy stream, behind the plan's
 * completion (the next compile runs meanwhile): block = one host buffer of
 * r+1 + 2M + N*W 64-bit words receiving row_ptr, col_ind (int64), val
 * (uint64) and the reference dictionary keys [N][W] (as
 * f4b_plan_download_ref_keys) — symbolic.py:383-388's host arrays, built by
 * one kernel and copied in one D2H.  Page-locked memory copies at full link
 * rate.  f4b_plan_wait blocks until the block is complete; freeing the plan
 * waits too. */
int f4b_plan_prefetch(f4b_plan* plan, uint64_t* block, int W);
int f4b_plan_wait(f4b_plan* plan);

/* LayoutPlan.validate (symbolic.py:125-163, called by compile_batch at
 * :383-387) on the device buffers: row_ptr tiles [0, M), rows nonempty with
 * strictly ascending in-range columns, values nonzero (and < p), dictionary
 * strictly descending in the ring order.  F4B_ERR_PROPERTY with the
 * reference's message on the first violation in its check order;
 * *violation (optional) = -1 or the encoded (kind << 40 | index). */
int f4b_plan_validate(const f4b_plan* plan, int64_t* violation);

/* fault injection for validation tests: plan row_ptr (0) / col_ind (1) /
 * val (2) entry `index` := value (device write, synchronous). */
int f4b_plan_poke(f4b_plan* plan, int which, int64_t index, uint32_t value);

/* ---- sharded compile_batch (one rank per GPU) ----
 * The stages of compile_batch (symbolic.py:293-388) between which the caller
 * all-gathers the small per-rank outputs (NCCL or gloo).  Every rank passes
 * the SAME rows, candidates and gathered data; rank k owns the contiguous,
 * length-balanced input rows [row_lo, row_hi), frontier slice
 * [f_lo, f_hi) per round and final rows [row_lo, row_hi) of the join.
 * Concatenating the finish() slices in rank order is the single-GPU plan.
 * Run / rank / reducer buffers may be host or device pointers.  grevlex
 * rank path only (else F4B_ERR_PRECONDITION).
 *   begin        -> *n_run = length of this rank's sorted unique run of
 *                   monomial ranks (ascending = ascending key)
 *   take_run     copy it out (n_run u32)
 *   merge        all gathered runs (concatenated) -> dictionary, round-1
 *                frontier size
 *   round        this rank's frontier slice: red_out[f_hi - f_lo] = reducer
 *                basis index or -1, *n_run = its run of new monomials
 *   round_merge  all reducer indices (frontier order) + all new runs -> the
 *                round's rows, next frontier size (0 = closure done)
 *   rows         final row count and row starts (r_total + 1, may be NULL)
 *   finish       the join of final rows [row_lo, row_hi) -> a plan slice */
typedef struct f4b_shard f4b_shard;
int f4b_shard_begin(f4b_ctx* ctx, int64_t n_rows, const int32_t* row_basis, const uint16_t* row_shift,
                    int closure, const int32_t* candidates, int64_t n_candidates, int64_t dict_cap,
                    int64_t row_lo, int64_t row_hi, f4b_shard** out, int64_t* n_run);
int f4b_shard_take_run(f4b_shard* sh, uint32_t* out, int64_t n_run);
int f4b_shard_merge(f4b_shard* sh, const uint32_t* ranks, int64_t n, int64_t* n_frontier);
int f4b_shard_round(f4b_shard* sh, int64_t f_lo, int64_t f_hi, int32_t* red_out, int64_t* n_run);
int f4b_shard_round_merge(f4b_shard* sh, const int32_t* red_all, int64_t n_frontier, const uint32_t* ranks,
                          int64_t n, int64_t* n_next_frontier);
int f4b_shard_rows(f4b_shard* sh, int64_t* r_total, uint32_t* row_start);
int f4b_shard_finish(f4b_shard* sh, int64_t row_lo, int64_t row_hi, f4b_plan** out);
/* closure rounds so far, dictionary size, this rank's summed device time */
int f4b_shard_info(const f4b_shard* sh, int64_t* rounds, int64_t* n_dict, int64_t* device_ns);
int f4b_shard_free(f4b_shard* sh);

typedef struct {
  int64_t n_rows, n_cols, rank, zero_rows;
  int64_t n_pivot_rows, n_nonpivot_rows;  /* pivot rows valid once full */
  int64_t pivot_nnz, nonpivot_nnz;
  int64_t full;                           /* 1 once pivot rows are computed */
  int64_t numeric_ns, backsub_ns;         /* device time (CUDA events) */
  int64_t dense_rows, dense_cols;         /* D' block shape */
  int64_t sweep_pivots;                   /* pivot-row applications in the C-row sweep */
  int64_t sweep_tail_nnz;                 /* pivot-row tail entries those applications read */
} f4b_echelon_info;

/* psge_reduce (sparselin.py:281-369) on a compiled plan (no copy) or on a
 * host CSR (csr_from_arrays, sparselin.py:80-90).  F4B_NEW_ONLY computes the
 * rows with new leading columns (all the F4 driver consumes,
 * groebner.py:285-287); F4B_FULL_RREF also back-reduces the pivot rows. */
int f4b_psge_plan(f4b_ctx* ctx, const f4b_plan* plan, int mode, f4b_echelon** out);
int f4b_psge_csr(f4b_ctx* ctx, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                 const int64_t* col_ind, const uint64_t* val, int mode, f4b_echelon** out);
int f4b_echelon_complete(f4b_ctx* ctx, f4b_echelon* ech); /* NEW_ONLY -> FULL_RREF */
/* FULL_RREF restricted to the pivot rows led by the n given columns (the
 * final interreduction needs only the rows led by the basis' leading
 * monomials, groebner.py:314-332): those rows are back-reduced exactly as
 * f4b_echelon_complete does it, the other pivot rows come back empty and
 * f4b_echelon_info.full reports 2. */
int f4b_echelon_complete_rows(f4b_ctx* ctx, f4b_echelon* ech, const int64_t* lead_cols, int64_t n);
int f4b_echelon_get_info(const f4b_echelon* ech, f4b_echelon_info* info);
/* which = 0: pivot rows, 1: nonpivot rows; rows ascending by lead column.
 * leads[k], row_ptr[k+1], cols/vals concatenated (standard residues). */
int f4b_echelon_download(const f4b_echelon* ech, int which, int64_t* leads, int64_t* row_ptr,
                         int64_t* cols, uint64_t* vals);
/* pivot_cols (ascending, rank entries) — available in both modes. */
int f4b_echelon_pivot_cols(const f4b_echelon* ech, int64_t* cols);
int f4b_echelon_free(f4b_echelon* ech);
/* The F4 harvest on the device (groebner.py:285-290): append
 * the echelon's nonpivot rows (new leading monomials) to the device basis in
 * the driver's order (ascending key(LM)), exponents gathered from the plan's
 * dictionary (plan = the echelon's input), coefficients from the echelon —
 * device to device, no host copy of the terms. */
int f4b_basis_append_echelon(f4b_ctx* ctx, const f4b_plan* plan, const f4b_echelon* ech);

/* csr_transpose (sparselin.py:108-121): stable counting-sort transpose on
 * the device; host CSR in (n_rows x n_cols), host CSR out (n_cols x n_rows:
 * t_row_ptr [n_cols + 1], t_col_ind / t_val [nnz]). */
int f4b_csr_transpose(f4b_ctx* ctx, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                      const int64_t* col_ind, const uint64_t* val, int64_t* t_row_ptr,
                      int64_t* t_col_ind, uint64_t* t_val);

/* spmm (sparselin.py:142-173): Y = A X mod p; A host CSR (n_rows x n_cols),
 * X host [n_cols][b], Y host [n_rows][b]; u64 standard residues. */
int f4b_spmm(f4b_ctx* ctx, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
             const int64_t* col_ind, const uint64_t* val, const uint64_t* X, int64_t b,
             uint64_t* Y);

/* ---- isolated primitives of the reference microbenchmarks (bench.py:244-300) ----
 * DEVICE pointers (e.g. torch tensors); synchronous on the context stream.
 *
 * f4b_dict_build replaces radix_sort + unique_sorted (bulk.py:86-124, :135-150)
 * as called by microbench("dict_build") (bench.py:253-256): keys [n][words]
 * (words in {1,2}, every word < 2^key_bits) -> ascending unique keys in
 * out [n_unique][words] (out must hold n keys). */
int f4b_dict_build(f4b_ctx* ctx, const uint64_t* keys, int64_t n, int words, int key_bits,
                   uint64_t* out, int64_t* n_unique);
/* f4b_join_index replaces merge_join_index (bulk.py:207-241), microbench
 * ("row_assemble") (bench.py:278-282): pos[i] = index of keys[i] in the ascending
 * dictionary dict [n_dict][words] (words 1..4); F4B_ERR_MISSING_KEY on a miss. */
int f4b_join_index(f4b_ctx* ctx, const uint64_t* dict, int64_t n_dict, const uint64_t* keys,
                   int64_t n, int words, int64_t* pos);
/* f4b_mod_fma: out = (acc + a b) mod p (fp.py:335-400 KernelArith lazy
 * multiply-add; microbench("mod_fma"), bench.py:293-300); 3 <= p < 2^31,
 * inputs < p, 16-byte aligned buffers. */
int f4b_mod_fma(f4b_ctx* ctx, uint32_t p, const uint64_t* a, const uint64_t* b,
                const uint64_t* acc, int64_t n, uint64_t* out);

/* berlekamp_massey (sparselin.py:377-413) for b sequences of length len
 * (seqs [b][len] u64 residues) side by side, one CTA per sequence: polys
 * [b][len + 1] receives each minimal polynomial ascending and monic
 * (reversed connection polynomial, the reference's return value) in its first
 * degrees[j] + 1 entries. */
int f4b_bm(f4b_ctx* ctx, const uint64_t* seqs, int64_t len, int64_t b, uint64_t* polys, int64_t* degrees);

/* Device-resident black-box operator for Block Wiedemann (sparselin.py:450-548):
 * B = A (square, normal = 0) or B = AᵀA (normal = 1, Aᵀ built once).  The CSR
 * stays in HBM across applications; vectors are host [dim][b] u64 residues. */
typedef struct f4b_op f4b_op;
int f4b_op_create(f4b_ctx* ctx, int64_t n_rows, int64_t n_cols, const int64_t* row_ptr,
                  const int64_t* col_ind, const uint64_t* val, int normal, f4b_op** out);
int f4b_op_free(f4b_op* op);
/* Y = B X */
int f4b_op_apply(f4b_op* op, const uint64_t* X, int64_t b, uint64_t* Y);
/* seqs[k][j] = sum_i U[i][j] (B^k V)[i][j] mod p for k < steps (the Krylov
 * projections, sparselin.py:408-412), all applications on the device */
int f4b_op_krylov(f4b_op* op, const uint64_t* U, const uint64_t* V, int64_t b, int64_t steps,
                  uint64_t* seqs);
/* out = sum_i g[i] B^i v, Horner from g[len-1] (sparselin.py:425-429) */
int f4b_op_horner(f4b_op* op, const uint64_t* g, int64_t len, const uint64_t* v, uint64_t* out);
/* acc = v; repeat up to max_steps: nxt = B acc, stop before nxt == 0, acc = nxt
 * (sparselin.py:430-434); *taken = applications kept */
int f4b_op_power_until_zero(f4b_op* op, const uint64_t* v, int64_t max_steps, uint64_t* out,
                            int64_t* taken);

#ifdef __cplusplus
}
#endif
#endif /* F4B200_H */
