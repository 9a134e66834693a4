"""Device engine: one C-ABI context per (device, ring), the device-resident
basis, and handles for device plans / echelon forms.

The basis lives in HBM across F4 steps (SURVEY.md §1 "Boundaries in the
build"): ``sync_basis`` appends only the polynomials the device has not seen
(the F4 driver appends harvested rows directly), replacing the reference's
full ``soa_pack`` every step (``groebner.py:143-146``).
"""

from __future__ import annotations

import ctypes as C
import itertools
import weakref

import numpy as np

from . import _capi
from ._capi import EchelonInfo, PlanInfo, ptr
from .errors import LaneOverflowError
from .monomials import ORDER_CODE

_EXP_MAX = 0xFFFF
_PINNED_MIN = 1 << 16


def host_empty(shape, dtype):
    """Host array for a device download: page-locked (torch's caching host
    allocator) above 64 KiB so the copy runs at full PCIe / C2C rate."""
    dtype = np.dtype(dtype)
    count = int(np.prod(shape)) if np.ndim(shape) else int(shape)
    nbytes = count * dtype.itemsize
    if nbytes < _PINNED_MIN:
        return np.empty(shape, dtype=dtype)
    import torch

    t = torch.empty(nbytes, dtype=torch.uint8, pin_memory=True)
    return t.numpy().view(dtype).reshape(shape)
_ids = itertools.count(1)


def _current_device() -> int:
    import torch

    return torch.cuda.current_device() if torch.cuda.is_available() else 0


def _free_plan(free_fn, handle, keep):
    free_fn(handle)  # waits for a pending prefetch before the host block in `keep` is released


class DevicePlan:
    """Handle of an ``f4b_plan`` (device CSR + dictionary + closure rows)."""

    def __init__(self, engine, handle):
        self.engine = engine
        self.h = handle
        info = PlanInfo()
        engine.ctx.check(engine.lib.f4b_plan_get_info(handle, C.byref(info)), "plan info")
        self.info = {k: int(getattr(info, k)) for k, _ in PlanInfo._fields_}
        self._fin = weakref.finalize(self, engine.lib.f4b_plan_free, handle)

    def left_apply(self, V):
        """Aᵀ V over the device plan (V: r x b) -> N x b."""
        V = np.ascontiguousarray(V, dtype=np.uint64)
        vec = V.ndim == 1
        V2 = V.reshape(self.info["r"], -1)
        Y = np.empty((self.info["N"], V2.shape[1]), dtype=np.uint64)
        self.engine.ctx.check(self.engine.lib.f4b_plan_left_apply(self.h, ptr(V2, C.c_uint64), V2.shape[1],
                                                                   ptr(Y, C.c_uint64)), "plan left apply")
        return Y[:, 0] if vec else Y

    def download_ref_keys(self, n_key_words):
        """LayoutPlan.dict_keys built on the device (reference key format)."""
        out = host_empty((self.info["N"], n_key_words), np.uint64)
        if self.info["N"]:
            self.engine.ctx.check(self.engine.lib.f4b_plan_download_ref_keys(self.h, ptr(out, C.c_uint64)),
                                  "plan keys")
        return out

    def prefetch(self, n_key_words):
        """Start the host download of (row_ptr, col_ind, val) and the
        reference dictionary keys on the copy stream (f4b_plan_prefetch: one
        kernel, one D2H into one page-locked block); ``prefetched()`` waits
        and returns the views."""
        e = self.engine
        r, M, N = self.info["r"], self.info["M"], self.info["N"]
        blk = host_empty(r + 1 + 2 * M + N * n_key_words, np.int64)
        e.ctx.check(e.lib.f4b_plan_prefetch(self.h, blk.ctypes.data, int(n_key_words)), "plan prefetch")
        self._pf = (blk, n_key_words)
        # the host block must outlive any pending copy: the finalizer (which
        # frees the plan, waiting for the copy) keeps it alive
        self._fin.detach()
        self._fin = weakref.finalize(self, _free_plan, e.lib.f4b_plan_free, self.h, blk)

    def prefetched(self):
        if getattr(self, "_pf", None) is None:
            return None
        self.engine.ctx.check(self.engine.lib.f4b_plan_wait(self.h), "plan wait")
        blk, W = self._pf
        r, M, N = self.info["r"], self.info["M"], self.info["N"]
        o = r + 1 + 2 * M
        return {"row_ptr": blk[:r + 1], "col_ind": blk[r + 1:r + 1 + M], "val": blk[r + 1 + M:o].view(np.uint64),
                "dict_keys": blk[o:o + N * W].view(np.uint64).reshape(N, W)}

    def validate(self):
        """LayoutPlan.validate (reference symbolic.py:125-163) on the device
        buffers (f4b_plan_validate); PropertyViolationError on failure."""
        self.engine.ctx.check(self.engine.lib.f4b_plan_validate(self.h, None), "validate")

    def poke(self, which: str, index: int, value: int):
        """Fault injection for tests: overwrite one device entry."""
        code = {"row_ptr": 0, "col_ind": 1, "val": 2}[which]
        self.engine.ctx.check(self.engine.lib.f4b_plan_poke(self.h, code, index, value), "poke")

    _TEXT = {"row_ptr": 0, "col_ind": 1, "val": 2, "dict_keys": 3}

    def text(self, which: str) -> bytes:
        """One number list of plan_to_text (reference symbolic.py:438-460)
        formatted on the device (decimal, space separated)."""
        e = self.engine
        n = C.c_int64()
        code = self._TEXT[which]
        e.ctx.check(e.lib.f4b_plan_text(self.h, code, None, 0, C.byref(n)), "plan text")
        buf = C.create_string_buffer(max(n.value, 1))
        e.ctx.check(e.lib.f4b_plan_text(self.h, code, buf, n.value, C.byref(n)), "plan text")
        return buf.raw[: n.value]

    def download(self, arrays=True, dict_exps=True, closure=True):
        e, n = self.engine, self.engine.n_vars
        r, M, N, ncl = (self.info[k] for k in ("r", "M", "N", "n_closure_rows"))
        out = {}
        if arrays:
            # one page-locked block, three views: the library copies it in one go
            blk = host_empty(r + 1 + 2 * M, np.int64)
            out["row_ptr"] = blk[:r + 1]
            out["col_ind"] = blk[r + 1:r + 1 + M]
            out["val"] = blk[r + 1 + M:].view(np.uint64)
        if dict_exps:
            out["dict_exps"] = np.empty((N, n), dtype=np.uint16)
        if closure:
            out["cl_basis"] = np.empty(ncl, dtype=np.int32)
            out["cl_shift"] = np.empty((ncl, n), dtype=np.uint16)
            out["cl_round"] = np.empty(ncl, dtype=np.int32)
        g = out.get
        e.ctx.check(e.lib.f4b_plan_download(
            self.h, ptr(g("row_ptr"), C.c_int64), ptr(g("col_ind"), C.c_int64), ptr(g("val"), C.c_uint64),
            ptr(g("dict_exps"), C.c_uint16), ptr(g("cl_basis"), C.c_int32), ptr(g("cl_shift"), C.c_uint16),
            ptr(g("cl_round"), C.c_int32)), "plan download")
        return out


class DeviceOperator:
    """Handle of an ``f4b_op``: the CSR stays in HBM across applications."""

    def __init__(self, engine, handle, dim):
        self.engine = engine
        self.h = handle
        self.dim = dim
        self._fin = weakref.finalize(self, engine.lib.f4b_op_free, handle)

    def _chk(self, code, what):
        self.engine.ctx.check(code, what)

    def apply(self, X):
        X = np.ascontiguousarray(X, dtype=np.uint64)
        vec = X.ndim == 1
        X2 = X.reshape(self.dim, -1)
        Y = np.empty_like(X2)
        self._chk(self.engine.lib.f4b_op_apply(self.h, ptr(X2, C.c_uint64), X2.shape[1], ptr(Y, C.c_uint64)),
                  "operator apply")
        return Y[:, 0] if vec else Y

    def krylov(self, U, V, steps):
        U = np.ascontiguousarray(U, dtype=np.uint64)
        V = np.ascontiguousarray(V, dtype=np.uint64)
        b = V.shape[1]
        seqs = np.empty((steps, b), dtype=np.uint64)
        self._chk(self.engine.lib.f4b_op_krylov(self.h, ptr(U, C.c_uint64), ptr(V, C.c_uint64), b, int(steps),
                                                ptr(seqs, C.c_uint64)), "operator krylov")
        return seqs

    def horner(self, g, v):
        g = np.ascontiguousarray(g, dtype=np.uint64)
        v = np.ascontiguousarray(v, dtype=np.uint64).reshape(-1)
        out = np.empty(self.dim, dtype=np.uint64)
        self._chk(self.engine.lib.f4b_op_horner(self.h, ptr(g, C.c_uint64), len(g), ptr(v, C.c_uint64),
                                                ptr(out, C.c_uint64)), "operator horner")
        return out

    def power_until_zero(self, v, max_steps):
        v = np.ascontiguousarray(v, dtype=np.uint64).reshape(-1)
        out = np.empty(self.dim, dtype=np.uint64)
        taken = np.zeros(1, dtype=np.int64)
        self._chk(self.engine.lib.f4b_op_power_until_zero(self.h, ptr(v, C.c_uint64), int(max_steps),
                                                          ptr(out, C.c_uint64), ptr(taken, C.c_int64)),
                  "operator power")
        return out, int(taken[0])


class DeviceEchelon:
    """Handle of an ``f4b_echelon``; pivot rows are computed on demand."""

    def __init__(self, engine, handle, keepalive=None):
        self.engine = engine
        self.h = handle
        self._keep = keepalive  # the plan whose CSR the echelon reads
        self._fin = weakref.finalize(self, engine.lib.f4b_echelon_free, handle)

    def info(self):
        inf = EchelonInfo()
        self.engine.lib.f4b_echelon_get_info(self.h, C.byref(inf))
        return {k: int(getattr(inf, k)) for k, _ in EchelonInfo._fields_}

    def complete(self):
        self.engine.ctx.sync_stream()
        self.engine.ctx.check(self.engine.lib.f4b_echelon_complete(self.engine.ctx.h, self.h), "echelon complete")

    def complete_rows(self, lead_cols):
        """Back-reduce only the pivot rows led by ``lead_cols``
        (f4b_echelon_complete_rows); the other pivot rows stay empty."""
        lc = np.ascontiguousarray(lead_cols, dtype=np.int64)
        self.engine.ctx.sync_stream()
        self.engine.ctx.check(self.engine.lib.f4b_echelon_complete_rows(self.engine.ctx.h, self.h, ptr(lc, C.c_int64),
                                                                        len(lc)), "echelon complete rows")

    def pivot_cols(self):
        inf = self.info()
        out = np.empty(inf["rank"], dtype=np.int64)
        self.engine.ctx.check(self.engine.lib.f4b_echelon_pivot_cols(self.h, ptr(out, C.c_int64)), "pivot cols")
        return out

    def rows(self, which: int):
        """Return (leads, row_ptr, cols, vals) for pivot (0) or nonpivot (1) rows."""
        inf = self.info()
        if which == 0 and not inf["full"]:
            self.complete()
            inf = self.info()
        n = inf["n_pivot_rows"] if which == 0 else inf["n_nonpivot_rows"]
        nnz = inf["pivot_nnz"] if which == 0 else inf["nonpivot_nnz"]
        leads = np.empty(n, dtype=np.int64)
        rp = np.empty(n + 1, dtype=np.int64)
        cols = np.empty(max(nnz, 1), dtype=np.int64)
        vals = np.empty(max(nnz, 1), dtype=np.uint64)
        self.engine.ctx.check(self.engine.lib.f4b_echelon_download(
            self.h, which, ptr(leads, C.c_int64), ptr(rp, C.c_int64), ptr(cols, C.c_int64),
            ptr(vals, C.c_uint64)), "echelon download")
        return leads, rp, cols[:nnz], vals[:nnz]


class Engine:
    """Device engine for one ring on one GPU."""

    _registry: dict = {}
    _forced: dict = {}  # f4b_ctx_set_option settings applied to every engine

    @classmethod
    def force_option(cls, name: str, value: int):
        """Apply a path-selection option (see set_option) to every engine,
        existing and future; value 0 restores the automatic choice."""
        if value:
            cls._forced[name] = int(value)
        else:
            cls._forced.pop(name, None)
        for eng in cls._registry.values():
            eng.set_option(name, value)

    @classmethod
    def for_ring(cls, ring, device: int | None = None) -> "Engine":
        """The engine of ``ring`` on ``device`` (default: the current CUDA
        device, so one process per GPU under torchrun uses its own GPU)."""
        if device is None:
            device = _current_device()
        key = (device, ring.modulus.p, ring.n_vars, ring.order)
        eng = cls._registry.get(key)
        if eng is None:
            eng = cls(ring.modulus.p, ring.n_vars, ring.order, device)
            cls._registry[key] = eng
        return eng

    def __init__(self, p, n_vars, order, device=0):
        self.ctx = _capi.Context(p, n_vars, ORDER_CODE[order], device)
        self.lib = self.ctx.lib
        self.p, self.n_vars, self.order, self.device = p, n_vars, order, device
        self.uid = next(_ids)
        self.generation = 0
        self._reset_mirror()
        for name, value in self._forced.items():
            self.set_option(name, value)

    def _reset_mirror(self):
        # host mirror of the device basis: lengths + the appended chunks (no
        # concatenation, so appends stay O(new terms)), and the buffers of the
        # last synced SoaPolySet for the append-only fast path of sync_basis
        self._lens = np.zeros(0, dtype=np.int64)
        self._chunks = []  # (t0, exps u16 chunk, coeff u32 chunk)
        self._T = 0
        self._src = None
        self._src_refs = None

    # -- path selection (f4b_ctx_set_option) ---------------------------------
    def set_option(self, name: str, value: int):
        """Force a fallback path ("sweep", "dense", "fbsp", "dict_sort",
        "dict_lsd"; 0 = the automatic choice).  Every setting computes the
        same bytes; the tests use this to reach every kernel."""
        self.ctx.check(self.lib.f4b_ctx_set_option(self.ctx.h, name.encode(), int(value)), f"set_option {name}")

    # -- instrumentation -----------------------------------------------------
    def profile(self, enable: bool):
        """Bracket every kernel launch with CUDA events (f4b_ctx_profile)."""
        self.ctx.check(self.lib.f4b_ctx_profile(self.ctx.h, 1 if enable else 0), "profile")

    def profile_read(self):
        """-> ({kernel: (launches, total_ns)}, total launches since context creation)."""
        buf = C.create_string_buffer(1 << 16)
        tot = np.zeros(1, dtype=np.int64)
        self.ctx.check(self.lib.f4b_ctx_profile_read(self.ctx.h, buf, len(buf), ptr(tot, C.c_int64)), "profile read")
        out = {}
        for line in buf.value.decode().splitlines():
            name, cnt, ns = line.rsplit(" ", 2)
            out[name] = (int(cnt), float(ns))
        return out, int(tot[0])

    # -- basis -------------------------------------------------------------
    @property
    def token(self):
        return (self.uid, self.generation)

    @property
    def n_polys(self) -> int:
        return len(self._lens)

    def basis_lengths(self) -> np.ndarray:
        """Term counts of the device basis polynomials (host mirror)."""
        return self._lens

    def clear_basis(self):
        self.ctx.check(self.lib.f4b_basis_clear(self.ctx.h), "basis clear")
        self._reset_mirror()
        self.generation += 1

    def append_polys(self, lengths, exps, coeffs, defer: bool = False, keys=None):
        """Append polynomials to the device basis.  With ``defer`` (the
        reference-format int64 / uint64 streams only) the call returns without
        waiting for the device; range errors then surface from the next
        compile (the caller keeps ``exps`` / ``coeffs`` alive until then).
        ``keys`` (with ``defer``): the SoaPolySet's reference keys of the same
        terms, uploaded instead of the exponent rows (8 W instead of 8 n bytes
        per term; the device unpacks the lanes)."""
        lengths = np.ascontiguousarray(lengths, dtype=np.int64)
        exps = np.asarray(exps)
        coeffs = np.asarray(coeffs)
        W = ((32 if self.order != "lex" else 0) + 16 * self.n_vars + 63) // 64  # reference key words (monomials.Ring)
        if (defer and keys is not None and keys.dtype == np.uint64 and keys.ndim == 2 and keys.shape[1] == W
                and keys.flags.c_contiguous and coeffs.dtype == np.uint64 and coeffs.flags.c_contiguous
                and W < self.n_vars):
            self.ctx.sync_stream()
            self.ctx.check(self.lib.f4b_basis_append_keys_async(self.ctx.h, len(lengths), ptr(lengths, C.c_int64),
                                                                ptr(keys, C.c_uint64), W, ptr(coeffs, C.c_uint64)),
                           "basis append")
            self._deferred = (lengths, keys, coeffs)  # host buffers read by the pending copy
            self._lens = np.concatenate([self._lens, lengths])
            if len(coeffs):
                self._chunks.append((self._T, exps, coeffs))
            self._T += len(coeffs)
            self._src = None
            self.generation += 1
            return
        if (exps.dtype == np.int64 and coeffs.dtype == np.uint64 and exps.ndim == 2
                and exps.flags.c_contiguous and coeffs.flags.c_contiguous):
            # the reference's SoaPolySet streams as they are: narrowing, range
            # checks and per-polynomial metadata on the device
            self.ctx.sync_stream()
            fn = self.lib.f4b_basis_append_wide_async if defer else self.lib.f4b_basis_append_wide
            self.ctx.check(fn(self.ctx.h, len(lengths), ptr(lengths, C.c_int64), ptr(exps, C.c_int64),
                              ptr(coeffs, C.c_uint64)), "basis append")
            if defer:
                self._deferred = (lengths, exps, coeffs)  # host buffers read by the pending copy
            self._lens = np.concatenate([self._lens, lengths])
            if len(coeffs):
                self._chunks.append((self._T, exps, coeffs))
            self._T += len(coeffs)
            self._src = None
            self.generation += 1
            return
        if exps.size and (exps.min() < 0 or exps.max() > _EXP_MAX):
            raise LaneOverflowError("exponent does not fit a 16-bit lane")
        exps = np.ascontiguousarray(exps, dtype=np.uint16).reshape(-1, self.n_vars)
        coeffs = np.ascontiguousarray(coeffs, dtype=np.uint32)
        self.ctx.sync_stream()
        self.ctx.check(self.lib.f4b_basis_append(self.ctx.h, len(lengths), ptr(lengths, C.c_int64),
                                                 ptr(exps, C.c_uint16), ptr(coeffs, C.c_uint32)), "basis append")
        self._lens = np.concatenate([self._lens, lengths])
        if len(coeffs):
            self._chunks.append((self._T, exps, coeffs))
        self._T += len(coeffs)
        self._src = None
        self.generation += 1

    def append_from_echelon(self, plan: DevicePlan, ech: DeviceEchelon, lengths, exps, coeffs):
        """The F4 harvest on the device (f4b_basis_append_echelon): the
        echelon's nonpivot rows appended to the device basis straight from
        the plan dictionary and the echelon pool (device to device).  The
        host arrays (the same polynomials, which the driver already holds)
        only extend the prefix-check mirror; nothing is uploaded."""
        self.ctx.sync_stream()
        self.ctx.check(self.lib.f4b_basis_append_echelon(self.ctx.h, plan.h, ech.h), "basis append (echelon)")
        lengths = np.ascontiguousarray(lengths, dtype=np.int64)
        self._lens = np.concatenate([self._lens, lengths])
        if len(coeffs):
            self._chunks.append((self._T, np.asarray(exps), np.asarray(coeffs)))
        self._T += len(coeffs)
        self._src = None
        self.generation += 1

    @staticmethod
    def _buffers(soa):
        # (address, strides) of the streams; the arrays themselves are kept in
        # self._src_refs so the addresses cannot be recycled by another array
        return tuple((a.__array_interface__["data"][0], a.strides) for a in (soa.exps, soa.coeff))

    def _prefix_equal(self, soa) -> bool:
        n_dev, T_dev = self.n_polys, self._T
        if len(soa) < n_dev or soa.total_terms() < T_dev:
            return False
        if not np.array_equal(soa.length[:n_dev], self._lens):
            return False
        if self._src is not None and self._src == self._buffers(soa):
            # same append-only buffers as the last sync (the F4 driver's
            # growing SoaPolySet): the synced prefix cannot have changed
            return True
        for t0, ex, co in self._chunks:
            t1 = t0 + len(co)
            if not (np.array_equal(soa.coeff[t0:t1], co) and np.array_equal(soa.exps[t0:t1], ex)):
                return False
        return True

    def sync_basis(self, soa):
        """Make the device basis equal to ``soa`` (a SoaPolySet).  Appends
        only the polynomials beyond the device prefix when that prefix is
        unchanged (SoaPolySet streams are append-only, as in the reference)."""
        if getattr(soa, "_f4b_token", None) == self.token:
            return
        if not self._prefix_equal(soa):
            self.clear_basis()
        n_dev, T_dev = self.n_polys, self._T
        if len(soa) > n_dev:
            self.append_polys(soa.length[n_dev:], soa.exps[T_dev:], soa.coeff[T_dev:], defer=True,
                              keys=soa.mon_key[T_dev:])
        self._src = self._buffers(soa)
        self._src_refs = (soa.exps, soa.coeff)
        soa._f4b_token = self.token

    # -- hot path ----------------------------------------------------------
    def compile(self, row_basis, row_shift, closure: bool, candidates=None, dict_cap=10**6) -> DevicePlan:
        rb = np.ascontiguousarray(row_basis, dtype=np.int32)
        sh = np.asarray(row_shift)
        if sh.size and (sh.min() < 0 or sh.max() > _EXP_MAX):
            raise LaneOverflowError("shift exponent does not fit a 16-bit lane")
        sh = np.ascontiguousarray(sh, dtype=np.uint16).reshape(len(rb), self.n_vars)
        cand = None if candidates is None else np.ascontiguousarray(candidates, dtype=np.int32)
        self.ctx.sync_stream()
        h = C.c_void_p()
        code = self.lib.f4b_compile_batch(
            self.ctx.h, len(rb), ptr(rb, C.c_int32), ptr(sh, C.c_uint16), 1 if closure else 0,
            ptr(cand, C.c_int32) if cand is not None else None, 0 if cand is None else len(cand),
            int(dict_cap), C.byref(h))
        self._deferred = None
        if code:
            # a failed compile may also carry the error of a deferred append:
            # forget the device basis mirror so the next sync re-uploads it
            self.clear_basis()
        self.ctx.check(code, "compile_batch")
        return DevicePlan(self, h)

    def psge_plan(self, plan: DevicePlan, full: bool) -> DeviceEchelon:
        self.ctx.sync_stream()
        h = C.c_void_p()
        self.ctx.check(self.lib.f4b_psge_plan(self.ctx.h, plan.h, 1 if full else 0, C.byref(h)), "psge")
        return DeviceEchelon(self, h, keepalive=plan)

    def csr_transpose(self, n_rows, n_cols, row_ptr, col_ind, val):
        """Stable transpose on the device (f4b_csr_transpose) -> (row_ptr,
        col_ind, val) of the n_cols x n_rows matrix."""
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_ind, dtype=np.int64)
        va = np.ascontiguousarray(val, dtype=np.uint64)
        nnz = int(rp[n_rows]) if len(rp) else 0
        trp = np.empty(n_cols + 1, dtype=np.int64)
        tci = np.empty(max(nnz, 1), dtype=np.int64)
        tva = np.empty(max(nnz, 1), dtype=np.uint64)
        self.ctx.sync_stream()
        self.ctx.check(self.lib.f4b_csr_transpose(self.ctx.h, n_rows, n_cols, ptr(rp, C.c_int64), ptr(ci, C.c_int64),
                                                  ptr(va, C.c_uint64), ptr(trp, C.c_int64), ptr(tci, C.c_int64),
                                                  ptr(tva, C.c_uint64)), "csr transpose")
        return trp, tci[:nnz], tva[:nnz]

    def psge_csr(self, n_rows, n_cols, row_ptr, col_ind, val, full: bool) -> DeviceEchelon:
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_ind, dtype=np.int64)
        va = np.ascontiguousarray(val, dtype=np.uint64)
        self.ctx.sync_stream()
        h = C.c_void_p()
        self.ctx.check(self.lib.f4b_psge_csr(self.ctx.h, int(n_rows), int(n_cols), ptr(rp, C.c_int64),
                                             ptr(ci, C.c_int64), ptr(va, C.c_uint64), 1 if full else 0,
                                             C.byref(h)), "psge")
        return DeviceEchelon(self, h)

    def operator(self, n_rows, n_cols, row_ptr, col_ind, val, normal: bool) -> "DeviceOperator":
        """Resident black-box operator B = A (square) or AᵀA (normal) for Wiedemann."""
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_ind, dtype=np.int64)
        va = np.ascontiguousarray(val, dtype=np.uint64)
        h = C.c_void_p()
        self.ctx.sync_stream()
        self.ctx.check(self.lib.f4b_op_create(self.ctx.h, int(n_rows), int(n_cols), ptr(rp, C.c_int64),
                                              ptr(ci, C.c_int64), ptr(va, C.c_uint64), 1 if normal else 0,
                                              C.byref(h)), "operator")
        return DeviceOperator(self, h, int(n_cols))

    def bm(self, seqs):
        """Berlekamp–Massey of the columns of ``seqs`` ([len][b]) on the
        device; returns one ascending monic minimal polynomial per column."""
        S = np.ascontiguousarray(np.asarray(seqs, dtype=np.uint64).T)  # [b][len]
        b, n = S.shape
        polys = np.zeros((b, n + 1), dtype=np.uint64)
        degs = np.zeros(b, dtype=np.int64)
        self.ctx.sync_stream()
        self.ctx.check(self.lib.f4b_bm(self.ctx.h, ptr(S, C.c_uint64), int(n), int(b), ptr(polys, C.c_uint64),
                                       ptr(degs, C.c_int64)), "berlekamp_massey")
        return [[int(x) for x in polys[j, :degs[j] + 1]] for j in range(b)]

    def spmm(self, n_rows, n_cols, row_ptr, col_ind, val, X):
        X = np.ascontiguousarray(X, dtype=np.uint64)
        b = X.shape[1]
        Y = np.zeros((n_rows, b), dtype=np.uint64)
        rp = np.ascontiguousarray(row_ptr, dtype=np.int64)
        ci = np.ascontiguousarray(col_ind, dtype=np.int64)
        va = np.ascontiguousarray(val, dtype=np.uint64)
        self.ctx.sync_stream()
        self.ctx.check(self.lib.f4b_spmm(self.ctx.h, int(n_rows), int(n_cols), ptr(rp, C.c_int64),
                                         ptr(ci, C.c_int64), ptr(va, C.c_uint64), ptr(X, C.c_uint64), b,
                                         ptr(Y, C.c_uint64)), "spmm")
        return Y
