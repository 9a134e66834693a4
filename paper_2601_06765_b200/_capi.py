"""ctypes binding of ``libf4b200.so`` (C ABI in ``include/f4b200.h``).

Device memory comes from the library's own stream-ordered pool (a
``cudaMemPool`` per context; ``F4B_TORCH_ALLOC=1`` registers an allocator
callback that hands out ``torch.empty(..., dtype=uint8)`` blocks from the
PyTorch caching allocator instead), and kernels run on
``torch.cuda.current_stream()``.  There is no CPU fallback: without the
built library or without a CUDA device every engine call raises
``DeviceError``.
"""

from __future__ import annotations

import ctypes as C
import os
import threading

import numpy as np

from .errors import DeviceError, raise_for_code

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.path.join(_HERE, "libf4b200.so")

_lib = None
_lock = threading.Lock()

ALLOC_FN = C.CFUNCTYPE(C.c_void_p, C.c_size_t, C.c_void_p)
FREE_FN = C.CFUNCTYPE(None, C.c_void_p, C.c_void_p)

i64p = C.POINTER(C.c_int64)
u64p = C.POINTER(C.c_uint64)
i32p = C.POINTER(C.c_int32)
u32p = C.POINTER(C.c_uint32)
u16p = C.POINTER(C.c_uint16)


class PlanInfo(C.Structure):
    _fields_ = [(k, C.c_int64) for k in (
        "r", "N", "M", "closure_rounds", "n_closure_rows", "key_words", "lane_bits",
        "dict_build_ns", "row_assemble_ns", "sort_passes", "kernel_launches", "row_lo", "r_total", "validated")]


class EchelonInfo(C.Structure):
    _fields_ = [(k, C.c_int64) for k in (
        "n_rows", "n_cols", "rank", "zero_rows", "n_pivot_rows", "n_nonpivot_rows",
        "pivot_nnz", "nonpivot_nnz", "full", "numeric_ns", "backsub_ns", "dense_rows", "dense_cols",
        "sweep_pivots", "sweep_tail_nnz")]


# name -> (restype, argtypes)
SIGNATURES = {
    "f4b_abi_version": (C.c_int, []),
    "f4b_ctx_create": (C.c_int, [C.c_int, C.c_uint32, C.c_int, C.c_int, ALLOC_FN, FREE_FN, C.c_void_p,
                                 C.POINTER(C.c_void_p)]),
    "f4b_ctx_destroy": (C.c_int, [C.c_void_p]),
    "f4b_ctx_set_stream": (C.c_int, [C.c_void_p, C.c_void_p]),
    "f4b_ctx_last_error": (C.c_char_p, [C.c_void_p]),
    "f4b_ctx_set_option": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64]),
    "f4b_ctx_profile": (C.c_int, [C.c_void_p, C.c_int]),
    "f4b_ctx_profile_read": (C.c_int, [C.c_void_p, C.c_char_p, C.c_int64, i64p]),
    "f4b_basis_clear": (C.c_int, [C.c_void_p]),
    "f4b_basis_append": (C.c_int, [C.c_void_p, C.c_int64, i64p, u16p, u32p]),
    "f4b_basis_append_wide": (C.c_int, [C.c_void_p, C.c_int64, i64p, i64p, u64p]),
    "f4b_basis_append_wide_async": (C.c_int, [C.c_void_p, C.c_int64, i64p, i64p, u64p]),
    "f4b_basis_append_keys_async": (C.c_int, [C.c_void_p, C.c_int64, i64p, u64p, C.c_int, u64p]),
    "f4b_basis_sync": (C.c_int, [C.c_void_p]),
    "f4b_bm": (C.c_int, [C.c_void_p, u64p, C.c_int64, C.c_int64, u64p, i64p]),
    "f4b_basis_size": (C.c_int, [C.c_void_p, i64p, i64p]),
    "f4b_compile_batch": (C.c_int, [C.c_void_p, C.c_int64, i32p, u16p, C.c_int, i32p, C.c_int64, C.c_int64,
                                    C.POINTER(C.c_void_p)]),
    "f4b_plan_get_info": (C.c_int, [C.c_void_p, C.POINTER(PlanInfo)]),
    "f4b_shard_begin": (C.c_int, [C.c_void_p, C.c_int64, i32p, u16p, C.c_int, i32p, C.c_int64, C.c_int64,
                                  C.c_int64, C.c_int64, C.POINTER(C.c_void_p), i64p]),
    "f4b_shard_take_run": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64]),
    "f4b_shard_merge": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, i64p]),
    "f4b_shard_round": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.c_void_p, i64p]),
    "f4b_shard_round_merge": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, i64p]),
    "f4b_shard_rows": (C.c_int, [C.c_void_p, i64p, C.c_void_p]),
    "f4b_shard_finish": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, C.POINTER(C.c_void_p)]),
    "f4b_shard_info": (C.c_int, [C.c_void_p, i64p, i64p, i64p]),
    "f4b_shard_free": (C.c_int, [C.c_void_p]),
    "f4b_plan_download": (C.c_int, [C.c_void_p, i64p, i64p, u64p, u16p, i32p, u16p, i32p]),
    "f4b_plan_download_ref_keys": (C.c_int, [C.c_void_p, u64p]),
    "f4b_plan_text": (C.c_int, [C.c_void_p, C.c_int, C.c_void_p, C.c_int64, i64p]),
    "f4b_plan_validate": (C.c_int, [C.c_void_p, i64p]),
    "f4b_plan_prefetch": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int]),
    "f4b_plan_wait": (C.c_int, [C.c_void_p]),
    "f4b_plan_poke": (C.c_int, [C.c_void_p, C.c_int, C.c_int64, C.c_uint32]),
    "f4b_csr_transpose": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, i64p, i64p, u64p, i64p, i64p, u64p]),
    "f4b_plan_left_apply": (C.c_int, [C.c_void_p, u64p, C.c_int64, u64p]),
    "f4b_op_create": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, i64p, i64p, u64p, C.c_int, C.POINTER(C.c_void_p)]),
    "f4b_op_free": (C.c_int, [C.c_void_p]),
    "f4b_op_apply": (C.c_int, [C.c_void_p, u64p, C.c_int64, u64p]),
    "f4b_op_krylov": (C.c_int, [C.c_void_p, u64p, u64p, C.c_int64, C.c_int64, u64p]),
    "f4b_op_horner": (C.c_int, [C.c_void_p, u64p, C.c_int64, u64p, u64p]),
    "f4b_op_power_until_zero": (C.c_int, [C.c_void_p, u64p, C.c_int64, u64p, i64p]),
    "f4b_plan_free": (C.c_int, [C.c_void_p]),
    "f4b_psge_plan": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int, C.POINTER(C.c_void_p)]),
    "f4b_psge_csr": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, i64p, i64p, u64p, C.c_int,
                               C.POINTER(C.c_void_p)]),
    "f4b_echelon_complete": (C.c_int, [C.c_void_p, C.c_void_p]),
    "f4b_echelon_complete_rows": (C.c_int, [C.c_void_p, C.c_void_p, i64p, C.c_int64]),
    "f4b_echelon_get_info": (C.c_int, [C.c_void_p, C.POINTER(EchelonInfo)]),
    "f4b_echelon_download": (C.c_int, [C.c_void_p, C.c_int, i64p, i64p, i64p, u64p]),
    "f4b_echelon_pivot_cols": (C.c_int, [C.c_void_p, i64p]),
    "f4b_echelon_free": (C.c_int, [C.c_void_p]),
    "f4b_basis_append_echelon": (C.c_int, [C.c_void_p, C.c_void_p, C.c_void_p]),
    "f4b_spmm": (C.c_int, [C.c_void_p, C.c_int64, C.c_int64, i64p, i64p, u64p, u64p, C.c_int64, u64p]),
    "f4b_dict_build": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_int, C.c_int, C.c_void_p, i64p]),
    "f4b_join_index": (C.c_int, [C.c_void_p, C.c_void_p, C.c_int64, C.c_void_p, C.c_int64, C.c_int, C.c_void_p]),
    "f4b_mod_fma": (C.c_int, [C.c_void_p, C.c_uint32, C.c_void_p, C.c_void_p, C.c_void_p, C.c_int64,
                              C.c_void_p]),
}


def load_library(path: str = LIB_PATH):
    """Load and type the shared library (no GPU needed just to load)."""
    global _lib
    with _lock:
        if _lib is not None:
            return _lib
        if not os.path.exists(path):
            raise DeviceError(f"{path} is missing: build it with __graft_entry__.build() "
                              "(there is no CPU fallback)")
        lib = C.CDLL(path)
        for name, (res, args) in SIGNATURES.items():
            fn = getattr(lib, name)
            fn.restype = res
            fn.argtypes = args
        _lib = lib
        return lib


def ptr(a: np.ndarray, ctype):
    return a.ctypes.data_as(C.POINTER(ctype)) if a is not None else None


class Context:
    """One C-ABI context = one (device, p, n_vars, order)."""

    def __init__(self, p: int, n_vars: int, order_code: int, device: int = 0):
        import torch

        if not torch.cuda.is_available():
            raise DeviceError("no CUDA device visible: the f4b200 engine has no CPU fallback")
        self.lib = load_library()
        self.device = device
        self.torch = torch
        self._blocks = {}
        dev = torch.device("cuda", device)

        def _alloc(nbytes, _user):
            try:
                t = torch.empty(int(nbytes), dtype=torch.uint8, device=dev)
            except RuntimeError:
                return None
            p_ = t.data_ptr()
            self._blocks[p_] = t
            return p_

        def _free(p_, _user):
            self._blocks.pop(p_, None)

        # Default: the library's own stream-ordered memory pool (no host
        # callback per device buffer).  F4B_TORCH_ALLOC=1 routes every device
        # buffer through the PyTorch caching allocator instead.
        if os.environ.get("F4B_TORCH_ALLOC"):
            self._alloc_cb = ALLOC_FN(_alloc)
            self._free_cb = FREE_FN(_free)
        else:
            self._alloc_cb = ALLOC_FN()
            self._free_cb = FREE_FN()
        h = C.c_void_p()
        with torch.cuda.device(dev):
            code = self.lib.f4b_ctx_create(device, p, n_vars, order_code, self._alloc_cb, self._free_cb, None,
                                           C.byref(h))
        if code:
            raise_for_code(code, "f4b_ctx_create failed")
        self.h = h
        self.sync_stream()

    def sync_stream(self):
        s = self.torch.cuda.current_stream(self.device).cuda_stream
        self.lib.f4b_ctx_set_stream(self.h, C.c_void_p(s))

    def check(self, code: int, what: str):
        if code:
            msg = self.lib.f4b_ctx_last_error(self.h)
            raise_for_code(code, f"{what}: {msg.decode() if msg else ''}")

    def close(self):
        if getattr(self, "h", None):
            self.lib.f4b_ctx_destroy(self.h)
            self.h = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass
