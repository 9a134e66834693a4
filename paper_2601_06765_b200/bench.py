"""Microbenchmarks of the three isolated primitives (reference
``src/bench.py:237-312`` ``_synth_keys`` / ``microbench``), run on the GPU.

Same signature, same synthetic inputs (the reference's NumPy generator and
seed), same correctness-before-timing rule and the reference's result keys;
timing is device time (CUDA events on the launching stream, median of
``reps`` launches, inputs resident in HBM), and each result adds the
algorithmic HBM bytes of one launch and the achieved fraction of the
measured copy bandwidth (``MEASURED_PEAKS.json``).

  dict_build    radix_sort + unique_sorted   -> f4b_dict_build  (micro.cu)
  row_assemble  merge_join_index             -> f4b_join_index
  mod_fma       KernelArith acc + a*b mod p  -> f4b_mod_fma

The checks compare against NumPy on the host (the reference checks against
Python sets / naive arithmetic); no result is produced on the CPU.
"""

from __future__ import annotations

import ctypes as C
import json
import os
import statistics

import numpy as np

from ._capi import Context, ptr
from .errors import PreconditionError

KEY_BITS = 48  # reference keys: uniform 48-bit words (bench.py:239)
_CTX = {}


def _synth_keys(rng, size: int, duplicate_rate: float, words: int = 2):
    """Reference bench.py:237-241, same draws."""
    n_unique = max(1, int(round(size * (1.0 - duplicate_rate))))
    pool = rng.integers(0, 1 << 48, (n_unique, words)).astype(np.uint64)
    picks = rng.integers(0, n_unique, size)
    return pool[picks]


def _host_unique(keys):
    """Ascending unique rows of a [n, W] u64 array (host check; lexsort is
    much faster than np.unique(axis=0) at 2^24 keys)."""
    order = np.lexsort(keys.T[::-1])
    s = keys[order]
    keep = np.ones(len(s), dtype=bool)
    keep[1:] = np.any(s[1:] != s[:-1], axis=1)
    return s[keep]


def _ctx(device: int) -> Context:
    c = _CTX.get(device)
    if c is None:
        c = _CTX[device] = Context(32003, 1, 0, device)
    return c


def hbm_peak_gbs() -> float:
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    try:
        with open(os.path.join(root, "MEASURED_PEAKS.json")) as fh:
            return float(json.load(fh)["hbm_gbs"])
    except Exception:
        return 6650.0  # B200_PROFILING.md fallback


def _time(torch, fn, reps: int) -> float:
    """Median device time (ns) of fn() over reps launches (CUDA events on the
    current stream, one synchronize on both sides of each)."""
    st = torch.cuda.current_stream()
    out = []
    for _ in range(reps):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(st)
        fn()
        b.record(st)
        torch.cuda.synchronize()
        out.append(a.elapsed_time(b) * 1e6)
    return statistics.median(out)


def _dev(torch, arr, device):
    return torch.from_numpy(np.ascontiguousarray(arr).view(np.int64)).to(f"cuda:{device}")


def _p(t):
    return C.c_void_p(t.data_ptr())


def dict_build(keys_dev, words: int = 2, key_bits: int = KEY_BITS, device: int = 0):
    """Ascending unique keys of a device tensor [n, words] (int64 view of u64)."""
    import torch

    c = _ctx(device)
    c.sync_stream()
    n = keys_dev.shape[0]
    out = torch.empty((max(n, 1), words), dtype=torch.int64, device=keys_dev.device)
    nu = np.zeros(1, dtype=np.int64)
    c.check(c.lib.f4b_dict_build(c.h, _p(keys_dev), n, words, key_bits, _p(out), ptr(nu, C.c_int64)), "dict_build")
    return out[:int(nu[0])]


def join_index(dict_dev, keys_dev, device: int = 0):
    """Position of each key (device [n, W]) in an ascending dictionary (device [N, W])."""
    import torch

    c = _ctx(device)
    c.sync_stream()
    pos = torch.empty(keys_dev.shape[0], dtype=torch.int64, device=keys_dev.device)
    c.check(c.lib.f4b_join_index(c.h, _p(dict_dev), dict_dev.shape[0], _p(keys_dev), keys_dev.shape[0],
                                 keys_dev.shape[1], _p(pos)), "join_index")
    return pos


def mod_fma(p: int, a_dev, b_dev, acc_dev, device: int = 0):
    import torch

    c = _ctx(device)
    c.sync_stream()
    out = torch.empty_like(a_dev)
    c.check(c.lib.f4b_mod_fma(c.h, p, _p(a_dev), _p(b_dev), _p(acc_dev), a_dev.numel(), _p(out)), "mod_fma")
    return out


def microbench(kind: str, size: int, duplicate_rate: float = 0.5, seed: int = 0, device: int = 0,
               reps: int = 5) -> dict:
    """Reference bench.py:244-312 on the GPU (see module docstring)."""
    import torch

    if size < 1:
        raise PreconditionError("size must be >= 1")
    _ctx(device)  # DeviceError without a GPU or the library: no CPU fallback
    rng = np.random.default_rng(seed)
    peak = hbm_peak_gbs()
    out = {"kind": kind, "size": size, "seed": seed, "device": "cuda"}
    if kind == "dict_build":
        keys = _synth_keys(rng, size, duplicate_rate)
        kd = _dev(torch, keys, device)
        uniq = dict_build(kd, device=device).cpu().numpy().view(np.uint64)
        want = _host_unique(keys)
        assert np.array_equal(uniq, want), "dict_build disagrees with the host unique"
        dt = _time(torch, lambda: dict_build(kd, device=device), reps)
        nbytes = keys.nbytes + uniq.nbytes  # read every key once, write the dictionary once
        passes = -(-2 * KEY_BITS // 8)
        # micro.cu: up to 2^24 + 2^22 keys take the MSD bucket path (read 4x:
        # top-bit scan, histogram, scatter, bucket sort; write the packed keys
        # once and the dictionary once); larger inputs the one-sweep LSD sort
        if size <= (1 << 24) + (1 << 22):
            path = "MSD buckets (one global scatter, sub-buckets sorted in shared memory)"
            streamed = 4 * keys.nbytes + keys.nbytes + uniq.nbytes
            passes = 1
        else:
            path = "LSD one-sweep sort of every key"
            streamed = keys.nbytes + 2 * (passes + 2) * keys.nbytes + uniq.nbytes
        out.update(
            duplicate_rate=duplicate_rate,
            unique_out=len(uniq),
            radix_passes=passes,
            reference_radix_passes=8 * keys.shape[1],
            keys_total=size,
            keys_per_s=size / max(dt, 1) * 1e9,
            bytes_per_s=keys.nbytes / max(dt, 1) * 1e9,
            elapsed_ns=dt,
            algorithmic_bytes=nbytes,
            hbm_frac=nbytes / max(dt, 1) / peak,
            dict_path=path,
            hbm_frac_streamed=streamed / max(dt, 1) / peak,
        )
    elif kind == "row_assemble":
        dic = _host_unique(_synth_keys(rng, size, 0.0))
        lens = np.clip(rng.geometric(0.2, max(1, size // 16)), 1, 64)
        picks = np.sort(rng.integers(0, len(dic), int(lens.sum())))
        seg = dic[picks]
        dd, sd = _dev(torch, dic, device), _dev(torch, seg, device)
        got = join_index(dd, sd, device=device).cpu().numpy()
        assert np.array_equal(dic[got], seg), "join_index disagrees"
        dt = _time(torch, lambda: join_index(dd, sd, device=device), reps)
        bucket_counts = np.bincount(np.minimum(lens, 64))
        busiest = int(bucket_counts.max())
        nbytes = seg.nbytes + 8 * len(seg) + dic.nbytes
        out.update(
            rows=len(lens),
            joins_total=len(seg),
            joins_per_s=len(seg) / max(dt, 1) * 1e9,
            bucket_imbalance=busiest / max(1.0, bucket_counts[bucket_counts > 0].mean()),
            elapsed_ns=dt,
            algorithmic_bytes=nbytes,
            hbm_frac=nbytes / max(dt, 1) / peak,
        )
    elif kind == "mod_fma":
        p = 2147483629
        a = rng.integers(0, p, size, dtype=np.uint64)
        b = rng.integers(0, p, size, dtype=np.uint64)
        acc = rng.integers(0, p, size, dtype=np.uint64)
        want = (acc + a * b) % np.uint64(p)
        ad, bd, cd = (_dev(torch, x, device) for x in (a, b, acc))
        got = mod_fma(p, ad, bd, cd, device=device).cpu().numpy().view(np.uint64)
        assert np.array_equal(got, want), "mod_fma disagrees with naive"
        dt = _time(torch, lambda: mod_fma(p, ad, bd, cd, device=device), reps)
        nbytes = 32 * size
        # one device kernel (Barrett); the reference's three backends agree bit for bit
        out["updates_per_s.barrett"] = size / max(dt, 1) * 1e9
        out["elapsed_ns.barrett"] = dt
        out.update(algorithmic_bytes=nbytes, hbm_frac=nbytes / max(dt, 1) / peak)
    else:
        raise PreconditionError(f"unknown microbench kind {kind!r}")
    return out
