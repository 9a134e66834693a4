"""Multi-rank plumbing for the hot path: one process per GPU,
``torch.distributed`` for the collectives (NCCL on GPUs, gloo for the CPU
tests).

What shards and how:

* the benchmark replay (bench.py ``--gpus N``): every rank replays the whole
  cyclic-8 run on its own GPU — replicas, weak scaling, no data-path
  collective; the step time is the max over ranks (``max_over_ranks``);
* FBSP on G ranks (§8e): the deterministic row list splits into contiguous
  ranges balanced by term counts (``balanced_ranges``); each rank builds the
  sorted unique key run of its range, the runs are all-gathered
  (``allgather_arrays``) and merged redundantly on every rank
  (``merge_key_runs``) into the identical global dictionary; concatenating
  the per-rank CSR slices in rank order reproduces the global CSR
  (``concat_csr``);
* Block Wiedemann on G ranks (§8e): the b block columns of each round are
  dealt round-robin (``shard_round_robin``); every rank runs its columns'
  Krylov sequences, Berlekamp-Massey and generator evaluations on its own
  resident operator, and only the candidate kernel vectors are all-gathered
  once per round (``sparselin._kernel_rounds``).

Everything here is compute-agnostic host logic; the per-rank compute is the
CUDA engine (``engine.Engine``) on that rank's device.
"""

from __future__ import annotations

import os
from dataclasses import dataclass

import numpy as np


@dataclass(frozen=True)
class RankInfo:
    rank: int
    world: int
    local_rank: int


def rank_info() -> RankInfo:
    """RANK / WORLD_SIZE / LOCAL_RANK as set by torch.distributed.run."""
    return RankInfo(int(os.environ.get("RANK", "0")), int(os.environ.get("WORLD_SIZE", "1")),
                    int(os.environ.get("LOCAL_RANK", "0")))


def active_world() -> tuple:
    """(rank, world) of the initialised default process group, else (0, 1)."""
    try:
        import torch.distributed as dist
    except ImportError:  # pragma: no cover
        return 0, 1
    if dist.is_available() and dist.is_initialized():
        return dist.get_rank(), dist.get_world_size()
    return 0, 1


def init(backend: str | None = None):
    """Initialise the default process group from the torchrun environment
    (127.0.0.1 rendezvous when MASTER_ADDR is unset).  Returns RankInfo."""
    import torch
    import torch.distributed as dist

    info = rank_info()
    if info.world > 1 and not dist.is_initialized():
        os.environ.setdefault("MASTER_ADDR", "127.0.0.1")
        os.environ.setdefault("MASTER_PORT", "29511")
        if backend is None:
            backend = "nccl" if torch.cuda.is_available() else "gloo"
        kw = {}
        if backend == "nccl":
            torch.cuda.set_device(info.local_rank)
            kw["device_id"] = torch.device("cuda", info.local_rank)
        dist.init_process_group(backend, rank=info.rank, world_size=info.world, **kw)
    return info


def _dev():
    import torch
    import torch.distributed as dist

    if dist.is_initialized() and dist.get_backend() == "nccl":
        return torch.device("cuda", torch.cuda.current_device())
    return torch.device("cpu")


def max_over_ranks(x: float) -> float:
    """Max of a scalar over all ranks (the step time of a multi-rank run)."""
    import torch
    import torch.distributed as dist

    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.MAX)
    return float(t.item())


def sum_over_ranks(x: float) -> float:
    import torch
    import torch.distributed as dist

    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return float(x)
    t = torch.tensor([float(x)], dtype=torch.float64, device=_dev())
    dist.all_reduce(t, op=dist.ReduceOp.SUM)
    return float(t.item())


def balanced_ranges(weights, world: int) -> list:
    """Contiguous [lo, hi) ranges of len(weights) items, one per rank, with
    near-equal weight sums (a scan of the weights; §8e row partition)."""
    w = np.asarray(weights, dtype=np.int64)
    n = len(w)
    if world <= 1 or n == 0:
        return [(0, n)] + [(n, n)] * max(0, world - 1)
    pre = np.concatenate([[0], np.cumsum(w)])
    total = pre[-1]
    cuts = [0]
    for k in range(1, world):
        cuts.append(int(np.searchsorted(pre, total * k / world, side="left")))
    cuts.append(n)
    cuts = np.maximum.accumulate(np.minimum(cuts, n))
    return [(int(cuts[k]), int(cuts[k + 1])) for k in range(world)]


def shard_round_robin(n_units: int, rank: int, world: int) -> list:
    """Independent units (e.g. replayed batches) dealt round-robin."""
    return list(range(rank, n_units, world))


def allgather_arrays(arr: np.ndarray) -> list:
    """All-gather variable-length 2-D arrays (same dtype / row width on every
    rank): sizes first, then one padded all_gather.  Returns the per-rank
    arrays in rank order."""
    import torch
    import torch.distributed as dist

    arr = np.ascontiguousarray(arr)
    if not (dist.is_initialized() and dist.get_world_size() > 1):
        return [arr]
    world = dist.get_world_size()
    dev = _dev()
    row_shape = arr.shape[1:]
    width = int(np.prod(row_shape, dtype=np.int64)) * arr.dtype.itemsize
    # (0, width) for an empty local array: reshape(0, -1) is ambiguous
    as_bytes = arr.view(np.uint8).reshape(len(arr), width) if len(arr) else np.zeros((0, width), np.uint8)
    n = torch.tensor([len(arr)], dtype=torch.int64, device=dev)
    sizes = [torch.zeros_like(n) for _ in range(world)]
    dist.all_gather(sizes, n)
    sizes = [int(s.item()) for s in sizes]
    cap = max(1, max(sizes))
    buf = torch.zeros((cap, max(width, 1)), dtype=torch.uint8, device=dev)
    if len(arr):
        buf[: len(arr), :width] = torch.from_numpy(as_bytes).to(dev)
    outs = [torch.zeros_like(buf) for _ in range(world)]
    dist.all_gather(outs, buf)
    res = []
    for s, o in zip(sizes, outs):
        b = o[:s, :width].cpu().numpy().copy()
        res.append(b.view(arr.dtype).reshape((s,) + row_shape))
    return res


def merge_key_runs(runs) -> np.ndarray:
    """Merge per-rank sorted unique runs of reference keys (rows of big-endian
    u64 words, DESCENDING term order as in LayoutPlan.dict_keys) into the
    global descending unique dictionary."""
    runs = [np.asarray(r) for r in runs if len(r)]
    if not runs:
        return np.zeros((0, 1), dtype=np.uint64)
    allk = np.concatenate(runs)
    uniq = np.unique(allk, axis=0)  # ascending lexicographic = ascending term order
    return uniq[::-1].copy()


def concat_csr(slices):
    """Concatenate per-rank CSR slices (row_ptr local to the slice, columns in
    the global dictionary) in rank order -> (row_ptr, col_ind, val)."""
    rps, cis, vas = [], [], []
    base = 0
    for rp, ci, va in slices:
        rp = np.asarray(rp, dtype=np.int64)
        rps.append(rp[:-1] + base if len(rp) else rp)
        cis.append(np.asarray(ci))
        vas.append(np.asarray(va))
        base += int(rp[-1]) if len(rp) else 0
    row_ptr = np.concatenate(rps + [np.array([base], dtype=np.int64)])
    return row_ptr, np.concatenate(cis) if cis else np.zeros(0, np.int64), np.concatenate(vas) if vas else np.zeros(0)


def remap_columns(local_keys_desc: np.ndarray, global_keys_desc: np.ndarray) -> np.ndarray:
    """Column index of every local dictionary key in the global descending
    dictionary (the join of a rank's slice against the merged dictionary)."""
    if len(local_keys_desc) == 0:
        return np.zeros(0, dtype=np.int64)
    g_asc = global_keys_desc[::-1]
    view = lambda a: np.ascontiguousarray(a).view([("", a.dtype)] * a.shape[1]).ravel()  # noqa: E731
    pos_asc = np.searchsorted(view(g_asc), view(local_keys_desc))
    return (len(global_keys_desc) - 1 - pos_asc).astype(np.int64)


class ShardedCompiler:
    """compile_batch split across the ranks of a process group,
    on each rank's CUDA engine (csrc/shard.cu, C ABI f4b_shard_*).

    Per call, every rank passes the same rows:

    1. rows split into contiguous ranges balanced by term count; each rank
       materialises its range and builds its sorted unique run of monomial
       ranks (rank order = key order) -> all-gather of the runs -> every rank
       holds the identical dictionary (reference _materialize + radix_sort +
       unique_sorted, symbolic.py:204-225, :330-333);
    2. closure rounds (symbolic.py:335-363): the frontier (identical on every
       rank, ascending key(m)) split into contiguous slices; each rank finds the
       reducers of its slice and ranks their rows' terms -> all-gather of the
       reducer indices (frontier order, so rows stay in ascending key(m)) and
       of the new-monomial runs -> identical rows and next frontier everywhere;
    3. the final row list split by term count; each rank joins its range
       against the dictionary (merge_join_index) -> its plan slice.

    Collectives: torch.distributed all_gather of int32 tensors on the rank's
    GPU (NCCL) or on the host (gloo); two per exchange (sizes, then the padded
    payload).  ``compile`` returns (DevicePlan slice, device ns of the whole
    call incl. collectives, stats).  Concatenating the slices of all ranks in
    rank order is the single-GPU plan byte for byte."""

    def __init__(self, engine, group=None):
        import torch
        import torch.distributed as dist

        self.eng = engine
        self.group = group
        self.world = dist.get_world_size(group)
        self.rank = dist.get_rank(group)
        nccl = dist.get_backend(group) == "nccl"
        self.dev = torch.device("cuda", torch.cuda.current_device()) if nccl else torch.device("cpu")
        self.exchanges = 0
        self.bytes = 0

    def _allgather(self, t):
        """Variable-length all-gather of a 1-D int32 tensor -> concatenation
        in rank order."""
        import torch
        import torch.distributed as dist

        n = torch.tensor([t.numel()], dtype=torch.int64, device=self.dev)
        sizes = [torch.empty_like(n) for _ in range(self.world)]
        dist.all_gather(sizes, n, group=self.group)
        sizes = [int(x) for x in sizes]
        cap = max(1, max(sizes))
        buf = torch.zeros(cap, dtype=torch.int32, device=self.dev)
        if t.numel():
            buf[: t.numel()] = t
        outs = [torch.empty(cap, dtype=torch.int32, device=self.dev) for _ in range(self.world)]
        dist.all_gather(outs, buf, group=self.group)
        self.exchanges += 1
        self.bytes += 4 * sum(sizes)
        return torch.cat([o[:s] for o, s in zip(outs, sizes)]) if sum(sizes) else buf[:0]

    def _take_run(self, h, n):
        import torch

        run = torch.empty(int(n), dtype=torch.int32, device=self.dev)
        if n:
            self.eng.ctx.check(self.eng.lib.f4b_shard_take_run(h, C_ptr(run), int(n)), "shard take_run")
        return run

    def compile(self, row_basis, row_shift, closure: bool = True, candidates=None, dict_cap=10**6):
        import ctypes as C

        import torch

        from .engine import DevicePlan, ptr

        eng = self.eng
        lib, ctx = eng.lib, eng.ctx
        rb = np.ascontiguousarray(row_basis, dtype=np.int32)
        sh = np.ascontiguousarray(np.asarray(row_shift), dtype=np.uint16).reshape(len(rb), eng.n_vars)
        cand = None if candidates is None else np.ascontiguousarray(candidates, dtype=np.int32)
        ctx.sync_stream()
        stream = torch.cuda.current_stream()
        ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        ev0.record(stream)
        lens = eng.basis_lengths()[rb]
        lo, hi = balanced_ranges(lens, self.world)[self.rank]
        h = C.c_void_p()
        nrun = C.c_int64()
        ctx.check(lib.f4b_shard_begin(ctx.h, len(rb), ptr(rb, C.c_int32), ptr(sh, C.c_uint16), 1 if closure else 0,
                                      ptr(cand, C.c_int32) if cand is not None else None,
                                      0 if cand is None else len(cand), int(dict_cap), lo, hi, C.byref(h),
                                      C.byref(nrun)), "shard begin")
        try:
            runs = self._allgather(self._take_run(h, nrun.value))
            nf = C.c_int64()
            ctx.check(lib.f4b_shard_merge(h, C_ptr(runs), runs.numel(), C.byref(nf)), "shard merge")
            rounds = 0
            while nf.value > 0:
                per = -(-nf.value // self.world)
                f_lo, f_hi = min(nf.value, self.rank * per), min(nf.value, (self.rank + 1) * per)
                red = torch.empty(max(f_hi - f_lo, 0), dtype=torch.int32, device=self.dev)
                ctx.check(lib.f4b_shard_round(h, f_lo, f_hi, C_ptr(red), C.byref(nrun)), "shard round")
                run = self._take_run(h, nrun.value)
                red_all = self._allgather(red)
                runs = self._allgather(run)
                ctx.check(lib.f4b_shard_round_merge(h, C_ptr(red_all), nf.value, C_ptr(runs), runs.numel(),
                                                    C.byref(nf)), "shard round merge")
                rounds += 1
            r_total = C.c_int64()
            ctx.check(lib.f4b_shard_rows(h, C.byref(r_total), None), "shard rows")
            starts = np.empty(r_total.value + 1, dtype=np.uint32)
            ctx.check(lib.f4b_shard_rows(h, C.byref(r_total), starts.ctypes.data_as(C.c_void_p)), "shard rows")
            lo2, hi2 = balanced_ranges(np.diff(starts.astype(np.int64)), self.world)[self.rank]
            ph = C.c_void_p()
            ctx.check(lib.f4b_shard_finish(h, lo2, hi2, C.byref(ph)), "shard finish")
            plan = DevicePlan(eng, ph)
        finally:
            lib.f4b_shard_free(h)
        ev1.record(stream)
        ev1.synchronize()
        ns = int(ev0.elapsed_time(ev1) * 1e6)
        return plan, ns, {"rows": (lo2, hi2), "input_rows": (lo, hi), "exchange_rounds": rounds}


def C_ptr(t):
    """Raw data pointer of a torch tensor (host or device) for the C ABI."""
    import ctypes as C

    return C.c_void_p(t.data_ptr()) if t.numel() else None
