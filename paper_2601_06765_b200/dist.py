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
