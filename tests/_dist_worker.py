"""Worker for tests/test_dist.py (gloo, CPU): the multi-rank FBSP join scheme
of SURVEY.md §8e checked against the single-rank oracle plan.  Test
infrastructure: the per-rank compute here is the oracle, not the engine."""

import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for pth in (ROOT, HERE):
    if pth not in sys.path:
        sys.path.insert(0, pth)


def run(rank, world, port, snap_name, step, out_dir):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    import torch.distributed as dist

    import oracle
    from paper_2601_06765_b200 import dist as pdist
    from paper_2601_06765_b200.groebner import select_batch
    from paper_2601_06765_b200.symbolic import select_rows
    from conftest import load_snapshots, state_from_snapshot

    info = pdist.init("gloo")
    assert (info.rank, info.world) == (rank, world)
    ring, st = state_from_snapshot(load_snapshots(snap_name)[step])
    spec, _ = select_batch(st)
    soa = st.soa()
    rows = [(r.shift, r.basis_index, r.role.value, r.provenance) for r in select_rows(spec, soa)]
    basis = (soa.exps, soa.coeff, soa.offset, soa.length)
    full = oracle.compile_batch_arrays(rows, basis, ring.order, closure=True)
    all_rows = [(tuple(r.shift) if hasattr(r, "shift") else tuple(r[0]),
                 r.basis_index if hasattr(r, "basis_index") else r[1], 0, 0) for r in full["row_meta"]]
    lens = [int(soa.length[b]) for _, b, _, _ in all_rows]
    lo, hi = pdist.balanced_ranges(lens, world)[rank]
    local = oracle.compile_batch_arrays(all_rows[lo:hi], basis, ring.order, closure=False)
    runs = pdist.allgather_arrays(local["dict_keys"])
    gdict = pdist.merge_key_runs(runs)
    cols = pdist.remap_columns(local["dict_keys"], gdict)[local["col_ind"]] if len(local["col_ind"]) else local["col_ind"]
    slices = pdist.allgather_arrays(np.asarray(local["row_ptr"], dtype=np.int64).reshape(-1, 1))
    colsl = pdist.allgather_arrays(np.asarray(cols, dtype=np.int64).reshape(-1, 1))
    valsl = pdist.allgather_arrays(np.asarray(local["val"], dtype=np.uint64).reshape(-1, 1))
    rp, ci, va = pdist.concat_csr([(a.ravel(), b.ravel(), c.ravel()) for a, b, c in zip(slices, colsl, valsl)])
    tmax = pdist.max_over_ranks(float(rank + 1))
    tsum = pdist.sum_over_ranks(1.0)
    ok = (np.array_equal(gdict, full["dict_keys"]) and np.array_equal(rp, full["row_ptr"])
          and np.array_equal(ci, full["col_ind"]) and np.array_equal(va, full["val"])
          and tmax == float(world) and tsum == float(world))
    with open(os.path.join(out_dir, f"rank{rank}.txt"), "w") as fh:
        fh.write(f"{int(ok)} {lo} {hi} {len(gdict)} {len(full['dict_keys'])}\n")
    dist.barrier()
    dist.destroy_process_group()


class NumpyKrylovOperator:
    """Test stand-in for the device operator (engine.DeviceOperator): B = A
    (square) or AᵀA, dense NumPy mod p, with the reference loop semantics
    (sparselin.py:482-528).  Test infrastructure only: it lets the multi-rank
    Block Wiedemann control flow run on CPU ranks."""

    def __init__(self, A, p):
        self.A = np.asarray(A, dtype=np.uint64)
        self.p = np.uint64(p)
        self.square = self.A.shape[0] == self.A.shape[1]
        self.dim = self.A.shape[1]

    def apply(self, X):
        Y = self.A @ X % self.p
        return Y if self.square else self.A.T @ Y % self.p

    def krylov(self, U, V, steps):
        W = np.array(V, dtype=np.uint64)
        out = np.empty((steps, W.shape[1]), dtype=np.uint64)
        for k in range(steps):
            out[k] = (U * W % self.p).sum(axis=0, dtype=np.uint64) % self.p
            W = self.apply(W)
        return out

    def horner(self, g, v):
        v = np.asarray(v, dtype=np.uint64).reshape(-1, 1)
        acc = np.uint64(g[-1]) * v % self.p
        for c in list(g[:-1])[::-1]:
            acc = (self.apply(acc) + np.uint64(c) * v) % self.p
        return acc[:, 0]

    def power_until_zero(self, v, max_steps):
        acc = np.asarray(v, dtype=np.uint64).reshape(-1, 1)
        taken = 0
        for _ in range(max_steps):
            nxt = self.apply(acc)
            if (nxt == 0).all():
                break
            acc = nxt
            taken += 1
        return acc[:, 0], taken


def wiedemann_case(p=31, seed=7):
    """A rank-deficient 40 x 30 matrix (rank 20) over F_p."""
    rng = np.random.default_rng(seed)
    L = rng.integers(0, p, (40, 20), dtype=np.uint64)
    R = rng.integers(0, p, (20, 30), dtype=np.uint64)
    return L @ R % np.uint64(p)


def wiedemann_rounds(A, p, rank, world, seed=3, target=6):
    import oracle
    from paper_2601_06765_b200.sparselin import _kernel_rounds

    op = NumpyKrylovOperator(A, p)

    def bm(seqs):
        return [oracle.berlekamp_massey(seqs[:, k].tolist(), p) for k in range(seqs.shape[1])]

    def check(w):
        return not (A @ w % np.uint64(p)).any()

    return _kernel_rounds(op, bm, check, A.shape[1], p, seed, 4, target, 12, 3, rank, world)


def run_wiedemann(rank, world, port, out_dir):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK=str(rank), MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    from paper_2601_06765_b200 import dist as pdist

    info = pdist.init("gloo")
    assert pdist.active_world() == (rank, world) == (info.rank, info.world)
    p = 31
    vectors, trail = wiedemann_rounds(wiedemann_case(p), p, rank, world)
    np.save(os.path.join(out_dir, f"wied_rank{rank}.npy"), np.array(vectors, dtype=np.uint64))
    import torch.distributed as dist

    dist.barrier()
    dist.destroy_process_group()
