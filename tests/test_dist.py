"""Multi-rank host logic on CPU (gloo, world_size 2): SURVEY.md §8e.

The FBSP row partition (contiguous ranges balanced by Σ lengths), the
all-gather + merge of per-rank dictionary runs, the column remap and the
rank-order CSR concatenation must reproduce the single-rank plan exactly;
the max / sum reductions used for multi-rank timing must agree on every rank.
"""

import socket

import numpy as np
import pytest

from paper_2601_06765_b200 import dist as pdist


def _free_port():
    with socket.socket() as s:
        s.bind(("127.0.0.1", 0))
        return s.getsockname()[1]


def test_balanced_ranges_cover_and_balance():
    w = np.array([5, 1, 1, 1, 9, 2, 2, 3, 3, 3])
    for world in (1, 2, 3, 4, 16):
        rs = pdist.balanced_ranges(w, world)
        assert len(rs) == world
        assert rs[0][0] == 0 and rs[-1][1] == len(w)
        assert all(a[1] == b[0] for a, b in zip(rs, rs[1:]))
        sums = [int(w[lo:hi].sum()) for lo, hi in rs]
        assert sum(sums) == int(w.sum())
        if world <= 3:
            assert max(sums) <= w.sum() / world + w.max()


def test_merge_and_remap_single_process():
    rng = np.random.default_rng(1)
    keys = np.unique(rng.integers(0, 1 << 20, size=(300, 2), dtype=np.uint64), axis=0)[::-1]
    parts = [keys[i::3] for i in range(3)]
    g = pdist.merge_key_runs(parts)
    assert np.array_equal(g, keys)
    for p in parts:
        idx = pdist.remap_columns(p, g)
        assert np.array_equal(g[idx], p)


@pytest.mark.parametrize("snap,step", [("cyclic6_p32003", 4)])
def test_fbsp_join_world2_gloo(tmp_path, snap, step):
    import torch.multiprocessing as mp

    import _dist_worker
    from conftest import load_snapshots

    snaps = load_snapshots(snap)
    if step not in snaps:
        pytest.skip("snapshot missing")
    world = 2
    mp.spawn(_dist_worker.run, args=(world, _free_port(), snap, step, str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        ok, lo, hi, n, nfull = (tmp_path / f"rank{r}.txt").read_text().split()
        assert ok == "1", f"rank {r}: distributed plan differs (rows {lo}:{hi}, N {n} vs {nfull})"


def test_block_wiedemann_columns_world2_gloo(tmp_path):
    """§8e Block Wiedemann: the b block columns dealt over 2 ranks, candidates
    all-gathered once per round; every rank ends with the single-rank
    vectors, in the same order, all in ker(A)."""
    import torch.multiprocessing as mp

    import _dist_worker

    p = 31
    A = _dist_worker.wiedemann_case(p)
    single, _ = _dist_worker.wiedemann_rounds(A, p, 0, 1)
    assert single, "expected kernel vectors"
    for w in single:
        assert not (A @ w % np.uint64(p)).any()
    world = 2
    mp.spawn(_dist_worker.run_wiedemann, args=(world, _free_port(), str(tmp_path)), nprocs=world, join=True)
    for r in range(world):
        got = np.load(tmp_path / f"wied_rank{r}.npy")
        assert np.array_equal(got, np.array(single, dtype=np.uint64))
