"""Worker for tests/test_gpu_shard.py: the sharded compile_batch of SURVEY
§8e on the CUDA engine (csrc/shard.cu) — `world` processes share cuda:0 and
exchange over gloo (host all-gathers; the kernels never wait on each other).
Every rank compiles the same batches twice: the single-GPU compile_batch and
its slice of the sharded compile; the slices are gathered to rank 0 and
concatenated in rank order, which must equal the single-GPU plan array for
array (row_ptr, col_ind, val, dictionary exponents, closure rows, counters)."""

import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
ROOT = os.path.dirname(HERE)
for pth in (ROOT, HERE):
    if pth not in sys.path:
        sys.path.insert(0, pth)


def _batches(name):
    """(ring, soa, rb, sh, n_basis) of every batch of a whole GPU F4 run
    (cyclicN) or of the reference snapshots (north-star replays)."""
    from paper_2601_06765_b200.groebner import GroebnerState, f4_step, select_batch, update_pairs
    from paper_2601_06765_b200.polynomials import poly_monic
    from paper_2601_06765_b200.symbolic import select_rows
    from paper_2601_06765_b200.systems import gen_cyclic, gen_katsura

    out = []
    if name.startswith("snap:"):
        from conftest import load_snapshots, state_from_snapshot

        _, cfg, steps = name.split(":")
        snaps = load_snapshots(cfg)
        for k in [int(x) for x in steps.split(",")]:
            ring, st = state_from_snapshot(snaps[k])
            spec, _ = select_batch(st)
            soa = st.soa()
            rows = select_rows(spec, soa)
            out.append((ring, soa, rows))
        return out
    fam, n = name[:-1], int(name[-1])
    ring, polys = (gen_cyclic if fam == "cyclic" else gen_katsura)(n, 32003)
    st = GroebnerState(ring)
    for f in polys:
        update_pairs(st, poly_monic(f))

    def cap(rows, soa, plan):
        out.append((ring, soa, list(rows)))

    while st.n_pairs():
        f4_step(st, _capture=cap)
    return out


def run(rank, world, port, name, out_dir):
    os.environ.update(RANK=str(rank), WORLD_SIZE=str(world), LOCAL_RANK="0", MASTER_ADDR="127.0.0.1",
                      MASTER_PORT=str(port))
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2601_06765_b200.dist import ShardedCompiler, allgather_arrays
    from paper_2601_06765_b200.engine import Engine

    report = []
    for ring, soa, rows in _batches(name):
        eng = Engine.for_ring(ring)
        eng.sync_basis(soa)
        rb = np.array([r.basis_index for r in rows], dtype=np.int64)
        sh = np.array([r.shift for r in rows], dtype=np.int64).reshape(len(rows), ring.n_vars)
        full = eng.compile(rb, sh, True, None)
        fd = full.download()
        sc = ShardedCompiler(eng)
        part, ns, stats = sc.compile(rb, sh, True, None)
        pd = part.download()
        rp = allgather_arrays(np.diff(pd["row_ptr"]).astype(np.int64).reshape(-1, 1))
        ci = allgather_arrays(pd["col_ind"].astype(np.int64).reshape(-1, 1))
        va = allgather_arrays(pd["val"].astype(np.int64).reshape(-1, 1))
        lens = np.concatenate([x.ravel() for x in rp])
        row_ptr = np.concatenate([[0], np.cumsum(lens)]).astype(np.int64)
        ok = {
            "row_ptr": bool(np.array_equal(row_ptr, fd["row_ptr"])),
            "col_ind": bool(np.array_equal(np.concatenate([x.ravel() for x in ci]), fd["col_ind"])),
            "val": bool(np.array_equal(np.concatenate([x.ravel() for x in va]), fd["val"].astype(np.int64))),
            "dict_exps": bool(np.array_equal(pd["dict_exps"], fd["dict_exps"])),
            "closure": bool(np.array_equal(pd["cl_basis"], fd["cl_basis"])
                            and np.array_equal(pd["cl_shift"], fd["cl_shift"])
                            and np.array_equal(pd["cl_round"], fd["cl_round"])),
            "counters": [full.info[k] for k in ("N", "closure_rounds")] == [part.info[k] for k in
                                                                          ("N", "closure_rounds")]
                        and part.info["r_total"] == full.info["r"],
        }
        report.append({"r": full.info["r"], "M": full.info["M"], "rows": list(stats["rows"]),
                       "rounds": stats["exchange_rounds"], "ok": ok})
    with open(os.path.join(out_dir, f"rank{rank}.json"), "w") as fh:
        json.dump(report, fh)
    dist.barrier()
    dist.destroy_process_group()


if __name__ == "__main__":
    run(int(sys.argv[1]), int(sys.argv[2]), int(sys.argv[3]), sys.argv[4], sys.argv[5])
