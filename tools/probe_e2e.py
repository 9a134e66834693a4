"""Where the end-to-end (host-buffer) time of bench.py's e2e leg goes.

Replays every cyclic-8 batch through the public API exactly like bench.py's
e2e loop (fresh device basis per batch) and splits the wall time into basis
upload, compile_batch and the LayoutPlan downloads.  Diagnostic only.
"""

import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    import torch

    from paper_2601_06765_b200.engine import Engine
    from paper_2601_06765_b200.polynomials import SoaPolySet
    from paper_2601_06765_b200.symbolic import compile_batch

    ring, st, batches, _ = bench.capture_workload()
    eng = Engine.for_ring(ring)
    final = st.soa()
    acc = {}
    M = 0
    import cProfile
    import pstats

    prof = cProfile.Profile()
    for rep in range(3):
        acc = {k: 0.0 for k in ("compile", "rowptr_col_val", "dict_keys")}
        M = 0
        eng.clear_basis()
        if rep == 2:
            prof.enable()
        for b in batches:
            nb_, nt = b["n_basis"], b["n_terms"]
            soa = SoaPolySet(ring, final.mon_key[:nt], final.coeff[:nt], final.offset[:nb_ + 1],
                             final.length[:nb_], final.exps[:nt])
            t2 = time.perf_counter()
            plan = compile_batch(b["rows"], soa)
            t3 = time.perf_counter()
            rp, ci, va = plan.row_ptr, plan.col_ind, plan.val
            t5 = time.perf_counter()
            dk = plan.dict_keys
            t6 = time.perf_counter()
            acc["compile"] += t3 - t2
            acc["rowptr_col_val"] += t5 - t3
            acc["dict_keys"] += t6 - t5
            M += b["M"]
            del rp, ci, va, dk
        if rep == 2:
            prof.disable()
    tot = sum(acc.values())
    print({k: round(v * 1e3, 2) for k, v in acc.items()}, "total_ms", round(tot * 1e3, 2), "nnz/s", M / tot)
    pstats.Stats(prof).sort_stats("cumulative").print_stats(25)


if __name__ == "__main__":
    main()
