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
    acc = {"clear": 0.0, "upload": 0.0, "compile": 0.0, "rowptr": 0.0, "colval": 0.0, "dict": 0.0}
    M = 0
    for rep in range(2):
        for k in acc:
            acc[k] = 0.0
        M = 0
        for b in batches:
            nb_, nt = b["n_basis"], b["n_terms"]
            soa = SoaPolySet(ring, final.mon_key[:nt], final.coeff[:nt], final.offset[:nb_ + 1],
                             final.length[:nb_], final.exps[:nt])
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            eng.clear_basis()
            t1 = time.perf_counter()
            eng.sync_basis(soa)
            torch.cuda.synchronize()
            t2 = time.perf_counter()
            plan = compile_batch(b["rows"], soa)
            t3 = time.perf_counter()
            rp = plan.row_ptr
            t4 = time.perf_counter()
            ci, va = plan.col_ind, plan.val
            t5 = time.perf_counter()
            dk = plan.dict_keys
            t6 = time.perf_counter()
            acc["clear"] += t1 - t0
            acc["upload"] += t2 - t1
            acc["compile"] += t3 - t2
            acc["rowptr"] += t4 - t3
            acc["colval"] += t5 - t4
            acc["dict"] += t6 - t5
            M += b["M"]
            del rp, ci, va, dk
    tot = sum(acc.values())
    print({k: round(v * 1e3, 2) for k, v in acc.items()}, "total_ms", round(tot * 1e3, 2), "nnz/s", M / tot)


if __name__ == "__main__":
    main()
