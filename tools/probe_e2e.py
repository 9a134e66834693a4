"""Where the end-to-end (host-buffer) time of bench.py's e2e leg goes.

Replays every cyclic-8 batch through the public API exactly like bench.py's
e2e loop (empty device basis per step, page-locked basis streams, the basis
grown batch by batch) and splits the wall time into: basis upload
(sync_basis), row-list conversion, the compile call, and the LayoutPlan
downloads.  Diagnostic only.
"""

import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    import torch

    from paper_2601_06765_b200.engine import Engine, host_empty
    from paper_2601_06765_b200.polynomials import SoaPolySet
    from paper_2601_06765_b200.hostglue import native
    from paper_2601_06765_b200.symbolic import DICT_CAP

    ring, st, batches, _ = bench.capture_workload()
    eng = Engine.for_ring(ring)
    final = st.soa()

    def pinned(a):
        out = host_empty(a.shape, a.dtype)
        out[...] = a
        return out

    f_key, f_coeff, f_exps = pinned(final.mon_key), pinned(final.coeff), pinned(final.exps)
    n = ring.n_vars
    from paper_2601_06765_b200.symbolic import LayoutPlan, PlanCounters

    for rep in range(3):
        acc = dict.fromkeys(("sync_basis", "rows", "compile", "validate", "prefetch", "consume"), 0.0)
        dev_ms = 0.0
        M = 0
        torch.cuda.synchronize()
        t_all = time.perf_counter()
        eng.clear_basis()
        pending = None
        for b in batches + [None]:
            t0 = time.perf_counter()
            plan = None
            if b is not None:
                nb_, nt = b["n_basis"], b["n_terms"]
                soa = SoaPolySet(ring, f_key[:nt], f_coeff[:nt], final.offset[:nb_ + 1], final.length[:nb_],
                                 f_exps[:nt])
                eng.sync_basis(soa)
            t1 = time.perf_counter()
            if b is not None:
                rows = b["rows"]
                rb = np.empty(len(rows), dtype=np.int32)
                sh = np.empty((len(rows), n), dtype=np.uint16)
                native().pack_rows(rows, n, rb, sh)
            t2 = time.perf_counter()
            if b is not None:
                dev = eng.compile(rb, sh, True, None, DICT_CAP)
            t3 = time.perf_counter()
            if b is not None:
                info = dev.info
                dev_ms += (info["dict_build_ns"] + info["row_assemble_ns"]) / 1e6
                plan = LayoutPlan(ring, counters=PlanCounters(r=info["r"], N=info["N"], M=info["M"], nnz=info["M"],
                                                              keys_emitted=info["M"], keys_generated_total=info["M"]),
                                  device=dev, input_rows=rows)
                plan.validate()
            t4 = time.perf_counter()
            if plan is not None:
                plan.prefetch()
            t5 = time.perf_counter()
            if pending is not None:
                _ = (pending.row_ptr, pending.col_ind, pending.val, pending.dict_keys)
            t6 = time.perf_counter()
            pending = plan
            for k, v in zip(acc, (t1 - t0, t2 - t1, t3 - t2, t4 - t3, t5 - t4, t6 - t5)):
                acc[k] += v
            if b is not None:
                M += b["M"]
        torch.cuda.synchronize()
        tot = time.perf_counter() - t_all
        print({k: round(v * 1e3, 2) for k, v in acc.items()}, "device_compile_ms", round(dev_ms, 2), "total_ms",
              round(tot * 1e3, 2), "nnz/s", round(M / tot), flush=True)


if __name__ == "__main__":
    main()
