"""cProfile of bench.py's e2e loop (one warm step): where the host time of
the public compile_batch path goes.  Diagnostic only."""

import cProfile
import os
import pstats
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    import torch

    from paper_2601_06765_b200.engine import Engine, host_empty
    from paper_2601_06765_b200.polynomials import SoaPolySet
    from paper_2601_06765_b200.symbolic import compile_batch

    ring, st, batches, _ = bench.capture_workload()
    eng = Engine.for_ring(ring)
    final = st.soa()

    def pinned(a):
        out = host_empty(a.shape, a.dtype)
        out[...] = a
        return out

    f_key, f_coeff, f_exps = pinned(final.mon_key), pinned(final.coeff), pinned(final.exps)

    def step():
        eng.clear_basis()
        pending = None
        for b in batches:
            nb_, nt = b["n_basis"], b["n_terms"]
            soa = SoaPolySet(ring, f_key[:nt], f_coeff[:nt], final.offset[:nb_ + 1], final.length[:nb_], f_exps[:nt])
            plan = compile_batch(b["rows"], soa).prefetch()
            if pending is not None:
                _ = (pending.row_ptr, pending.col_ind, pending.val, pending.dict_keys)
            pending = plan
        _ = (pending.row_ptr, pending.col_ind, pending.val, pending.dict_keys)
        torch.cuda.synchronize()

    step()
    step()
    pr = cProfile.Profile()
    pr.enable()
    step()
    pr.disable()
    pstats.Stats(pr).sort_stats("tottime").print_stats(25)


if __name__ == "__main__":
    main()
