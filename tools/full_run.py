"""Full F4 run of a named system on the GPU with per-step shapes and timings.

usage: python tools/full_run.py katsura 11 [--p 32003] [--max-steps N]
Prints one line per F4 step (degree, r, N, M, rank, new, closure rounds,
symbolic / elimination device ms, |G|, pairs) and a final JSON line with the
wall time, the reduced basis size and the sha256 of its text (the reference's
digest recipe: format_system of the reduced basis).  Diagnostic / evidence
tool; the steps the reference can finish are pinned by tests/golden.
"""

import argparse
import hashlib
import json
import os
import sys
import time

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def standard_monomials(lms, n, cap=10**6):
    """Number of monomials divisible by no leading monomial (the vector-space
    dimension of the quotient ring for a zero-dimensional ideal; Katsura-n
    has 2^n solutions), by a breadth-first walk of the order ideal; None when
    it exceeds `cap` (positive-dimensional ideal)."""
    import numpy as np

    L = np.asarray([list(m) for m in lms], dtype=np.int64).reshape(-1, n)
    seen = {tuple([0] * n)}
    if (L == 0).all(axis=1).any():
        return 0
    frontier = [tuple([0] * n)]
    while frontier:
        nxt = []
        for m in frontier:
            for v in range(n):
                c = list(m)
                c[v] += 1
                c = tuple(c)
                if c in seen:
                    continue
                if (L <= np.asarray(c)).all(axis=1).any():
                    continue
                seen.add(c)
                nxt.append(c)
        if len(seen) > cap:
            return None
        frontier = nxt
    return len(seen)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("family", choices=["cyclic", "katsura", "mq"])
    ap.add_argument("n", type=int)
    ap.add_argument("--p", type=int, default=32003)
    ap.add_argument("--max-steps", type=int, default=10**6)
    ap.add_argument("--numeric", default="psge", choices=["psge", "wiedemann"])
    ap.add_argument("--profile-step", type=int, default=-1,
                    help="wrap that step in cudaProfilerStart/Stop (ncu --profile-from-start off)")
    args = ap.parse_args()
    from paper_2601_06765_b200.groebner import F4Config, GroebnerState, f4_step, reduce_basis_device, update_pairs
    from paper_2601_06765_b200.polynomials import poly_monic
    from paper_2601_06765_b200.systems import format_system, gen_cyclic, gen_katsura, gen_random_quadratic

    if args.family == "cyclic":
        ring, polys = gen_cyclic(args.n, args.p)
    elif args.family == "katsura":
        ring, polys = gen_katsura(args.n, args.p)
    else:
        ring, polys = gen_random_quadratic(args.n, 2 * args.n, density=1.0, seed=0, p=args.p)
    st = GroebnerState(ring)
    for f in polys:
        update_pairs(st, poly_monic(f))
    cfg = F4Config(numeric=args.numeric)
    t0 = time.perf_counter()
    k = 0
    tot_sym = tot_num = 0.0
    while st.n_pairs() and k < args.max_steps:
        ts = time.perf_counter()
        if k == args.profile_step:
            import torch

            torch.cuda.synchronize()
            torch.cuda.profiler.start()
        plan, ech, _ = f4_step(st, cfg)
        if k == args.profile_step:
            torch.cuda.synchronize()
            torch.cuda.profiler.stop()
        c = plan.counters
        sym = (plan.timings_ns["dict_build_ns"] + plan.timings_ns["row_assemble_ns"]) / 1e6
        num = ech.timings().get("numeric_ns", 0) / 1e6
        tot_sym += sym
        tot_num += num
        print(f"step {k:3d} r={c.r:6d} N={c.N:6d} M={c.M:9d} rank={ech.rank:6d} new={len(ech.nonpivot_arrays()[0]):4d} "
              f"rounds={c.closure_rounds} sym={sym:.3f}ms elim={num:.3f}ms wall={time.perf_counter() - ts:.3f}s "
              f"G={len(st.basis)} pairs={st.n_pairs()}", flush=True)
        k += 1
    loop_s = time.perf_counter() - t0
    t1 = time.perf_counter()
    gb = reduce_basis_device(st.basis, ring, st.soa()) if not st.n_pairs() else []
    red_s = time.perf_counter() - t1
    text = format_system(ring, gb) if gb else ""
    staircase = standard_monomials([f.lm() for f in gb], ring.n_vars) if gb else None
    print(json.dumps({"system": f"{args.family}-{args.n}/F_{args.p}", "steps": k, "finished": not st.n_pairs(),
                      "f4_loop_s": round(loop_s, 3), "reduce_basis_s": round(red_s, 3), "gb_size": len(gb),
                      "sum_sym_ms": round(tot_sym, 3), "sum_elim_ms": round(tot_num, 3),
                      "standard_monomials": staircase,
                      "digest": hashlib.sha256(text.encode()).hexdigest() if gb else None}), flush=True)


if __name__ == "__main__":
    main()
