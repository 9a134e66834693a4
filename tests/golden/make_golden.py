"""Generate golden fixtures by running the REAL reference (`fpgb`, /root/reference).

Runs only in the build container (the reference does not exist on the GPU box).
Outputs (committed, small):

* ``<config>.json``   per-F4-step shape counters, ``plan_digest`` (reference
  ``src/symbolic.py:463-466``) and an RREF digest (recipe of SURVEY.md
  Appendix A: sha256 over ``f"{lead}:{cols}:{vals};"`` for pivot rows then
  nonpivot rows), plus the sha256 of the final reduced basis text
  (reference ``src/bench.py:296-297``, ``src/systems.py:125-132``).
* ``<config>.snap.json.gz`` (optional) state snapshots before selected steps:
  the basis as system text plus the queued pair list ``[(i, j)]`` — enough to
  rebuild a ``GroebnerState`` and replay the step.

Usage::

    python tests/golden/make_golden.py cyclic 5 32003 [--snap all|k1,k2] [--max-steps K]
"""
import argparse
import gzip
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from fpgb.groebner import GroebnerState, f4_step, reduce_basis, update_pairs  # noqa: E402
from fpgb.polynomials import poly_monic  # noqa: E402
from fpgb.symbolic import plan_digest  # noqa: E402
from fpgb.systems import format_system, gen_cyclic, gen_katsura, gen_random_quadratic  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def rref_digest(ech):
    h = hashlib.sha256()
    for lead, cols, vals in list(ech.pivot_rows) + list(ech.nonpivot_rows):
        h.update(f"{lead}:{cols.tolist()}:{vals.tolist()};".encode())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("family")
    ap.add_argument("n", type=int)
    ap.add_argument("p", type=int)
    ap.add_argument("--m", type=int, default=0)
    ap.add_argument("--snap", default="")
    ap.add_argument("--max-steps", type=int, default=10**9)
    args = ap.parse_args()
    if args.family == "cyclic":
        ring, polys = gen_cyclic(args.n, args.p)
        name = f"cyclic{args.n}_p{args.p}"
    elif args.family == "katsura":
        ring, polys = gen_katsura(args.n, args.p)
        name = f"katsura{args.n}_p{args.p}"
    else:
        ring, polys = gen_random_quadratic(args.n, args.m, 1.0, 0, args.p)
        name = f"mq{args.n}x{args.m}_p{args.p}"
    snap_all = args.snap == "all"
    snap_set = set(int(x) for x in args.snap.split(",") if x and x != "all")
    st = GroebnerState(ring)
    for f in polys:
        update_pairs(st, poly_monic(f))
    steps, snaps = [], {}
    k = 0
    t_loop = time.time()
    while st.pairs and k < args.max_steps:
        if snap_all or k in snap_set:
            snaps[k] = {
                "basis": format_system(ring, st.basis),
                "pairs": [[q.i, q.j] for q in st.pairs],
            }
        t0 = time.time()
        plan, ech, _ = f4_step(st)
        s = st.stats[-1]
        steps.append({
            "step": k, "degree": s.degree, "r": s.r, "N": s.N, "M": s.M,
            "closure_rounds": s.closure_rounds, "rank": s.rank, "new_polys": s.new_polys,
            "zero_reductions": s.zero_reductions,
            "plan_sha256": plan_digest(plan), "rref_sha256": rref_digest(ech),
            "ref_ns": {k2: int(v) for k2, v in s.timings_ns.items()},
            "ref_wall_s": round(time.time() - t0, 3),
        })
        print(json.dumps(steps[-1]), flush=True)
        k += 1
    out = {"config": name, "p": args.p, "family": args.family, "n": args.n,
           "complete": not st.pairs, "steps": steps,
           "f4_loop_s": round(time.time() - t_loop, 2)}
    if not st.pairs:
        t0 = time.time()
        gb = reduce_basis(st.basis, ring)
        text = format_system(ring, gb)
        out.update(final_sha256=hashlib.sha256(text.encode()).hexdigest(), gb_size=len(gb),
                   reduce_basis_s=round(time.time() - t0, 2))
    with open(os.path.join(HERE, f"{name}.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    if snaps:
        with gzip.open(os.path.join(HERE, f"{name}.snap.json.gz"), "wt") as fh:
            json.dump({"config": name, "snapshots": snaps}, fh)
    print("done", name, out.get("final_sha256"))


if __name__ == "__main__":
    main()
