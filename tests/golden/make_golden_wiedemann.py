"""Golden left-kernel vectors from the REAL reference (`fpgb`, /root/reference).

Runs the reference F4 loop with ``F4Config(numeric="wiedemann")`` (the BASELINE
MQ-16 config: ``gen_random_quadratic(16, 32, 1.0, 0, 31)``, block_width 4,
seed 0) for the first ``--steps`` steps and records, per step, what
``f4_step`` returns as ``kernel`` (reference ``src/groebner.py:276-283`` →
``left_kernel``, ``src/sparselin.py:551-569``; Wiedemann above DENSE_CAP,
``:450-548``):

* ``kernel_sha256``  sha256 over ``"v:" + ",".join(vector) + ";"`` per vector
  (in the order returned);
* ``dimension_found``, ``seed_trail``, the vector count and the first vector
  (small) so a mismatch can be diagnosed;
* the plan and RREF digests (same recipe as make_golden.py).

Runs only in the build container (the reference does not exist on the GPU box).
Step 1 (584 x 968) takes about 2-3 minutes on one core.

Usage::

    python tests/golden/make_golden_wiedemann.py [--steps 2]
"""
import argparse
import hashlib
import json
import os
import sys
import time

sys.path.insert(0, "/root/reference/pkg/src")
sys.dont_write_bytecode = True

from fpgb.groebner import F4Config, GroebnerState, f4_step, update_pairs  # noqa: E402
from fpgb.polynomials import poly_monic  # noqa: E402
from fpgb.symbolic import plan_digest  # noqa: E402
from fpgb.systems import gen_random_quadratic  # noqa: E402

HERE = os.path.dirname(os.path.abspath(__file__))


def rref_digest(ech):
    h = hashlib.sha256()
    for lead, cols, vals in list(ech.pivot_rows) + list(ech.nonpivot_rows):
        h.update(f"{lead}:{cols.tolist()}:{vals.tolist()};".encode())
    return h.hexdigest()


def kernel_digest(vectors):
    h = hashlib.sha256()
    for v in vectors:
        h.update(("v:" + ",".join(str(int(x)) for x in v) + ";").encode())
    return h.hexdigest()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--steps", type=int, default=2)
    args = ap.parse_args()
    ring, polys = gen_random_quadratic(16, 32, 1.0, 0, 31)
    cfg = F4Config(numeric="wiedemann", block_width=4, seed=0)
    st = GroebnerState(ring)
    for f in polys:
        update_pairs(st, poly_monic(f))
    steps = []
    for k in range(args.steps):
        t0 = time.time()
        plan, ech, kb = f4_step(st, cfg)
        s = st.stats[-1]
        steps.append({
            "step": k, "r": s.r, "N": s.N, "M": s.M, "rank": s.rank,
            "plan_sha256": plan_digest(plan), "rref_sha256": rref_digest(ech),
            "kernel_side": kb.side, "dimension_found": kb.dimension_found,
            "n_vectors": len(kb.vectors),
            "seed_trail": [list(t) for t in kb.seed_trail],
            "kernel_sha256": kernel_digest(kb.vectors),
            "first_vector": [int(x) for x in kb.vectors[0]] if kb.vectors else [],
            "ref_wall_s": round(time.time() - t0, 2),
        })
        print(json.dumps({k2: v for k2, v in steps[-1].items() if k2 != "first_vector"}), flush=True)
    out = {"config": "mq16x32_p31", "numeric": "wiedemann", "block_width": 4, "seed": 0, "steps": steps}
    with open(os.path.join(HERE, "mq16x32_p31_wiedemann.json"), "w") as fh:
        json.dump(out, fh, indent=1)
    print("done")


if __name__ == "__main__":
    main()
