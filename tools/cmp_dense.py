"""Per-batch device time of the F_p elimination (psge, NEW_ONLY) of the cyclic-8
replay under two "dense" options (diagnostic): python tools/cmp_dense.py 0 2"""

import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    import torch

    from paper_2601_06765_b200.engine import Engine

    opts = [int(x) for x in sys.argv[1:]] or [0, 2]
    ring, st, batches, setup = bench.capture_workload()
    eng = Engine.for_ring(ring)
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    tot = {o: 0.0 for o in opts}
    for i, b in enumerate(batches):
        plan = eng.compile(b["rb"], b["sh"], True, list(range(b["n_basis"])))
        row = []
        for o in opts:
            eng.set_option("dense", o)
            best = 1e9
            for _ in range(3):
                flush.fill_(1)
                torch.cuda.synchronize()
                inf = eng.psge_plan(plan, full=False).info()
                best = min(best, inf["numeric_ns"] / 1e3)
            tot[o] += best
            row.append(best)
        print(i, b["r"], " ".join(f"{x:8.1f}" for x in row), flush=True)
    eng.set_option("dense", 0)
    print("total_us", " ".join(f"{tot[o]:.1f}" for o in opts))


if __name__ == "__main__":
    main()
