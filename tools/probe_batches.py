"""Per-batch kernel breakdown of the cyclic-8 replay (diagnostic tool).

Replays the largest batches one at a time with per-kernel CUDA-event timing
and prints, per batch: shape, t_sym / t_elim (device), launch counts and the
top kernels.  Usage: python tools/probe_batches.py [--top 6] [--full]
"""

import argparse
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import bench  # noqa: E402


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--top", type=int, default=6)
    ap.add_argument("--full", action="store_true")
    ap.add_argument("--brief", action="store_true", help="one short line per batch (symbolic time vs kernel time)")
    ap.add_argument("--reps", type=int, default=2)
    ap.add_argument("--batches", default="", help="comma-separated batch indices (overrides --top)")
    ap.add_argument("--profile-region", action="store_true",
                    help="wrap the last replay of each batch in cudaProfilerStart/Stop (ncu --profile-from-start off)")
    args = ap.parse_args()
    import torch

    from paper_2601_06765_b200.engine import Engine

    ring, st, batches, setup = bench.capture_workload()
    eng = Engine.for_ring(ring)
    order = sorted(range(len(batches)), key=lambda i: -batches[i]["M"])[: args.top]
    if args.batches:
        order = [int(x) for x in args.batches.split(",")]
    flush = torch.empty(256 << 20, dtype=torch.uint8, device="cuda")
    for i in order:
        b = batches[i]
        sprof = {}
        for rep in range(args.reps):
            flush.fill_(1)
            torch.cuda.synchronize()
            last = rep == args.reps - 1
            eng.profile(last and not args.profile_region)
            if last and args.profile_region:
                torch.cuda.profiler.start()
            plan = eng.compile(b["rb"], b["sh"], True, list(range(b["n_basis"])))
            if last and not args.profile_region:
                sprof, _ = eng.profile_read()
                eng.profile(True)
            ech = eng.psge_plan(plan, full=args.full)
            inf = ech.info()
            if last and args.profile_region:
                torch.cuda.synchronize()
                torch.cuda.profiler.stop()
            prof, _ = eng.profile_read() if rep == args.reps - 1 else ({}, 0)
            eng.profile(False)
        if args.brief:
            t_sym = (plan.info["dict_build_ns"] + plan.info["row_assemble_ns"]) / 1e6
            ks = sum(v[1] for v in sprof.values()) / 1e6
            print(f"batch {i:2d} M={b['M']:8d} rounds={plan.info['closure_rounds']} t_sym={t_sym:.3f}ms "
                  f"sym_kernels={ks:.3f}ms gap={t_sym - ks:.3f}ms launches={plan.info['kernel_launches']} "
                  f"elim={inf['numeric_ns'] / 1e6:.3f}ms", flush=True)
            continue
        top = sorted(prof.items(), key=lambda kv: -kv[1][1])[:8]
        ksum = sum(v[1] for v in prof.values()) / 1e6
        print(json.dumps({
            "batch": i, "r": b["r"], "N": b["N"], "M": b["M"], "rounds": plan.info["closure_rounds"],
            "t_sym_ms": (plan.info["dict_build_ns"] + plan.info["row_assemble_ns"]) / 1e6,
            "dict_ms": plan.info["dict_build_ns"] / 1e6, "join_ms": plan.info["row_assemble_ns"] / 1e6,
            "elim_ms": inf["numeric_ns"] / 1e6, "backsub_ms": inf["backsub_ns"] / 1e6,
            "C": inf["dense_rows"], "K": inf["dense_cols"], "rank": inf["rank"],
            "pivots": inf["sweep_pivots"], "tail_nnz": inf["sweep_tail_nnz"],
            "launches_sym": plan.info["kernel_launches"], "kernel_ms_total": round(ksum, 3),
            "sym_kernel_ms": round(sum(v[1] for v in sprof.values()) / 1e6, 3),
            "sym_top": {k: [v[0], round(v[1] / 1e6, 3)] for k, v in sorted(sprof.items(), key=lambda kv: -kv[1][1])},
            "top": {k: [v[0], round(v[1] / 1e6, 3)] for k, v in top}}), flush=True)


if __name__ == "__main__":
    main()
