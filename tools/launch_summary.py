"""Summarise an ncu launch list (--metrics gpu__time_duration.sum,
dram__bytes_read.sum,dram__bytes_write.sum --csv) into the committed
profiles/<round>/launches_bench_summary.txt and traffic_bench.json
(per-kernel mean DRAM bytes per launch, read by bench.py's roofline).

usage: python tools/launch_summary.py launches.csv profiles/r02 "<command line>"
"""

import collections
import csv
import json
import os
import re
import sys


def _profile_name(n):
    """ncu's demangled template name -> the library's launch-profile name."""
    m = re.match(r"(k_fbsp|k_dense_blk)<", n)
    if m:
        return m.group(1)
    m = re.match(r"k_sweep_win<(\d), (\d)", n)
    if m:
        pk = "true" if m.group(1) == "1" else "false"
        return f"k_sweep_win<{pk}>" if m.group(2) == "0" else f"k_sweep_win<{pk},1>"
    m = re.match(r"k_tail_copy<(\d)>", n)
    if m:
        return "k_tail_copy<true>" if m.group(1) == "1" else "k_tail_copy<false>"
    return n


def main():
    src, outdir, cmd = sys.argv[1], sys.argv[2], sys.argv[3]
    rows = list(csv.reader(open(src)))
    hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hdr]
    ki, mi, vi, ii = h.index("Kernel Name"), h.index("Metric Name"), h.index("Metric Value"), h.index("ID")
    per = collections.OrderedDict()
    for r in rows[hdr + 1:]:
        if len(r) <= vi:
            continue
        per.setdefault(r[ii], {"name": r[ki]})[r[mi]] = float(r[vi].replace(",", ""))
    agg = collections.defaultdict(lambda: [0, 0.0, 0.0])
    for d in per.values():
        name = re.sub(r"\(.*", "", d["name"]).strip()
        name = re.sub(r"^void ", "", name)
        a = agg[name]
        a[0] += 1
        a[1] += d.get("gpu__time_duration.sum", 0.0) / 1e6  # ns -> ms
        a[2] += d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    tot = sum(a[1] for a in agg.values())
    lines = [f"# ncu launch list of `{cmd}`",
             "# (--metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none; cold,",
             "#  serialised replays: use the SHARE, not the absolute times).  Includes the setup F4 run, the warm-up and",
             "#  timed replay steps and the FULL_RREF pass (k_sweep_win<true,1> = the pivot-row back-reduction).",
             f"{'kernel':70s} {'launches':>9s} {'total_ms':>9s} {'share':>6s} {'dram_MB/launch':>14s}"]
    traffic = {}
    for name, (n, ms, by) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
        lines.append(f"{name[:70]:70s} {n:9d} {ms:9.3f} {ms / tot:6.3f} {by / n / 1e6:14.3f}")
        short = _profile_name(re.sub(r"^f4b::", "", name))
        traffic[short] = {"dram_bytes_per_launch": int(by / n), "launches": n,
                          "source": f"{outdir}/launches_bench_summary.txt (ncu dram__bytes_read.sum + "
                                    "dram__bytes_write.sum, mean per launch over the same 38 cyclic-8 batches the "
                                    "bench replays)"}
    with open(os.path.join(outdir, "launches_bench_summary.txt"), "w") as fh:
        fh.write("\n".join(lines) + "\n")
    with open(os.path.join(outdir, "traffic_bench.json"), "w") as fh:
        json.dump(traffic, fh, indent=1)
    print("\n".join(lines[:20]))


if __name__ == "__main__":
    main()
