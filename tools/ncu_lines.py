"""Top CUDA source lines of an ncu report by warp-stall samples.

usage: python tools/ncu_lines.py report.ncu-rep [--kernel-index 0] [--top 30]
(needs a report captured with --import-source on from a -lineinfo build)
"""

import argparse
import csv
import io
import subprocess


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("report")
    ap.add_argument("--top", type=int, default=30)
    ap.add_argument("--kernel", default="", help="kernel name regex (ncu --kernel-name regex:...)")
    args = ap.parse_args()
    flt = ["--kernel-name", "regex:" + args.kernel, "--launch-count", "1"] if args.kernel else []
    out = subprocess.run(["ncu", "-i", args.report, *flt, "--page", "source", "--csv", "--print-source", "cuda,sass"],
                         capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(out)))
    lines = []  # (samples, file, line, src, stall breakdown)
    fname = ""
    hdr = None
    for r in rows:
        if not r:
            continue
        if r[0] == "File Path":
            fname = r[1].rsplit("/", 1)[-1]
            continue
        if r[0] == "Line No":
            hdr = r
            continue
        if hdr is None or r[0] in ("", "Function Name", "Kernel Name"):
            continue
        ci = {k: i for i, k in enumerate(hdr) if k not in ("Source",)}
        try:
            smp = float(r[hdr.index("Warp Stall Sampling (All Samples)")] or 0)
        except (ValueError, IndexError):
            continue
        if smp <= 0:
            continue
        stalls = {k[6:]: float(r[i] or 0) for k, i in ci.items() if k.startswith("stall_") and "Not Issued" not in k}
        top = sorted(stalls.items(), key=lambda kv: -kv[1])[:3]
        lines.append((smp, fname, r[0], r[1].strip()[:70], top))
    tot = sum(x[0] for x in lines) or 1.0
    for smp, f, ln, src, top in sorted(lines, key=lambda x: -x[0])[: args.top]:
        st = ", ".join(f"{k} {v / smp * 100:.0f}%" for k, v in top if v)
        print(f"{smp / tot * 100:5.1f}%  {f}:{ln:<5} {src:<70} [{st}]")


if __name__ == "__main__":
    main()
