"""Warp-stall samples of an `ncu --set full --import-source on` report per CUDA
source line (diagnostic).  The report's SASS view (addresses, samples, stall
reasons) is mapped to source lines through `nvdisasm -g` of the in-tree
library's cubins (the function with the same base name and instruction count).

usage: python tools/ncu_hot_lines.py report.ncu-rep kernel_regex [kernel_regex ...] > hot_lines.txt
"""
import csv
import glob
import io
import os
import re
import subprocess
import sys
import tempfile
from collections import defaultdict

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "paper_2601_06765_b200", "libf4b200.so")


def sass_functions():
    """{mangled name: [(offset, file:line), ...]} over every cubin in the library."""
    out = {}
    with tempfile.TemporaryDirectory() as d:
        subprocess.run(["cuobjdump", "-xelf", "all", LIB], cwd=d, capture_output=True, check=True)
        for cub in glob.glob(os.path.join(d, "*.cubin")):
            txt = subprocess.run(["nvdisasm", "-g", "-c", cub], capture_output=True, text=True).stdout
            fn, loc = None, None
            for line in txt.splitlines():
                m = re.match(r"\s*\.section\s+\.text\.(\S+),", line)
                if m:
                    fn, loc = m.group(1), None
                    out[fn] = []
                    continue
                m = re.search(r'//## File "([^"]+)", line (\d+)', line)
                if m:
                    loc = f"{os.path.basename(m.group(1))}:{m.group(2)}"
                    continue
                m = re.match(r"\s+/\*([0-9a-f]{4,})\*/", line)
                if m and fn is not None:
                    out[fn].append((int(m.group(1), 16), loc))
    return out


def main():
    rep, pats = sys.argv[1], sys.argv[2:]
    funcs = sass_functions()
    srcs = {}
    for path in glob.glob(os.path.join(ROOT, "paper_2601_06765_b200", "csrc", "*")):
        srcs[os.path.basename(path)] = open(path, errors="replace").read().splitlines()
    for pat in pats:
        txt = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{pat}", "-c", "1"],
                             capture_output=True, text=True).stdout
        lines = txt.splitlines()
        name = lines[0].split('","')[1].strip('",') if lines else pat
        rows = list(csv.reader(io.StringIO("\n".join(lines[1:]))))
        if len(rows) < 2:
            continue
        hdr = rows[0]
        ix = {c: i for i, c in enumerate(hdr)}
        body, last = [], -1
        for r in rows[1:]:  # one listing (the page may repeat it): stop where the addresses restart
            if len(r) != len(hdr) or not r[ix["Address"]].startswith("0x"):
                continue
            a = int(r[ix["Address"]], 16)
            if a <= last:
                break
            body.append(r)
            last = a
        base = re.sub(r"[<(].*", "", name.replace("void ", "")).split("::")[-1]
        cands = [f for f, ins in funcs.items() if base in f and len(ins) == len(body)]
        if not cands:
            print(f"## {name}: no matching function in {LIB}\n")
            continue
        ins = funcs[cands[0]]
        stall_cols = [c for c in hdr if c.startswith("stall_") and "(Not Issued)" not in c]
        per = defaultdict(lambda: [0, defaultdict(int)])
        total = 0
        for k, r in enumerate(body):
            s = int(float(r[ix["Warp Stall Sampling (All Samples)"]] or 0))
            if not s:
                continue
            loc = ins[k][1] or "?"
            per[loc][0] += s
            for c in stall_cols:
                per[loc][1][c[6:]] += int(float(r[ix[c]] or 0))
            total += s
        print(f"## {name.split('(')[0]} (warp-stall samples per source line, {total} samples)")
        for loc, (s, st) in sorted(per.items(), key=lambda kv: -kv[1][0])[:12]:
            f, _, ln = loc.partition(":")
            code = srcs.get(f, [])[int(ln) - 1].strip()[:70] if ln.isdigit() and f in srcs and int(ln) <= len(
                srcs[f]) else ""
            top = sorted(st.items(), key=lambda kv: -kv[1])[:3]
            why = ", ".join(f"{k} {100 * v // max(1, sum(st.values()))}%" for k, v in top)
            print(f" {100 * s / total:5.1f}%  {loc:24s} {code:70s} [{why}]")
        print()


if __name__ == "__main__":
    main()
