"""Summarise tools/probe_batches.py output (per-batch elimination breakdown)."""
import json
import sys

rows = [json.loads(l) for l in open(sys.argv[1]) if l.startswith("{")]
rows.sort(key=lambda r: r["batch"])
tot = {}
for r in rows:
    t = r["top"]
    sw = sum(v[1] for k, v in t.items() if "sweep" in k or "win_build" in k)
    df = sum(v[1] for k, v in t.items() if "dense_forward" in k or "dense_fwd" in k or "dense_rref" in k)
    db = sum(v[1] for k, v in t.items() if "dense_back" in k)
    print(f"{r['batch']:2d} r={r['r']:5d} N={r['N']:5d} M={r['M']:8d} C={r['C']:5d} K={r['K']:5d} "
          f"rank={r['rank']:5d} sym={r['t_sym_ms']:.3f} elim={r['elim_ms']:.3f} sweep={sw:.3f} dfwd={df:.3f} "
          f"dback={db:.3f}")
    for k, v in (("sym", r["t_sym_ms"]), ("elim", r["elim_ms"]), ("sweep", sw), ("dfwd", df), ("dback", db)):
        tot[k] = round(tot.get(k, 0) + v, 3)
print(tot)
