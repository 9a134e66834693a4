"""One-off probe: the REAL reference (installed in baseline/_ref) with its hot
path rebound to the GPU engine via compat.install; digest must equal the
reference's own CPU digest (tests/golden)."""
import hashlib, json, os, sys, time
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "baseline", "_ref"))
import fpgb
from fpgb.bench import PipelineConfig, make_instance, run_pipeline
from paper_2601_06765_b200 import compat

compat.install(fpgb)
for fam, n, p, name in (("cyclic", 6, 32003, "cyclic6_p32003"), ("katsura", 6, 32003, "katsura6_p32003"),
                        ("cyclic", 7, 65521, "cyclic7_p65521")):
    cfg = PipelineConfig()
    ring, polys, desc = make_instance(fam, cfg, n=n, p=p)
    t0 = time.time()
    rep, text, basis = run_pipeline(ring, polys, cfg, desc)
    want = json.load(open(os.path.join(ROOT, "tests", "golden", f"{name}.json")))["final_sha256"]
    print(name, "fpgb.run_pipeline with GPU hot path:", rep.digest == want, f"{time.time()-t0:.1f}s",
          "numeric_core_ns", rep.totals["numeric_core_ns"])
compat.uninstall(fpgb)
