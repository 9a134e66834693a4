"""Drop-in shim for an existing `fpgb` installation (SURVEY.md §8b option ii).

    import fpgb
    from paper_2601_06765_b200 import compat
    compat.install(fpgb)          # fpgb.groebner now runs the hot path on the GPU

`f4_step` (reference groebner.py:253-311) resolves `compile_batch`,
`csr_from_plan`, `psge_reduce` and `left_kernel` from the `fpgb.groebner`
module namespace (imported at groebner.py:32-50), so rebinding those four
names routes every F4 step of `f4_groebner`, `run_pipeline` and
`verify_instance` through the CUDA engine, including the kernel-solver
variant (`numeric="wiedemann"`, groebner.py:276-283).  The GPU functions accept the reference's own objects by duck
typing (rows with .shift/.basis_index/.role/.provenance, a SoaPolySet with
.ring/.exps/.coeff/.length/.offset) and return objects with the attributes
the reference reads (LayoutPlan .counters/.timings_ns/.dict_keys/.row_meta,
EchelonResult .nonpivot_rows/.pivot_rows/.rank/.zero_row_count/
.fill_generated).  `fpgb.bench.microbench` (and the CLI's copy) become the
GPU microbenchmarks of `paper_2601_06765_b200.bench`.  `uninstall(fpgb)`
restores the originals.
"""

from __future__ import annotations

from . import sparselin, symbolic

_SAVED: dict = {}
PATCHED = ("compile_batch", "csr_from_plan", "psge_reduce", "left_kernel")


# microbench (reference bench.py:244-312) is looked up in fpgb.bench and, by
# the CLI, in fpgb.cli (imported by name at cli.py:17)
MICRO_MODULES = ("bench", "cli")


def install(fpgb_pkg) -> None:
    from . import bench

    g = fpgb_pkg.groebner
    for name in PATCHED:
        _SAVED.setdefault(("groebner", name), getattr(g, name))
    g.compile_batch = symbolic.compile_batch
    g.csr_from_plan = sparselin.csr_from_plan
    g.psge_reduce = sparselin.psge_reduce
    g.left_kernel = sparselin.left_kernel
    for mod in MICRO_MODULES:
        m = getattr(fpgb_pkg, mod, None)
        if m is not None and hasattr(m, "microbench"):
            _SAVED.setdefault((mod, "microbench"), m.microbench)
            m.microbench = bench.microbench


def uninstall(fpgb_pkg) -> None:
    for (mod, name), fn in _SAVED.items():
        setattr(getattr(fpgb_pkg, mod), name, fn)
    _SAVED.clear()
