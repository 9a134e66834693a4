"""paper_2601_06765_b200 — a B200-native F4 hot path over F_p.

Drop-in for the reference package ``fpgb`` (arXiv 2601.06765) on its one hot
path: per F4 step, ``symbolic.compile_batch`` (FBSP symbolic preprocessing)
followed by ``sparselin.psge_reduce`` (exact F_p elimination), both executed
by hand-written sm_100a CUDA kernels in ``libf4b200.so`` behind the C ABI
``include/f4b200.h``.  Host modules keep the reference's public names and
semantics so its call sites and tests read unchanged.
"""

__version__ = "0.1.0"

from .fp import Backend, Domain, FieldModulus, FpElem  # noqa: E402
from .monomials import Ring, count_monomials  # noqa: E402
from .polynomials import Poly, poly_format, poly_parse  # noqa: E402

__all__ = ["Backend", "Domain", "FieldModulus", "FpElem", "Ring", "Poly", "count_monomials", "poly_parse",
           "poly_format", "__version__"]
