"""CPU oracle — TEST INFRASTRUCTURE ONLY.

A NumPy restatement of the reference ``fpgb`` algorithms on the hot path
(symbolic preprocessing ``compile_batch`` and elimination ``psge_reduce``),
written against plain arrays so it runs anywhere (the reference itself lives
only in the build container).  Every function cites the reference file:line
it restates.

Pinning: ``tests/test_oracle_golden.py`` replays every F4 step of the
committed golden snapshots (``tests/golden/*.snap.json.gz``, produced by
running the real reference with ``tests/golden/make_golden.py``) through this
oracle and requires the reference's ``plan_digest`` and RREF digest byte for
byte.  Parity is therefore pinned to the reference, not to this restatement.

Rules (task contract): only ``tests/``, ``__graft_entry__.smoke()`` and the
``cpu_baseline`` / ``--impl reference`` legs of ``bench.py`` may import this
package, and only as the checker or the timed CPU baseline — never as a
product code path.  The product (``paper_2601_06765_b200``) never imports it.
"""

from .fbsp import compile_batch_arrays, plan_text, plan_sha256  # noqa: F401
from .psge import psge_arrays, rref_sha256  # noqa: F401
from .wiedemann import berlekamp_massey  # noqa: F401,E402
