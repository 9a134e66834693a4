"""Execution-policy shim of the reference bulk layer (``pkg/src/fpgb/bulk.py``).

The reference simulates data-parallel lanes sequentially (``ExecPolicy``,
:28-58) to prove its primitives are schedule independent.  On the device the
primitives (scan, radix sort, unique, compaction, lower_bound join) are
CUDA kernels inside ``compile_batch`` (``csrc/scan.cu``, ``csrc/radix.cu``,
``csrc/fbsp.cu``); they are deterministic by construction, so the policy is
accepted for API compatibility and does not change any output byte.
"""

from __future__ import annotations

from dataclasses import dataclass

MERGE_GRAIN = 4096


@dataclass(frozen=True)
class ExecPolicy:
    lanes: int = 1
    lane_order_seed: "int | None" = None


DEFAULT_POLICY = ExecPolicy()


def radix_pass_count(n_words: int) -> int:
    """Byte passes the reference radix sort runs for W-word keys (8 W)."""
    return 8 * n_words
