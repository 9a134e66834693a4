"""Access to the host-glue extension (``csrc/hostglue.cpp``, built in-tree by
``_build``): compile_batch's Row-list packing and the Gebauer–Möller
criteria of ``update_pairs``.  Host code only; the package does not run
without it (no Python fallback)."""

from __future__ import annotations

from .errors import DeviceError

_MOD = None


def native():
    global _MOD
    if _MOD is None:
        try:
            from . import _hostglue as m
        except ImportError as e:
            raise DeviceError("paper_2601_06765_b200/_hostglue is not built (run __graft_entry__.build())") from e
        _MOD = m
    return _MOD
