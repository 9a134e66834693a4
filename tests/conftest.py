import gzip
import json
import os
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
GOLDEN = os.path.join(ROOT, "tests", "golden")
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a CUDA device (run on the B200 box)")
    config.addinivalue_line("markers", "slow: long-running GPU parity (full-size configs)")


def load_golden(name):
    with open(os.path.join(GOLDEN, f"{name}.json")) as fh:
        return json.load(fh)


def load_snapshots(name):
    path = os.path.join(GOLDEN, f"{name}.snap.json.gz")
    if not os.path.exists(path):
        return {}
    with gzip.open(path, "rt") as fh:
        return {int(k): v for k, v in json.load(fh)["snapshots"].items()}


def state_from_snapshot(snap):
    """Rebuild a GroebnerState from a reference snapshot (SURVEY.md §8d replay)."""
    from paper_2601_06765_b200.groebner import GroebnerState, Pair, _make_pair
    from paper_2601_06765_b200.systems import parse_system

    ring, basis = parse_system(snap["basis"])
    st = GroebnerState(ring)
    for f in basis:
        st._push_basis(f)
    st.pairs = sorted([_make_pair(st, i, j) for i, j in snap["pairs"]], key=Pair.sort_tuple)
    return ring, st


@pytest.fixture(scope="session")
def built_lib():
    """Build (if stale) and load libf4b200.so — no GPU needed to load it."""
    from paper_2601_06765_b200 import _build, _capi

    _build.build()
    return _capi.load_library()


@pytest.fixture(scope="session")
def cuda():
    import torch

    if not torch.cuda.is_available():
        pytest.skip("no CUDA device")
    from paper_2601_06765_b200 import _build

    _build.build()
    return torch.device("cuda", 0)


@pytest.fixture
def force_option():
    """Force a path-selection option (f4b_ctx_set_option) on every engine for
    the duration of one test: force_option("dict_sort", 1)."""
    from paper_2601_06765_b200.engine import Engine

    touched = []

    def _set(name, value):
        Engine.force_option(name, value)
        touched.append(name)

    yield _set
    for name in touched:
        Engine.force_option(name, 0)
