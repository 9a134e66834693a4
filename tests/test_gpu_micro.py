"""The reference microbenchmark primitives on the GPU (reference
tests/test_cli.py:58-67 `test_microbench_kinds`, bench.py:237-312), plus the
edge cases of the device entry points (f4b_dict_build / f4b_join_index /
f4b_mod_fma).  Exact integer results: byte equality with NumPy."""

import numpy as np
import pytest

from paper_2601_06765_b200 import errors
from paper_2601_06765_b200.bench import dict_build, join_index, microbench, mod_fma

pytestmark = pytest.mark.gpu


def _dev(a):
    import torch

    return torch.from_numpy(np.ascontiguousarray(a, dtype=np.uint64).view(np.int64)).cuda()


def _host(t):
    return t.cpu().numpy().view(np.uint64)


def test_microbench_kinds():
    d = microbench("dict_build", 5000, duplicate_rate=1.0, seed=1)
    assert d["unique_out"] == 1  # all keys equal
    assert d["reference_radix_passes"] == 16 and d["radix_passes"] in (1, 12)
    sizes = [10_000, 20_000]
    counts = [microbench("dict_build", s, 0.5, 2)["keys_total"] for s in sizes]
    assert counts == sizes
    r = microbench("row_assemble", 5000, seed=3)
    assert r["joins_per_s"] > 0 and r["bucket_imbalance"] >= 1.0
    f = microbench("mod_fma", 10_000, seed=4)
    assert f["updates_per_s.barrett"] > 0


@pytest.mark.parametrize("size,dup", [(1, 0.0), (2, 0.5), (6000, 0.99), (70_000, 0.5), (1 << 20, 0.9)])
def test_dict_build_matches_unique(size, dup):
    # small sizes take the single-CTA sort, large ones the one-sweep radix sort
    microbench("dict_build", size, duplicate_rate=dup, seed=size, reps=1)


@pytest.mark.parametrize("bits", [1, 17, 48, 63, 64])
def test_dict_build_word_widths(bits):
    rng = np.random.default_rng(bits)
    hi = (1 << bits) - 1
    for words in (1, 2):
        keys = rng.integers(0, hi, (30_000, words), dtype=np.uint64, endpoint=True)
        keys[::7] = keys[3]  # duplicates
        keys[0] = hi  # extreme values
        keys[1] = 0
        got = _host(dict_build(_dev(keys), words=words, key_bits=bits))
        assert np.array_equal(got.reshape(-1, words), np.unique(keys, axis=0))


def test_dict_build_rejects_wide_words():
    keys = np.array([[1, 1 << 48]], dtype=np.uint64)
    with pytest.raises(errors.PreconditionError):
        dict_build(_dev(keys), words=2, key_bits=48)


def test_join_index_missing_key():
    dic = np.array([[0, 1], [0, 5], [2, 0]], dtype=np.uint64)
    ok = np.array([[2, 0], [0, 1], [0, 5], [0, 5]], dtype=np.uint64)
    assert join_index(_dev(dic), _dev(ok)).cpu().tolist() == [2, 0, 1, 1]
    with pytest.raises(errors.MissingKeyError):
        join_index(_dev(dic), _dev(np.array([[0, 2]], dtype=np.uint64)))


@pytest.mark.parametrize("n", [1, 2, 3, 1001])
def test_mod_fma_odd_lengths(n):
    p = 32003
    rng = np.random.default_rng(n)
    a, b, c = (rng.integers(0, p, n, dtype=np.uint64) for _ in range(3))
    a[0] = b[0] = c[0] = p - 1
    got = _host(mod_fma(p, _dev(a), _dev(b), _dev(c)))
    assert np.array_equal(got, (c + a * b) % np.uint64(p))


@pytest.mark.parametrize("size,dup", [(5_000_000, 0.3), (3_000_000, 0.999), (21_000_000, 0.5)])
def test_dict_build_large(size, dup):
    # MSD bucket path up to 2^24 + 2^22 keys, the LSD sort above
    microbench("dict_build", size, duplicate_rate=dup, seed=7, reps=1)


@pytest.mark.parametrize("skew", ["bucket", "sub_bucket", "crowded_sub_bucket", "constant_top", "one_key"])
def test_dict_build_skewed_inputs(skew):
    """Skewed key distributions: a bucket above its shared-memory capacity or
    a sub-bucket above 1,024 keys falls back to the LSD sort; a crowded
    sub-bucket below that is ranked in place; constant leading bits move the
    bucket window down.  Always equal to np.unique."""
    rng = np.random.default_rng(5)
    n = 200_000
    keys = rng.integers(0, 1 << 48, (n, 2), dtype=np.uint64)
    if skew == "bucket":  # 6,000 distinct keys under one 13-bit bucket digit
        keys[: n // 2, 0] = 12345
        keys[: n // 2, 1] = rng.integers(0, 6000, n // 2, dtype=np.uint64)
    elif skew == "sub_bucket":  # 1,500 keys (400 distinct) under one sub-bucket digit
        keys[:1500, 0] = 777
        keys[:1500, 1] = rng.integers(0, 400, 1500, dtype=np.uint64)
    elif skew == "crowded_sub_bucket":  # 800 keys (300 distinct) under one sub-bucket digit
        keys[:800, 0] = 777
        keys[:800, 1] = rng.integers(0, 300, 800, dtype=np.uint64)
    elif skew == "constant_top":
        keys[:, 0] = 5
        keys[:, 1] &= np.uint64((1 << 20) - 1)
    else:
        keys[:] = keys[0]
    got = _host(dict_build(_dev(keys), words=2, key_bits=48)).reshape(-1, 2)
    assert np.array_equal(got, np.unique(keys, axis=0))


@pytest.mark.parametrize("lsd", [0, 1])
def test_dict_build_lsd_option_matches(force_option, lsd):
    """dict_build through the MSD bucket path and forced onto the LSD sort
    (f4b_ctx_set_option "dict_lsd") against np.unique."""
    force_option("dict_lsd", lsd)
    rng = np.random.default_rng(11)
    keys = rng.integers(0, 1 << 20, (200_000, 2), dtype=np.uint64)
    keys[::3] = keys[5]
    got = _host(dict_build(_dev(keys), words=2, key_bits=20)).reshape(-1, 2)
    assert np.array_equal(got, np.unique(keys, axis=0))


@pytest.mark.parametrize("words", [1, 2, 3, 4])
def test_join_index_unsorted_queries(words):
    # the warp narrows its search to [lb(min query), lb(max query)]: correct
    # for queries in any order, including keys in the middle and the extremes
    rng = np.random.default_rng(words)
    keys = rng.integers(0, 1 << 40, (100_000, words), dtype=np.uint64)
    dic = np.unique(keys, axis=0)
    q = dic[rng.integers(0, len(dic), 77_777)]
    q[0], q[-1] = dic[0], dic[-1]
    got = join_index(_dev(dic), _dev(q)).cpu().numpy()
    assert np.array_equal(dic[got], q)
