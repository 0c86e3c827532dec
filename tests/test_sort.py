"""The K2 HBM sort (csrc/mk_sort.cuh, mk_sort_pairs_u64): a stable radix
sort on the low ``bits`` key bits must equal numpy's stable argsort on every
input shape the race sweeps produce -- empty, single, tile-boundary sizes,
heavy duplicates (many accesses of one granule), already ordered keys (a
coalesced store: no pass runs), ordered keys forced through every pass, and
a ragged last tile."""
import numpy as np
import pytest

TILE = 4096


@pytest.fixture(scope="module")
def engine():
    from paper_2603_24595_b200.native import Engine

    e = Engine(0)
    yield e
    e.close()


def _check(engine, keys, vals, bits, force=False):
    mask = np.uint64((1 << bits) - 1) if bits < 64 else np.uint64(0xFFFFFFFFFFFFFFFF)
    order = np.argsort(keys & mask, kind="stable")
    got = engine.sort_pairs(keys.copy(), vals.copy(), bits=bits, force=force)
    assert np.array_equal(got["keys"], keys[order])
    assert np.array_equal(got["vals"], vals[order])
    return got


@pytest.mark.gpu
@pytest.mark.parametrize("n", [0, 1, 2, 31, 2047, 2048, 2049, TILE - 1, TILE, TILE + 1, 3 * TILE + 17, 1 << 20])
@pytest.mark.parametrize("bits", [8, 26, 31, 64])
def test_random_keys(engine, n, bits):
    rng = np.random.default_rng(n * 131 + bits)
    hi = (1 << bits) if bits < 64 else None
    keys = (rng.integers(0, hi, n, dtype=np.uint64) if hi
            else rng.integers(0, 2 ** 63, n, dtype=np.uint64) * np.uint64(2) + np.uint64(1))
    vals = np.arange(n, dtype=np.uint64)
    _check(engine, keys, vals, bits)


@pytest.mark.gpu
def test_heavy_duplicates_are_stable(engine):
    rng = np.random.default_rng(7)
    n = 5 * TILE + 123
    keys = rng.integers(0, 5, n, dtype=np.uint64) << np.uint64(20)
    vals = rng.integers(0, 2 ** 63, n, dtype=np.uint64)
    got = _check(engine, keys, vals, 26)
    assert got["passes"] == 1          # only the digit that varies moves tuples


@pytest.mark.gpu
def test_ordered_keys_skip_or_force(engine):
    n = 7 * TILE + 5
    keys = np.repeat(np.arange(n // 4 + 1, dtype=np.uint64), 4)[:n]
    vals = np.arange(n, dtype=np.uint64)
    assert _check(engine, keys, vals, 31)["passes"] == 0
    assert _check(engine, keys, vals, 31, force=True)["passes"] == 4


@pytest.mark.gpu
def test_large_unsorted_matches_numpy(engine):
    rng = np.random.default_rng(11)
    n = 24_000_000
    keys = rng.integers(0, 1 << 31, n, dtype=np.uint64)
    vals = np.arange(n, dtype=np.uint64)
    _check(engine, keys, vals, 31)
