"""Pins for the oracle's ragged (CSR) clause against the (separately pinned) flat and segmented folds and numpy."""
import numpy as np
import pytest

import ipmgen
import oracle


def test_equal_rows_equal_segmented():
    rows, cols = 50, 37
    a = ipmgen.fill_host(ipmgen.Spec("int64", rows * cols, "random", seed=2))
    off = np.arange(rows + 1, dtype=np.int64) * cols
    for op in ["+", "^", "max", "&&"]:
        assert np.array_equal(oracle.reduce_ragged(op, a, off)[0], oracle.reduce_segmented(op, a, rows, cols)[0])


def test_single_row_is_flat_and_empty_rows_are_init():
    a = ipmgen.fill_host(ipmgen.Spec("float64", 1000, "random", seed=3))
    off = np.array([0, 1000], np.int64)
    assert oracle.reduce_ragged("+", a, off, init=2.0)[1][0] == oracle.reduce("+", a, init=2.0)[1]
    off = np.array([7, 7, 7, 7], np.int64)
    out, _ = oracle.reduce_ragged("min", a, off, init=5.0)
    assert list(out) == [5.0, 5.0, 5.0]
    out, _ = oracle.reduce_ragged("*", a, off)
    assert list(out) == [1.0, 1.0, 1.0]


@pytest.mark.parametrize("dt", ["int32", "int64"])
def test_random_degrees_vs_numpy(dt):
    d = ipmgen.degrees(3000, seed=5, cap=5000)
    off = ipmgen.offsets_from_degrees(d, start=11)
    a = ipmgen.fill_host(ipmgen.Spec(dt, int(off[-1]), "random", seed=6))
    T = np.int32 if dt == "int32" else np.int64
    out_add, _ = oracle.reduce_ragged("+", a, off)
    out_xor, _ = oracle.reduce_ragged("^", a, off)
    out_max, _ = oracle.reduce_ragged("max", a, off)
    for r in range(0, 3000, 7):
        seg = a[off[r]:off[r + 1]]
        assert out_add[r] == np.add.reduce(seg, dtype=T)
        assert out_xor[r] == np.bitwise_xor.reduce(seg)
        assert out_max[r] == (seg.max() if seg.size else np.iinfo(T).min)


def test_bad_offsets_rejected():
    with pytest.raises(ValueError):
        oracle.reduce_ragged("+", np.zeros(10), np.array([0, 5, 3], np.int64))
