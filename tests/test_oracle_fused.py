"""Pins for the oracle's multi-variable clause (oracle.reduce_fused): closed forms,
exact rational brute force, orthogonality, and agreement with the (separately pinned) single-variable fold."""
import math
from fractions import Fraction

import numpy as np
import pytest

import ipmgen
import oracle

NPT = {"int32": np.int32, "int64": np.int64, "float32": np.float32, "float64": np.float64}
W = {"int32": 32, "int64": 64}


def fr(ld):
    return Fraction(*np.longdouble(ld).as_integer_ratio())


@pytest.mark.parametrize("dt", ["int32", "int64", "float64"])
def test_sum_sumsq_closed_forms(dt):
    for n in [1, 2, 10, 1000, 65_537]:
        x = np.arange(1, n + 1, dtype=NPT[dt])
        out, ld = oracle.reduce_fused("sum_sumsq", x)
        s1, s2 = n * (n + 1) // 2, n * (n + 1) * (2 * n + 1) // 6
        if dt.startswith("int"):
            m = (1 << W[dt]) - 1
            assert int(out[0]) & m == s1 & m and int(out[1]) & m == s2 & m
        else:
            assert fr(ld[0]) == s1 and fr(ld[1]) == s2


def test_dot_closed_forms_and_orthogonality():
    n = 4096
    i = np.arange(n, dtype=np.float64)
    assert oracle.reduce_fused("dot", i, np.ones(n))[1][0] == n * (n - 1) // 2
    assert oracle.reduce_fused("dot", i, i)[1][0] == (n - 1) * n * (2 * n - 1) // 6
    # rows of a Sylvester-Hadamard matrix are orthogonal: every dot product is exactly 0
    H = np.array([[1.0]])
    while H.shape[0] < 256:
        H = np.block([[H, H], [H, -H]])
    for a, b in [(1, 2), (5, 200), (17, 255)]:
        for dt in ("float32", "float64"):
            assert oracle.reduce_fused("dot", H[a].astype(dt), H[b].astype(dt))[1][0] == 0
    # int32 dot wraps mod 2^32
    x = np.full(70_000, 1 << 16, np.int32)
    assert int(oracle.reduce_fused("dot", x, x)[0][0]) == 0           # 70000 * 2^32 ≡ 0 mod 2^32


@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_exact_rational_bruteforce(dt):
    rng = np.random.default_rng(7)
    for n in range(0, 17):
        x = (rng.standard_normal(n) * 8).astype(NPT[dt])
        y = (rng.standard_normal(n) * 8).astype(NPT[dt])
        init = np.array([0.5, -1.25], NPT[dt])
        _, ld = oracle.reduce_fused("sum_sumsq", x, init=init)
        ex1 = Fraction(0.5) + sum((Fraction(float(v)) for v in x), Fraction(0))
        ex2 = Fraction(-1.25) + sum((Fraction(float(v)) ** 2 for v in x), Fraction(0))
        assert abs(fr(ld[0]) - ex1) <= abs(ex1) * Fraction(1, 2**60) + Fraction(1, 2**100)
        assert abs(fr(ld[1]) - ex2) <= abs(ex2) * Fraction(1, 2**58) + Fraction(1, 2**100)
        _, ld = oracle.reduce_fused("dot", x, y)
        exd = sum((Fraction(float(a)) * Fraction(float(b)) for a, b in zip(x, y)), Fraction(0))
        tol = sum((abs(Fraction(float(a)) * Fraction(float(b))) for a, b in zip(x, y)), Fraction(0))
        assert abs(fr(ld[0]) - exd) <= tol * Fraction(1, 2**58) + Fraction(1, 2**100)


@pytest.mark.parametrize("dt", ["int32", "int64", "float32", "float64"])
def test_agrees_with_single_variable_folds(dt):
    spec = ipmgen.Spec(dt, 50_003, "signed" if dt.startswith("float") else "random", seed=3)
    x = ipmgen.fill_host(spec)
    out, ld = oracle.reduce_fused("stats", x)
    assert out[0] == oracle.reduce("+", x)[0]
    assert out[2] == oracle.reduce("min", x)[0] and out[3] == oracle.reduce("max", x)[0]
    mm, _ = oracle.reduce_fused("minmax", x)
    assert mm[0] == out[2] and mm[1] == out[3]
    if dt.startswith("int"):  # Σx² wraps: compare with Python big integers
        m = (1 << W[dt]) - 1
        assert int(out[1]) & m == sum(int(v) * int(v) for v in x) & m
    else:                     # exact squares: math.fsum of the float64 squares of float32 data is exact-ish
        sq = x.astype(np.float64) ** 2
        ex = math.fsum(sq) if dt == "float32" else float(sum(Fraction(float(v)) ** 2 for v in x[:2000]))
        if dt == "float32":
            assert abs(float(ld[1]) - ex) <= 2 * math.ulp(ex)


def test_init_and_empty():
    x = np.zeros(0, np.float64)
    out, _ = oracle.reduce_fused("stats", x, init=np.array([1.0, 2.0, 3.0, 4.0]))
    assert list(out) == [1.0, 2.0, 3.0, 4.0]
    out, _ = oracle.reduce_fused("minmax", x)
    assert out[0] == np.inf and out[1] == -np.inf
    out, _ = oracle.reduce_fused("sum_sumsq", np.array([3], np.int32), init=np.array([10, 20], np.int32))
    assert list(out) == [13, 29]
