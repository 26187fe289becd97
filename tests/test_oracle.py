"""Pins for the CPU oracle (oracle/ipm_oracle.c) against things other than itself.

Every pin cites what fixes it: a worked example in the SPEC.md written from the paper, a closed form, a
theorem, a library routine that computes the same definition (numpy ufunc.reduce with the wrapping dtype,
math.fsum, fractions.Fraction, Python big integers), or brute force on tiny inputs. Each group is chosen
so a plausible mistake in the oracle (a dropped term, a wrong sign or index, signed/unsigned confusion,
32-bit truncation, a missing init, a non-normalised logical value, plain instead of compensated summation)
fails at least one of them.
"""
import itertools
import math
import struct
from fractions import Fraction

import numpy as np
import pytest

import ipmgen
import oracle

INT = ["int32", "int64"]
FLT = ["float32", "float64"]
W = {"int32": 32, "int64": 64}
NPT = {"int32": np.int32, "int64": np.int64, "float32": np.float32, "float64": np.float64}


def fr(ld):
    """exact rational value of a long double (no detour through double)"""
    return Fraction(*np.longdouble(ld).as_integer_ratio())


def u(x, dt):
    """unsigned w-bit reading of an integer result"""
    return int(x) & ((1 << W[dt]) - 1)


# --------------------------------------------------------------------------- worked examples

def test_spec_worked_sum_1_to_1024():
    # SPEC.md:320 / :404 / :490 — reduction(+:s) over i=1..1024 -> 524800 (= n(n+1)/2)
    for dt in INT:
        v, ld = oracle.reduce("+", np.arange(1, 1025, dtype=NPT[dt]))
        assert int(v) == 524800 and ld == 524800


def test_spec_worked_max():
    # reduction(max:m) over {3,-1,7} -> 7
    for dt in INT + FLT:
        assert oracle.reduce("max", np.array([3, -1, 7], dtype=NPT[dt]))[0] == 7
        assert oracle.reduce("min", np.array([3, -1, 7], dtype=NPT[dt]))[0] == -1


def test_spec_float_sum_4096_uniform_30_seeds():
    # SPEC.md:322 / :490 — + over 4096 uniform floats in [0,1000], 30 seeds, within 1e-5 of the sequential
    # fold. We pin tighter: math.fsum is the correctly rounded exact sum, the oracle must agree to ~1e-15.
    for seed in range(30):
        a = np.random.default_rng(seed).uniform(0, 1000, 4096).astype(np.float32)
        _, ld = oracle.reduce("+", a)
        exact = math.fsum(float(x) for x in a)
        assert abs(float(ld) - exact) <= 1e-15 * exact


# --------------------------------------------------------------------------- integer +, closed forms

@pytest.mark.parametrize("dt", INT)
def test_int_sum_closed_form_wraps(dt):
    # Σ_{i=1}^{n} i = n(n+1)/2, reduced mod 2^w (reading R3: two's-complement wrap)
    for n in [1, 2, 1000, 1 << 16, 1 << 20, 3 * (1 << 18) + 7]:
        v, _ = oracle.reduce("+", np.arange(1, n + 1, dtype=NPT[dt]))
        assert u(v, dt) == (n * (n + 1) // 2) % (1 << W[dt])
    # n = 2^20 int32 -> 2^19 * (2^20 + 1) mod 2^32 = 524288 (SURVEY.md §8(c) pin table)
    if dt == "int32":
        assert oracle.reduce("+", np.arange(1, (1 << 20) + 1, dtype=np.int32))[0] == 524288


@pytest.mark.parametrize("dt", INT)
def test_int_sum_random_vs_bigint_and_numpy(dt):
    a = ipmgen.fill_host(ipmgen.Spec(dt, 100_003, "random", seed=7))
    v, _ = oracle.reduce("+", a)
    assert u(v, dt) == sum(int(x) for x in a) % (1 << W[dt])                      # Python big ints
    assert int(v) == int(np.add.reduce(a, dtype=NPT[dt]))                          # numpy, wrapping dtype


def test_sum_of_ones_is_n():
    # exactly-once: Σ 1 over n elements = n (SPEC.md:343 analogue)
    for dt in INT + FLT:
        for n in [0, 1, 255, 256, 257, 1000, 1024, 4097]:
            assert oracle.reduce("+", np.ones(n, dtype=NPT[dt]))[0] == n


# --------------------------------------------------------------------------- integer *

def test_int_product_factorials():
    f = lambda n: math.factorial(n)
    assert oracle.reduce("*", np.arange(1, 13, dtype=np.int32))[0] == 479001600              # 12!
    assert u(oracle.reduce("*", np.arange(1, 14, dtype=np.int32))[0], "int32") == 1932053504   # 13! mod 2^32
    assert u(oracle.reduce("*", np.arange(1, 14, dtype=np.int32))[0], "int32") == f(13) % 2**32
    assert oracle.reduce("*", np.arange(1, 21, dtype=np.int64))[0] == 2432902008176640000     # 20!
    # 2-adic valuation: v2(34!) = 32 -> 34! ≡ 0 mod 2^32 but 33! is not; v2(66!) = 64 for 2^64
    assert oracle.reduce("*", np.arange(1, 35, dtype=np.int32))[0] == 0
    assert u(oracle.reduce("*", np.arange(1, 34, dtype=np.int32))[0], "int32") == f(33) % 2**32 != 0
    assert oracle.reduce("*", np.arange(1, 67, dtype=np.int64))[0] == 0
    assert u(oracle.reduce("*", np.arange(1, 66, dtype=np.int64))[0], "int64") == f(65) % 2**64 != 0


def test_int_product_odd_residues_generalised_wilson():
    # Gauss: the product of all odd residues mod 2^k is 1 for k >= 3. With int32 wrap (mod 2^32) this needs
    # all 2^31 odd words (a GPU-size test); here we pin the k = 32 statement's structure on int64 by taking
    # the odd residues of 2^k inside an int64 fold and reducing mod 2^k.
    for k in [3, 8, 16, 20]:
        a = np.arange(1, 1 << k, 2, dtype=np.int64)
        v, _ = oracle.reduce("*", a)
        assert u(v, "int64") % (1 << k) == 1


@pytest.mark.parametrize("dt", INT)
def test_int_product_random_odd_vs_bigint_numpy(dt):
    a = ipmgen.fill_host(ipmgen.Spec(dt, 20_001, "odd", seed=3))
    v, _ = oracle.reduce("*", a)
    assert u(v, dt) == math.prod(int(x) for x in a) % (1 << W[dt])
    assert int(v) == int(np.multiply.reduce(a, dtype=NPT[dt]))
    assert u(v, dt) % 2 == 1  # a product of units is a unit


# --------------------------------------------------------------------------- max / min

@pytest.mark.parametrize("dt", INT + FLT)
def test_max_min_permutation(dt):
    n = 5000
    a = np.random.default_rng(1).permutation(n).astype(NPT[dt])
    assert oracle.reduce("max", a)[0] == n - 1
    assert oracle.reduce("min", a)[0] == 0


@pytest.mark.parametrize("dt", INT)
def test_int_max_min_signed(dt):
    # signed compare: an unsigned compare would call -1 the maximum
    a = np.array([-1, 5, -7], dtype=NPT[dt])
    assert oracle.reduce("max", a)[0] == 5 and oracle.reduce("min", a)[0] == -7
    info = np.iinfo(NPT[dt])
    # extremes equal to the identities
    assert oracle.reduce("max", np.array([info.min] * 3, dtype=NPT[dt]))[0] == info.min
    assert oracle.reduce("min", np.array([info.max] * 3, dtype=NPT[dt]))[0] == info.max
    assert oracle.identity("max", dt) == info.min and oracle.identity("min", dt) == info.max
    b = ipmgen.fill_host(ipmgen.Spec(dt, 30_000, "random", seed=11))
    assert oracle.reduce("max", b)[0] == np.max(b) and oracle.reduce("min", b)[0] == np.min(b)


@pytest.mark.parametrize("dt", FLT)
def test_float_max_min_planted_extreme(dt):
    # signed dyadic data in [-1024,1024) with a planted +1024 / -1025 (outside the range -> unique extreme)
    s = ipmgen.Spec(dt, 50_000, "signed", seed=5, plant="value", nplant=1, plant_param=1024.0)
    assert oracle.reduce("max", ipmgen.fill_host(s))[0] == 1024.0
    s = ipmgen.Spec(dt, 50_000, "signed", seed=5, plant="value", nplant=1, plant_param=-1025.0)
    assert oracle.reduce("min", ipmgen.fill_host(s))[0] == -1025.0
    b = ipmgen.fill_host(ipmgen.Spec(dt, 50_000, "signed", seed=9))
    assert oracle.reduce("max", b)[0] == np.max(b) and oracle.reduce("min", b)[0] == np.min(b)


def bits(x, dt):
    return struct.unpack("<I", struct.pack("<f", x))[0] if dt == "float32" else \
        struct.unpack("<Q", struct.pack("<d", x))[0]


@pytest.mark.parametrize("dt", FLT)
def test_float_max_min_ieee754_2019(dt):
    # reading R10: IEEE 754-2019 maximum/minimum: -0 < +0 in either order; NaN propagates (canonical qNaN)
    T = NPT[dt]
    for a in ([-0.0, 0.0], [0.0, -0.0]):
        assert bits(oracle.reduce("max", np.array(a, T))[0], dt) == bits(0.0, dt)
        assert bits(oracle.reduce("min", np.array(a, T))[0], dt) == bits(-0.0, dt)
    qnan = 0x7FC00000 if dt == "float32" else 0x7FF8000000000000
    for a in ([1.0, np.nan, 2.0], [np.nan], [-np.inf, -np.nan]):
        assert bits(oracle.reduce("max", np.array(a, T))[0], dt) == qnan
        assert bits(oracle.reduce("min", np.array(a, T))[0], dt) == qnan
    # identities (reading R2): -inf / +inf
    assert oracle.identity("max", dt) == -np.inf and oracle.identity("min", dt) == np.inf
    assert oracle.reduce("max", np.array([-np.inf], T))[0] == -np.inf


# --------------------------------------------------------------------------- bitwise

def xor_0_to(m):
    # XOR of 0..m = [m, 1, m+1, 0][m mod 4]
    return [m, 1, m + 1, 0][m % 4]


@pytest.mark.parametrize("dt", INT)
def test_bitwise_closed_forms(dt):
    for n in [1, 2, 3, 4, 5, 1000, 1 << 16, (1 << 20), 12345]:
        a = np.arange(n, dtype=NPT[dt])
        assert oracle.reduce("^", a)[0] == xor_0_to(n - 1)
    for k in [1, 5, 16, 20]:
        assert oracle.reduce("|", np.arange(1 << k, dtype=NPT[dt]))[0] == (1 << k) - 1
    assert oracle.reduce("^", np.arange(1 << 20, dtype=NPT[dt]))[0] == 0  # 2^20 -> 0
    # AND: all-ones background with planted single-bit clears -> ~(OR of the cleared bits)
    s = ipmgen.Spec(dt, 40_000, "allbits", seed=2, plant="clearbit", nplant=6)
    a = ipmgen.fill_host(s)
    cleared = 0
    for p in set(ipmgen.plant_positions(s)):
        cleared |= (~int(a[p])) & ((1 << W[dt]) - 1)
    assert u(oracle.reduce("&", a)[0], dt) == ((1 << W[dt]) - 1) & ~cleared
    # OR: zero background with planted single-bit words; bit 63 / bit 31 reachable (truncation check)
    z = np.zeros(100, dtype=NPT[dt])
    z[17] = np.array(1 << (W[dt] - 1), dtype=np.uint64).astype(NPT[dt])
    z[40] = 4
    assert u(oracle.reduce("|", z)[0], dt) == (1 << (W[dt] - 1)) | 4
    # XOR of duplicated pairs -> 0
    r = ipmgen.fill_host(ipmgen.Spec(dt, 5000, "random", seed=4))
    assert oracle.reduce("^", np.concatenate([r, r[::-1]]))[0] == 0


@pytest.mark.parametrize("dt", INT)
def test_bitwise_vs_numpy(dt):
    a = ipmgen.fill_host(ipmgen.Spec(dt, 77_777, "random", seed=21))
    assert oracle.reduce("&", a)[0] == np.bitwise_and.reduce(a)
    assert oracle.reduce("|", a)[0] == np.bitwise_or.reduce(a)
    assert oracle.reduce("^", a)[0] == np.bitwise_xor.reduce(a)


def test_bitwise_illegal_on_floats():
    # C forbids & | ^ on floating types (reading R5)
    for op in "&|^":
        for dt in FLT:
            assert not oracle.legal(op, dt)
            with pytest.raises(ValueError):
                oracle.reduce(op, np.zeros(3, NPT[dt]))
    assert sum(oracle.legal(op, dt) for op in oracle.OPS for dt in oracle.DTYPES) == 30


# --------------------------------------------------------------------------- logical && ||

@pytest.mark.parametrize("dt", INT + FLT)
def test_logical(dt):
    T = NPT[dt]
    nz = ipmgen.fill_host(ipmgen.Spec(dt, 10_000, "nonzero", seed=8))
    assert oracle.reduce("&&", nz)[0] == 1
    nz0 = nz.copy(); nz0[6543] = 0
    assert oracle.reduce("&&", nz0)[0] == 0
    z = np.zeros(10_000, T)
    assert oracle.reduce("||", z)[0] == 0
    z1 = z.copy(); z1[9999] = 3
    assert oracle.reduce("||", z1)[0] == 1
    # numpy's logical reductions compute the same definition
    assert oracle.reduce("&&", nz0)[0] == np.logical_and.reduce(nz0)
    assert oracle.reduce("||", z1)[0] == np.logical_or.reduce(z1)
    # the original var value participates and is normalised to 0/1 (readings R1, R5)
    assert oracle.reduce("&&", nz, init=0)[0] == 0
    assert oracle.reduce("||", z, init=5)[0] == 1
    assert oracle.reduce("&&", np.zeros(0, T), init=7)[0] == 1
    assert oracle.identity("&&", dt) == 1 and oracle.identity("||", dt) == 0


def test_logical_truthiness_edges():
    # int64: 1<<32 and 1<<63 are true (a 32-bit truncation would call them false)
    assert oracle.reduce("&&", np.array([1 << 32, 1 << 62, -(1 << 63)], np.int64))[0] == 1
    assert oracle.reduce("||", np.array([0, 1 << 33, 0], np.int64))[0] == 1
    # floats: -0.0 is false, NaN is true (C truthiness)
    for T in (np.float32, np.float64):
        assert oracle.reduce("||", np.array([-0.0, 0.0], T))[0] == 0
        assert oracle.reduce("&&", np.array([1.0, -0.0], T))[0] == 0
        assert oracle.reduce("&&", np.array([np.nan, 2.0], T))[0] == 1
        assert oracle.reduce("||", np.array([0.0, np.nan], T))[0] == 1


# --------------------------------------------------------------------------- float +

@pytest.mark.parametrize("dt", FLT)
def test_float_sum_integer_valued_closed_form(dt):
    # a_i = i mod 1024 -> Σ = (n/1024) * 523776 exactly (SURVEY.md §8(c) pin table)
    for n in [1024, 1 << 20, 5 * 1024]:
        a = ipmgen.fill_host(ipmgen.Spec(dt, n, "mod", param=1024))
        v, ld = oracle.reduce("+", a)
        assert ld == (n // 1024) * 523776 and v == (n // 1024) * 523776


def test_float_sum_needs_compensation():
    # reading R7: a plain long double fold loses the 1 (ulp(1e20) = 8 in 64-bit mantissa); Neumaier keeps it
    assert oracle.reduce("+", np.array([1e20, 1.0, -1e20]))[1] == 1
    assert oracle.reduce("+", np.array([1.0, 1e100, 1.0, -1e100]))[1] == 2


@pytest.mark.parametrize("dt", FLT)
def test_float_sum_vs_fsum_and_fraction(dt):
    a = ipmgen.fill_host(ipmgen.Spec(dt, 200_000, "signed", seed=12))
    _, ld = oracle.reduce("+", a)
    ex = math.fsum(float(x) for x in a)            # correctly rounded in double
    assert abs(float(ld) - ex) <= 2 * math.ulp(ex)
    # tiny random fp64 with wildly different magnitudes vs the exact rational sum
    rng = np.random.default_rng(3)
    for _ in range(50):
        b = (rng.standard_normal(12) * 10.0 ** rng.integers(-8, 9, 12)).astype(NPT[dt])
        exact = sum(Fraction(float(x)) for x in b)
        _, ld = oracle.reduce("+", b)
        assert abs(fr(ld) - exact) <= abs(exact) * Fraction(1, 2**50) + Fraction(1, 2**200)


@pytest.mark.parametrize("dt", FLT)
def test_float_sum_init_participates(dt):
    a = np.array([1.5, 2.25], NPT[dt])
    assert oracle.reduce("+", a, init=10.0)[0] == 13.75
    assert oracle.reduce("+", np.zeros(0, NPT[dt]), init=-2.5)[0] == -2.5


# --------------------------------------------------------------------------- float *

@pytest.mark.parametrize("dt", FLT)
def test_float_product_planted_factors_exact(dt):
    # ±1 background with 64 planted factors in [0.5,2) (reading R8): exact value = sign × Π planted
    s = ipmgen.Spec(dt, 300_000, "signs", seed=13, plant="factor", nplant=64)
    a = ipmgen.fill_host(s)
    exact = Fraction(1)
    for x in a:
        if x != 1.0:
            exact *= Fraction(float(x))
    v, ld = oracle.reduce("*", a)
    assert abs(fr(ld) - exact) <= abs(exact) * Fraction(64, 2**63)
    assert abs(float(v) - float(exact)) <= abs(float(exact)) * (2e-7 if dt == "float32" else 1e-15)


@pytest.mark.parametrize("dt", FLT)
def test_float_product_powers_of_two(dt):
    e = np.random.default_rng(4).integers(-3, 4, 200)
    a = (2.0 ** e).astype(NPT[dt])
    assert oracle.reduce("*", a)[1] == 2.0 ** int(e.sum())
    assert oracle.reduce("*", np.array([-1.0, -1.0, -1.0], NPT[dt]))[0] == -1.0


# --------------------------------------------------------------------------- empty, size-1, init

@pytest.mark.parametrize("op,dt", [(o, d) for o in oracle.OPS for d in oracle.DTYPES if oracle.legal(o, d)])
def test_empty_and_single(op, dt):
    T = NPT[dt]
    # n = 0 -> the var keeps its value, normalised to 0/1 for && ||
    init = T(3)
    v, _ = oracle.reduce(op, np.zeros(0, T), init=init)
    assert v == (1 if op in ("&&", "||") else 3)
    # n = 1 with identity init -> a[0] (normalised for && ||)
    v, _ = oracle.reduce(op, np.array([6], T))
    assert v == (1 if op in ("&&", "||") else 6)
    # init = identity -> the identity bits come back
    ident = oracle.identity(op, dt)
    assert np.array(oracle.reduce(op, np.zeros(0, T), init=ident)[0]).tobytes() == np.array(ident).tobytes()


# --------------------------------------------------------------------------- brute force on tiny inputs

def brute_int(op, xs, dt, init):
    m = (1 << W[dt]) - 1
    s = lambda v: v - (1 << W[dt]) if v >> (W[dt] - 1) else v
    r = int(init) & m
    if op in ("&&", "||"):
        r = int(r != 0)  # the var's value enters as a truth value
    for x in xs:
        x = int(x) & m
        if op == "+": r = (r + x) & m
        elif op == "*": r = (r * x) & m
        elif op == "max": r = x if s(x) > s(r) else r
        elif op == "min": r = x if s(x) < s(r) else r
        elif op == "&": r &= x
        elif op == "|": r |= x
        elif op == "^": r ^= x
        elif op == "&&": r = int(r != 0 and x != 0)
        elif op == "||": r = int(r != 0 or x != 0)
    return r


@pytest.mark.parametrize("dt", INT)
@pytest.mark.parametrize("op", list(oracle.OPS))
def test_bruteforce_int(op, dt):
    rng = np.random.default_rng(hash((op, dt)) & 0xFFFF)
    for n in range(0, 17):
        for _ in range(4):
            hi = np.iinfo(NPT[dt])
            xs = rng.integers(hi.min, hi.max, n, dtype=NPT[dt], endpoint=True)
            if op in ("&&", "||"):
                xs[rng.random(n) < 0.3] = 0
            init = rng.integers(hi.min, hi.max, dtype=NPT[dt], endpoint=True)
            v, _ = oracle.reduce(op, xs, init=init)
            assert u(v, dt) == brute_int(op, xs, dt, init)


@pytest.mark.parametrize("dt", FLT)
def test_bruteforce_float_sum_prod(dt):
    rng = np.random.default_rng(99)
    for n in range(0, 17):
        xs = (rng.standard_normal(n) * 4).astype(NPT[dt])
        init = NPT[dt](rng.standard_normal())
        ex_s = Fraction(float(init)) + sum((Fraction(float(x)) for x in xs), Fraction(0))
        ex_p = Fraction(float(init))
        for x in xs:
            ex_p *= Fraction(float(x))
        _, s = oracle.reduce("+", xs, init=init)
        _, p = oracle.reduce("*", xs, init=init)
        assert abs(fr(s) - ex_s) <= abs(ex_s) * Fraction(1, 2**52) + Fraction(1, 2**80)
        assert abs(fr(p) - ex_p) <= abs(ex_p) * Fraction(1, 2**50)


@pytest.mark.parametrize("dt", INT)
@pytest.mark.parametrize("op", list(oracle.OPS))
def test_exact_ops_order_and_split_invariant(op, dt):
    # For exact ops the two-level scheme reaches the same bits for any grouping: reorder the
    # elements, or fold two halves separately and merge the partials into the original var.
    rng = np.random.default_rng(5)
    xs = ipmgen.fill_host(ipmgen.Spec(dt, 16, "odd" if op == "*" else "random", seed=31))
    if op in ("&&", "||"):
        xs[[2, 9]] = 0
    init = NPT[dt](12345)
    ref = oracle.reduce(op, xs, init=init)[0]
    for perm in itertools.islice(itertools.permutations(range(16)), 0, 2000, 97):
        assert oracle.reduce(op, xs[list(perm)], init=init)[0] == ref
    for k in range(17):
        p1 = oracle.reduce(op, xs[:k])[0]
        p2 = oracle.reduce(op, xs[k:])[0]
        assert oracle.reduce(op, np.array([p1, p2], NPT[dt]), init=init)[0] == ref
    del rng


# --------------------------------------------------------------------------- segmented

@pytest.mark.parametrize("dt", INT + FLT)
def test_segmented_row_constant_closed_form(dt):
    rows, cols = 300, 77
    a = np.repeat((np.arange(rows) % 1024)[:, None], cols, axis=1).astype(NPT[dt])
    out, ld = oracle.reduce_segmented("+", a.ravel(), rows, cols)
    assert np.array_equal(out, (cols * (np.arange(rows) % 1024)).astype(NPT[dt]))


def test_segmented_stride_and_init():
    rows, cols, stride = 50, 13, 20
    a = np.full(rows * stride, 1e30, np.float64)  # poison in the gaps: must never be read
    body = np.random.default_rng(0).integers(-50, 50, (rows, cols)).astype(np.float64)
    a.reshape(rows, stride)[:, :cols] = body
    out, _ = oracle.reduce_segmented("+", a, rows, cols, stride, init=0.5)
    assert np.array_equal(out, body.sum(axis=1) + 0.5)  # integer-valued: numpy's sum is exact here
    out, _ = oracle.reduce_segmented("max", a, rows, cols, stride)
    assert np.array_equal(out, body.max(axis=1))
    # cols = 0 -> every row is the init (identity when absent)
    out, _ = oracle.reduce_segmented("+", a, rows, 0, stride, init=4.0)
    assert np.all(out == 4.0)
    out, _ = oracle.reduce_segmented("max", a, rows, 0, stride)
    assert np.all(out == -np.inf)


def test_streaming_fold_equals_whole_fold():
    s = ipmgen.Spec("float32", 1_000_003, "random", seed=1)
    whole = oracle.reduce("+", ipmgen.fill_host(s))
    streamed = oracle.reduce_spec("+", s, chunk=65_536)
    assert whole[1] == streamed[1] and whole[0] == streamed[0]


# --------------------------------------------------------------------------- split fold (ora_merge), the C5 oracle

@pytest.mark.parametrize("dt", INT)
def test_split_merge_closed_forms_int(dt):
    # Σ_{i=1}^{n} i mod 2^w (closed form) through 7 pieces on 3 threads, and the generalised Wilson theorem
    # (∏ of all odd residues mod 2^k is 1 for k >= 3) through pieces folded separately and merged
    n = 3_000_001
    s = ipmgen.Spec(dt, n, "iota", param=1)
    v, ld, _ = oracle.reduce_spec_split("+", s, pieces=7, threads=3, chunk=100_000)
    assert u(v, dt) == (n * (n + 1) // 2) % (1 << W[dt])
    odd = np.arange(1, 1 << 20, 2, dtype=np.int64)          # all odd residues mod 2^20
    f = oracle.Fold("*", "int64")
    for part in np.array_split(odd, 9):
        f.merge(oracle.Fold("*", "int64").fold(part))
    assert int(f.result()[0]) % (1 << 20) == 1


@pytest.mark.parametrize("op", list(oracle.OPS))
@pytest.mark.parametrize("dt", INT)
def test_split_merge_equals_bigint_fold(op, dt):
    # any split of the iteration space, merged in order, gives the bits of a Python big-integer left fold
    xs = ipmgen.fill_host(ipmgen.Spec(dt, 5000, "odd" if op == "*" else "random", seed=8))
    if op in ("&&", "||"):
        xs = xs % 3
    mask = (1 << W[dt]) - 1
    sg = lambda x: x - (1 << W[dt]) if x >> (W[dt] - 1) else x
    r = 77
    for x in xs.tolist():
        x &= mask
        r = {"+": lambda: (r + x) & mask, "*": lambda: (r * x) & mask, "max": lambda: r if sg(r) >= sg(x) else x,
             "min": lambda: r if sg(r) <= sg(x) else x, "&": lambda: r & x, "|": lambda: r | x, "^": lambda: r ^ x,
             "&&": lambda: int(r != 0 and x != 0), "||": lambda: int(r != 0 or x != 0)}[op]()
    for cuts in ([2500], [1, 2, 3, 4999], [0, 0, 5000], list(range(0, 5000, 333))):
        bounds = [0] + cuts + [5000]
        f = oracle.Fold(op, dt, NPT[dt](77))
        f.fold(xs[bounds[0]:bounds[1]])
        for a, b in zip(bounds[1:-1], bounds[2:]):
            f.merge(oracle.Fold(op, dt).fold(xs[a:b]))
        assert u(f.result()[0], dt) == r, (op, cuts)


@pytest.mark.parametrize("dt", FLT)
def test_split_merge_float_sum(dt):
    # i mod 1024 over n elements: closed form (n/1024)·523776, exact; random dyadic data: within 2^-60 of the
    # exact sum (integers in units of the grid), as the unsplit compensated fold
    n = 1 << 22
    v, ld, _ = oracle.reduce_spec_split("+", ipmgen.Spec(dt, n, "mod", param=1024), pieces=13, threads=4)
    assert ld == (n // 1024) * 523776 and v == (n // 1024) * 523776
    s = ipmgen.Spec(dt, 1 << 20, "random", seed=4)
    a = ipmgen.fill_host(s)
    g = 14 if dt == "float32" else 43                       # the generator's dyadic grid, 2^-g (ipmgen.h)
    exact = Fraction(sum((a.astype(np.float64) * 2.0**g).astype(np.int64).tolist()), 2**g)   # exact integers
    _, ld, _ = oracle.reduce_spec_split("+", s, init=NPT[dt](0.25), pieces=64, threads=8, chunk=10_000)
    assert abs(fr(ld) - (exact + Fraction(1, 4))) <= exact * Fraction(1, 2**60)
    # compensation survives the merge: [1e20, 1] | [-1e20] must give 1 (a plain merge of s would give 0)
    f = oracle.Fold("+", "float64").fold(np.array([1e20, 1.0]))
    f.merge(oracle.Fold("+", "float64").fold(np.array([-1e20])))
    assert f.result()[1] == 1


@pytest.mark.parametrize("dt", FLT)
def test_split_merge_float_product_and_extremes(dt):
    # ±1 background with 64 planted factors: the exact product (Fraction) within the rounding bound
    s = ipmgen.Spec(dt, 1 << 20, "signs", seed=3, plant="factor", nplant=64)
    a = ipmgen.fill_host(s)
    exact = Fraction(1)
    for x in a.tolist():
        if x != 1.0:
            exact *= Fraction(x)
    _, ld, _ = oracle.reduce_spec_split("*", s, pieces=10, threads=4)
    assert abs(fr(ld) - exact) <= abs(exact) * Fraction(64, 2**63)
    # IEEE maximum across pieces: -0 in one piece, +0 in a later one -> +0; NaN in any piece -> NaN
    x = np.full(100, -1.0, NPT[dt]); x[10] = -0.0; x[90] = 0.0
    f = oracle.Fold("max", dt).fold(x[:50]).merge(oracle.Fold("max", dt).fold(x[50:]))
    assert struct.pack("<d", float(f.result()[0])) == struct.pack("<d", 0.0)
    f = oracle.Fold("min", dt).fold(-x[:50]).merge(oracle.Fold("min", dt).fold(-x[50:]))
    assert struct.pack("<d", float(f.result()[0])) == struct.pack("<d", -0.0)
    x[60] = np.nan
    f = oracle.Fold("max", dt).fold(x[:50]).merge(oracle.Fold("max", dt).fold(x[50:]))
    assert np.isnan(f.result()[0])
    # && / || across pieces: C truthiness of the pieces' values
    y = np.ones(100, NPT[dt]); y[70] = -0.0
    f = oracle.Fold("&&", dt).fold(y[:50]).merge(oracle.Fold("&&", dt).fold(y[50:]))
    assert f.result()[0] == 0
    z = np.zeros(100, NPT[dt]); z[99] = np.nan
    f = oracle.Fold("||", dt).fold(z[:50]).merge(oracle.Fold("||", dt).fold(z[50:]))
    assert f.result()[0] == 1
