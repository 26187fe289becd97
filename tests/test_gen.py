"""The input generator (ipmgen) against its definition in ipmgen/ipmgen.h (host side; device == host is in
tests/test_gpu_parity.py)."""
import numpy as np
import pytest

import ipmgen


def test_splitmix64_reference_value():
    # splitmix64 with state 0: the first output is 0xE220A8397B1DCDAF (the published reference sequence)
    assert ipmgen.h(0, 0) == 0xE220A8397B1DCDAF
    assert ipmgen.h(0, 1) == 0x6E789E6AA1B965F4


@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_dyadic_ranges_and_exactness(dt):
    a = ipmgen.fill_host(ipmgen.Spec(dt, 100_000, "random", seed=3)).astype(np.float64)
    assert a.min() >= 0 and a.max() < 1024
    scale = 2.0 ** (14 if dt == "float32" else 43)
    assert np.all(np.floor(a * scale) == a * scale)           # multiples of 2^-14 / 2^-43
    s = ipmgen.fill_host(ipmgen.Spec(dt, 100_000, "signed", seed=3))
    assert s.min() >= -1024 and s.max() < 1024
    assert not np.any((s == 0) & np.signbit(s))               # never -0.0
    nz = ipmgen.fill_host(ipmgen.Spec(dt, 100_000, "nonzero", seed=3))
    assert np.all(nz != 0)


def test_chunked_equals_whole():
    for dt in ["int32", "int64", "float32", "float64"]:
        s = ipmgen.Spec(dt, 10_000, "signs" if dt[0] == "f" else "random", seed=9, plant="factor", nplant=40)
        whole = ipmgen.fill_host(s)
        parts = np.concatenate(list(ipmgen.chunks(s, 777)))
        assert whole.tobytes() == parts.tobytes()


def test_plants():
    s = ipmgen.Spec("float32", 1000, "signs", seed=1, plant="factor", nplant=64)
    a = ipmgen.fill_host(s)
    pos = ipmgen.plant_positions(s)
    assert all(0 <= p < 1000 for p in pos)
    others = np.setdiff1d(np.arange(1000), pos)
    assert set(np.unique(np.abs(a[others]))) == {1.0}
    f = a[sorted(set(pos))]
    assert np.all((f >= 0.5) & (f < 2.0))
    # 24-bit mantissas: exact in fp32
    assert np.all(f.astype(np.float64) * 2 ** 24 == np.floor(f.astype(np.float64) * 2 ** 24))
    s = ipmgen.Spec("int64", 1000, "allbits", seed=2, plant="clearbit", nplant=5)
    a = ipmgen.fill_host(s)
    for p in ipmgen.plant_positions(s):
        assert bin(int(a[p]) & (2**64 - 1)).count("1") == 63


def test_iota_mod_const():
    assert np.array_equal(ipmgen.fill_host(ipmgen.Spec("int32", 10, "iota", param=1)), np.arange(1, 11))
    assert np.array_equal(ipmgen.fill_host(ipmgen.Spec("float32", 3000, "mod", param=1024)),
                          (np.arange(3000) % 1024).astype(np.float32))
    assert np.all(ipmgen.fill_host(ipmgen.Spec("float64", 5, "const", param=2.5)) == 2.5)
    # int32 iota wraps mod 2^32
    a = ipmgen.fill_host(ipmgen.Spec("int32", 3, "iota", param=2**31 - 2))
    assert list(a) == [2**31 - 2, 2**31 - 1, -2**31]


def test_vectorised_draws_match_c():
    idx = np.array([0, 1, 2, 1000, 2**40 + 7], dtype=np.uint64)
    for seed in [0, 1, 0xD1B54A32D192ED03 ^ 5]:
        assert list(ipmgen.draws(seed, idx)) == [ipmgen.h(seed, int(i)) for i in idx]


def test_degrees():
    d = ipmgen.degrees(200_000, seed=3)
    assert d.min() >= 0 and 10 < d.mean() < 22 and d.max() > 1000      # heavy tail around mean 16
    off = ipmgen.offsets_from_degrees(d, start=5)
    assert off[0] == 5 and off[-1] == 5 + d.sum() and np.all(np.diff(off) == d)
    assert np.array_equal(ipmgen.degrees(10, kind="const", mean=4), np.full(10, 4))
