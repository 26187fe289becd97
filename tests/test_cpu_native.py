"""The OpenMP CPU baseline bench.py reports (BASELINE.md "CPU native baseline") computes the clause: a float32
`reduction(+:s)` over all host threads, checked against an exact float64 sum of integer-valued data."""
import ctypes
import os

import numpy as np
import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
LIB = os.path.join(ROOT, "tools", "bin", "libcpu_omp.so")


@pytest.fixture(scope="module")
def omp():
    if not os.path.exists(LIB):
        pytest.skip("tools/bin/libcpu_omp.so not built (tools/build.py build_cpu_omp)")
    L = ctypes.CDLL(LIB)
    L.cpu_omp_sum_f32.restype = ctypes.c_float
    L.cpu_omp_sum_f32.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    L.cpu_omp_sum_f32_f64.restype = ctypes.c_double
    L.cpu_omp_sum_f32_f64.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    L.cpu_omp_threads.restype = ctypes.c_int
    return L


def test_omp_sum_matches_exact(omp):
    for n in (0, 1, 7, 1000, 1 << 20):
        a = (np.arange(n) % 7).astype(np.float32)  # small integers: every partial sum below 2^24 is exact
        exact = float((np.arange(n) % 7).sum())
        assert omp.cpu_omp_sum_f32_f64(a.ctypes.data, n) == exact
        if exact < (1 << 24):
            assert omp.cpu_omp_sum_f32(a.ctypes.data, n) == exact
    assert omp.cpu_omp_threads() >= 1
