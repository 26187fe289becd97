"""ipmgen — the seeded, counter-based synthetic input generator (see ipmgen/ipmgen.h for the definition).

This module serves both sides of the parity check: the CPU oracle folds ``fill_host`` chunks, and tests /
bench.py create device inputs with ``fill_device``. It holds no reduction arithmetic (SURVEY.md §8(c),
"Input generator").
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "libipmgen.so")

I32, I64, F32, F64 = 0, 1, 2, 3
KINDS = {"random": 0, "signed": 1, "odd": 2, "iota": 3, "mod": 4, "const": 5, "signs": 6, "allbits": 7,
         "nonzero": 8}
PLANTS = {"none": 0, "value": 1, "factor": 2, "clearbit": 3, "setbit": 4, "random": 5}
DTYPES = {"int32": I32, "int64": I64, "float32": F32, "float64": F64}
NP_DTYPES = {I32: np.int32, I64: np.int64, F32: np.float32, F64: np.float64}


class _CSpec(ctypes.Structure):
    _fields_ = [("kind", ctypes.c_int32), ("dtype", ctypes.c_int32), ("seed", ctypes.c_uint64),
                ("n", ctypes.c_int64), ("param", ctypes.c_double), ("plant_kind", ctypes.c_int32),
                ("nplant", ctypes.c_int32), ("plant_param", ctypes.c_double)]


@dataclass(frozen=True)
class Spec:
    """What the i-th element of a synthetic buffer of length ``n`` is (see ipmgen.h)."""
    dtype: str
    n: int
    kind: str = "random"
    seed: int = 1
    param: float = 0.0
    plant: str = "none"
    nplant: int = 0
    plant_param: float = 0.0

    def c(self) -> _CSpec:
        return _CSpec(KINDS[self.kind], DTYPES[self.dtype], self.seed & (2**64 - 1), self.n, float(self.param),
                      PLANTS[self.plant], self.nplant, float(self.plant_param))

    @property
    def np_dtype(self):
        return NP_DTYPES[DTYPES[self.dtype]]


_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(_LIB_PATH)
        L.ipmgen_fill_host.argtypes = [ctypes.POINTER(_CSpec), ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p]
        L.ipmgen_fill_host.restype = ctypes.c_int
        L.ipmgen_fill_device.argtypes = [ctypes.POINTER(_CSpec), ctypes.c_int64, ctypes.c_int64, ctypes.c_void_p,
                                         ctypes.c_void_p]
        L.ipmgen_fill_device.restype = ctypes.c_int
        L.ipmgen_h.argtypes = [ctypes.c_uint64, ctypes.c_uint64]
        L.ipmgen_h.restype = ctypes.c_uint64
        L.ipmgen_plant_pos.argtypes = [ctypes.POINTER(_CSpec), ctypes.c_int32]
        L.ipmgen_plant_pos.restype = ctypes.c_int64
        _lib = L
    return _lib


def h(seed: int, i: int) -> int:
    return lib().ipmgen_h(seed & (2**64 - 1), i & (2**64 - 1))


def plant_positions(spec: Spec) -> list[int]:
    cs = spec.c()
    return [lib().ipmgen_plant_pos(ctypes.byref(cs), k) for k in range(spec.nplant)]


def fill_host(spec: Spec, lo: int = 0, count: int | None = None) -> np.ndarray:
    if count is None:
        count = spec.n - lo
    out = np.empty(count, dtype=spec.np_dtype)
    cs = spec.c()
    rc = lib().ipmgen_fill_host(ctypes.byref(cs), lo, count, out.ctypes.data if count else None)
    if rc:
        raise ValueError(f"ipmgen_fill_host failed ({rc})")
    return out


def chunks(spec: Spec, chunk: int = 1 << 22, lo: int = 0, hi: int | None = None):
    """Yield the elements of [lo, hi) in host chunks (streams inputs too large to materialise)."""
    hi = spec.n if hi is None else hi
    for a in range(lo, hi, chunk):
        yield fill_host(spec, a, min(chunk, hi - a))


def fill_device(spec: Spec, dev_ptr: int, lo: int = 0, count: int | None = None, stream: int = 0) -> None:
    """Write elements [lo, lo+count) to device memory at ``dev_ptr`` on CUDA stream ``stream`` (raw handle)."""
    if count is None:
        count = spec.n - lo
    cs = spec.c()
    rc = lib().ipmgen_fill_device(ctypes.byref(cs), lo, count, dev_ptr, stream)
    if rc:
        raise RuntimeError(f"ipmgen_fill_device failed (cudaError {rc})")


def fill_tensor(spec: Spec, t, lo: int = 0) -> None:
    """Fill a contiguous CUDA torch tensor with elements [lo, lo+t.numel())."""
    import torch
    fill_device(spec, t.data_ptr(), lo, t.numel(), torch.cuda.current_stream(t.device).cuda_stream)


DEGREE_TAG = 0xD1B54A32D192ED03


def draws(seed: int, idx: np.ndarray) -> np.ndarray:
    """Vectorised h(seed, i) for an array of indices (the same splitmix64 stream as ipmgen.h; tests compare it
    with the C implementation)."""
    G = np.uint64(0x9E3779B97F4A7C15)
    with np.errstate(over="ignore"):
        z = np.uint64(seed & (2**64 - 1)) * G + (idx.astype(np.uint64) + np.uint64(1)) * G
        z = (z ^ (z >> np.uint64(30))) * np.uint64(0xBF58476D1CE4E5B9)
        z = (z ^ (z >> np.uint64(27))) * np.uint64(0x94D049BB133111EB)
    return z ^ (z >> np.uint64(31))


def degrees(rows: int, seed: int = 1, kind: str = "powerlaw", mean: float = 16.0, alpha: float = 1.5,
            cap: int | None = None) -> np.ndarray:
    """Row lengths of a ragged (CSR) input — graph adjacency lists for the BFS-style nested loop.
    powerlaw: d = floor(dmin * u^(-1/alpha)) with u uniform in (0,1] from h(seed ^ TAG, r), dmin chosen so the mean
    is about `mean`, capped at `cap`; uniform: d in [0, 2*mean]; const: d = mean."""
    r = np.arange(rows, dtype=np.uint64)
    if kind == "const":
        return np.full(rows, int(mean), dtype=np.int64)
    z = draws(seed ^ DEGREE_TAG, r)
    u = ((z >> np.uint64(11)).astype(np.float64) + 1.0) * 2.0 ** -53          # (0, 1]
    if kind == "uniform":
        d = np.floor(u * (2 * mean + 1)).astype(np.int64)
        d = np.minimum(d, int(2 * mean))
    else:
        dmin = mean * (alpha - 1) / alpha
        d = np.floor(dmin * u ** (-1.0 / alpha)).astype(np.int64)
    if cap is not None:
        d = np.minimum(d, cap)
    return d


def offsets_from_degrees(d: np.ndarray, start: int = 0) -> np.ndarray:
    off = np.empty(d.size + 1, dtype=np.int64)
    off[0] = start
    np.cumsum(d, out=off[1:])
    off[1:] += start
    return off
