"""oracle — plain, slow, obviously correct CPU implementation of the OpenACC ``reduction(op:var)`` clause.

TEST INFRASTRUCTURE ONLY: only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s ``cpu_baseline`` /
``--impl reference`` legs may import this package. The product path (``paper_1412_1127_b200``) never does and
shares no code with it. The arithmetic lives in ``ipm_oracle.c`` (its header lists the paper passages and the
readings it follows); this file is argument marshalling only.

Parity pins for every function here are in ``tests/test_oracle.py`` (closed forms, brute force, fsum, numpy).
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB_PATH = os.path.join(_HERE, "liboracle.so")

OPS = {"+": 0, "*": 1, "max": 2, "min": 3, "&": 4, "|": 5, "^": 6, "&&": 7, "||": 8}
DTYPES = {"int32": 0, "int64": 1, "float32": 2, "float64": 3}
NP = {"int32": np.int32, "int64": np.int64, "float32": np.float32, "float64": np.float64}

_lib = None


def lib():
    global _lib
    if _lib is None:
        if not os.path.exists(_LIB_PATH):
            raise RuntimeError(f"{_LIB_PATH} missing: run `python -c 'import __graft_entry__ as g; g.build()'`")
        L = ctypes.CDLL(_LIB_PATH)
        vp, i64, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int
        L.ora_state_size.restype = ci
        L.ora_legal.argtypes = [ci, ci]
        L.ora_legal.restype = ci
        L.ora_begin.argtypes = [vp, ci, ci, vp]
        L.ora_begin.restype = ci
        L.ora_fold.argtypes = [vp, vp, i64]
        L.ora_fold.restype = None
        L.ora_result.argtypes = [vp, vp, vp]
        L.ora_result.restype = None
        L.ora_merge.argtypes = [vp, vp]
        L.ora_merge.restype = ci
        L.ora_reduce.argtypes = [ci, ci, vp, i64, vp, vp, vp]
        L.ora_reduce.restype = ci
        L.ora_reduce_segmented.argtypes = [ci, ci, vp, i64, i64, i64, vp, vp, vp]
        L.ora_reduce_segmented.restype = ci
        L.ora_reduce_ragged.argtypes = [ci, ci, vp, vp, i64, vp, vp, vp]
        L.ora_reduce_ragged.restype = ci
        L.ora_fused_nvars.argtypes = [ci]
        L.ora_fused_nvars.restype = ci
        L.ora_reduce_fused.argtypes = [ci, ci, vp, vp, i64, vp, vp, vp]
        L.ora_reduce_fused.restype = ci
        _lib = L
    return _lib


def _scalar_buf(dtype: str, value):
    if value is None:
        return None
    return np.array([value], dtype=NP[dtype])


def legal(op: str, dtype: str) -> bool:
    return bool(lib().ora_legal(OPS[op], DTYPES[dtype]))


class Fold:
    """A sequential left fold that can be fed in chunks (used to stream inputs larger than host RAM)."""

    def __init__(self, op: str, dtype: str, init=None):
        if not legal(op, dtype):
            raise ValueError(f"reduction({op}) is illegal on {dtype}")
        self.dtype = dtype
        self._st = ctypes.create_string_buffer(lib().ora_state_size())
        self._init = _scalar_buf(dtype, init)
        lib().ora_begin(self._st, OPS[op], DTYPES[dtype], None if self._init is None else self._init.ctypes.data)

    def fold(self, a: np.ndarray) -> "Fold":
        a = np.ascontiguousarray(a, dtype=NP[self.dtype])
        if a.size:
            lib().ora_fold(self._st, a.ctypes.data, a.size)
        return self

    def merge(self, later: "Fold") -> "Fold":
        """Continue this fold with the fold of the NEXT contiguous chunk (begun without init): ora_merge."""
        if lib().ora_merge(self._st, later._st):
            raise ValueError("merge of folds of different op / dtype")
        return self

    def result(self):
        """(value as a numpy scalar of the element type, the oracle's long double value)."""
        out = np.zeros(1, dtype=NP[self.dtype])
        ld = np.zeros(1, dtype=np.longdouble)  # not ctypes.c_longdouble: its .value rounds to a double
        lib().ora_result(self._st, out.ctypes.data, ld.ctypes.data)
        return out[0], ld[0]


def reduce(op: str, a, dtype: str | None = None, init=None):
    """var = init ⊕ a[0] ⊕ ... ⊕ a[n-1]; returns (T value, long double value)."""
    if dtype is None:
        dtype = np.asarray(a).dtype.name
    return Fold(op, dtype, init).fold(np.asarray(a, dtype=NP[dtype])).result()


def reduce_spec(op: str, spec, init=None, lo: int = 0, hi: int | None = None, chunk: int = 1 << 22):
    """The same fold over elements [lo, hi) of an ipmgen.Spec, generated chunk by chunk on the host."""
    import ipmgen
    f = Fold(op, spec.dtype, init)
    for c in ipmgen.chunks(spec, chunk, lo, hi):
        f.fold(c)
    return f.result()


def reduce_spec_split(op: str, spec, init=None, lo: int = 0, hi: int | None = None, pieces: int = 64,
                      threads: int | None = None, chunk: int = 1 << 22):
    """reduce_spec over [lo, hi) split into `pieces` contiguous pieces folded on `threads` host threads (each piece
    a plain left fold of generated chunks), then merged in piece order (ora_merge) — SURVEY.md §8(d)'s permitted
    split of the C5 oracle. Returns (T value, long double value, threads used)."""
    import concurrent.futures as cf
    hi = spec.n if hi is None else hi
    pieces = max(1, min(pieces, hi - lo)) if hi > lo else 1
    if threads is None:
        try:
            threads = len(os.sched_getaffinity(0))
        except Exception:
            threads = os.cpu_count() or 1
    bounds = [lo + (hi - lo) * k // pieces for k in range(pieces + 1)]

    def piece(k):
        f = Fold(op, spec.dtype, init if k == 0 else None)
        import ipmgen
        for c in ipmgen.chunks(spec, chunk, bounds[k], bounds[k + 1]):
            f.fold(c)   # ctypes releases the GIL: the pieces run in parallel
        return f

    with cf.ThreadPoolExecutor(max_workers=threads) as ex:
        folds = list(ex.map(piece, range(pieces)))
    total = folds[0]
    for f in folds[1:]:
        total.merge(f)
    v, ld = total.result()
    return v, ld, threads


def reduce_segmented(op: str, a, rows: int, cols: int, stride: int | None = None, dtype: str | None = None,
                     init=None):
    """out[r] = init ⊕ fold_j a[r*stride + j]; returns (out as T array, out as long double array)."""
    a = np.ascontiguousarray(a)
    dtype = dtype or a.dtype.name
    stride = cols if stride is None else stride
    if rows > 0 and cols > 0 and a.size < (rows - 1) * stride + cols:
        raise ValueError("array too small for rows/cols/stride")
    out = np.zeros(rows, dtype=NP[dtype])
    out_ld = np.zeros(rows, dtype=np.longdouble)
    ib = _scalar_buf(dtype, init)
    rc = lib().ora_reduce_segmented(OPS[op], DTYPES[dtype], a.ctypes.data if a.size else None, rows, cols, stride,
                                    None if ib is None else ib.ctypes.data, out.ctypes.data if rows else None,
                                    out_ld.ctypes.data if rows else None)
    if rc:
        raise ValueError(f"ora_reduce_segmented failed ({rc})")
    return out, out_ld


def identity(op: str, dtype: str):
    return reduce(op, np.zeros(0, dtype=NP[dtype]), dtype)[0]


FUSED = {"sum_sumsq": 0, "dot": 1, "minmax": 2, "stats": 3}


def reduce_fused(sig: str, x, y=None, dtype: str | None = None, init=None):
    """Several variables over one pass: returns (values as a T array, long double array), one per variable.
    sum_sumsq -> (Σx, Σx²); dot -> (Σxy,); minmax -> (min, max); stats -> (Σx, Σx², min, max)."""
    x = np.ascontiguousarray(x)
    dtype = dtype or x.dtype.name
    x = x.astype(NP[dtype], copy=False)
    f = FUSED[sig]
    nv = lib().ora_fused_nvars(f)
    yy = None if y is None else np.ascontiguousarray(y, dtype=NP[dtype])
    if f == 1 and (yy is None or yy.size != x.size):
        raise ValueError("dot needs y of the same length")
    out = np.zeros(nv, dtype=NP[dtype])
    out_ld = np.zeros(nv, dtype=np.longdouble)
    ib = None if init is None else np.ascontiguousarray(init, dtype=NP[dtype])
    rc = lib().ora_reduce_fused(f, DTYPES[dtype], x.ctypes.data if x.size else None,
                                None if yy is None or not yy.size else yy.ctypes.data, x.size,
                                None if ib is None else ib.ctypes.data, out.ctypes.data, out_ld.ctypes.data)
    if rc:
        raise ValueError(f"ora_reduce_fused failed ({rc})")
    return out, out_ld


def reduce_ragged(op: str, a, offsets, dtype: str | None = None, init=None):
    """out[r] = init ⊕ fold a[offsets[r]:offsets[r+1]]; returns (out as T array, long double array)."""
    a = np.ascontiguousarray(a)
    dtype = dtype or a.dtype.name
    a = a.astype(NP[dtype], copy=False)
    off = np.ascontiguousarray(offsets, dtype=np.int64)
    rows = off.size - 1
    out = np.zeros(max(rows, 0), dtype=NP[dtype])
    out_ld = np.zeros(max(rows, 0), dtype=np.longdouble)
    ib = _scalar_buf(dtype, init)
    rc = lib().ora_reduce_ragged(OPS[op], DTYPES[dtype], a.ctypes.data if a.size else None, off.ctypes.data, rows,
                                 None if ib is None else ib.ctypes.data, out.ctypes.data if rows else None,
                                 out_ld.ctypes.data if rows else None)
    if rc:
        raise ValueError(f"ora_reduce_ragged failed ({rc})")
    return out, out_ld
