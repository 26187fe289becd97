"""Python binding of libipm (include/ipm.h): argument marshalling only — every step of the reduction runs in
the CUDA kernels of ``csrc/``. PyTorch supplies device memory (its caching allocator is installed as the
library's allocator hook), streams and process groups.

There is no fallback: if ``libipm.so`` is missing or fails to load, importing this module raises.
"""
from __future__ import annotations

import ctypes
import functools
import os
import threading

import numpy as np
import torch

_HERE = os.path.dirname(os.path.abspath(__file__))
LIB_PATH = os.environ.get("IPM_LIB", os.path.join(_HERE, "libipm.so"))  # IPM_LIB: A/B of two builds (tools/ab_lib.py)

# operator names follow the clause syntax `reduction(op:var)` (OpenACC; SPEC.md:110 plus the BASELINE.json ops)
OPS = {"+": 0, "*": 1, "max": 2, "min": 3, "&": 4, "|": 5, "^": 6, "&&": 7, "||": 8}
DTYPES = {torch.int32: 0, torch.int64: 1, torch.float32: 2, torch.float64: 3}
NP_OF = {0: np.int32, 1: np.int64, 2: np.float32, 3: np.float64}
TORCH_OF = {0: torch.int32, 1: torch.int64, 2: torch.float32, 3: torch.float64}
STATUS = ["IPM_OK", "IPM_E_REDOP", "IPM_E_DTYPE", "IPM_E_NULL", "IPM_E_SIZE", "IPM_E_PRESENT", "IPM_E_ALIGN",
          "IPM_E_WORKSPACE", "IPM_E_CUDA", "IPM_E_NCCL", "IPM_E_ARG"]


class IpmError(RuntimeError):
    def __init__(self, code: int, where: str, detail: str):
        self.code = code
        self.status = STATUS[code] if 0 <= code < len(STATUS) else f"status {code}"
        super().__init__(f"{where}: {self.status}: {detail}")


def _load():
    if not os.path.exists(LIB_PATH):
        raise ImportError(f"{LIB_PATH} is missing — build it with `python -c 'import __graft_entry__ as g; g.build()'`"
                          " (there is no CPU fallback)")
    L = ctypes.CDLL(LIB_PATH)
    vp, i64, ci, sz = ctypes.c_void_p, ctypes.c_int64, ctypes.c_int, ctypes.c_size_t
    sigs = {
        "ipm_status_str": ([ci], ctypes.c_char_p),
        "ipm_last_error_message": ([], ctypes.c_char_p),
        "ipm_op_legal": ([ci, ci], ci),
        "ipm_dtype_size": ([ci], sz),
        "ipm_version": ([], ci),
        "ipm_set_allocator": ([vp], ci),
        "ipm_copyin": ([vp, sz, ctypes.POINTER(vp), vp], ci),
        "ipm_create": ([vp, sz, ctypes.POINTER(vp), vp], ci),
        "ipm_present": ([vp, sz, ctypes.POINTER(vp)], ci),
        "ipm_update_device": ([vp, sz, vp], ci),
        "ipm_update_host": ([vp, sz, vp], ci),
        "ipm_copyout": ([vp, sz, vp], ci),
        "ipm_delete": ([vp, vp], ci),
        "ipm_present_count": ([], ci),
        "ipm_workspace_bytes": ([], sz),
        "ipm_workspace_init": ([vp, vp], ci),
        "ipm_reduce": ([ci, ci, vp, i64, vp, vp, vp], ci),
        "ipm_reduce_async": ([ci, ci, vp, i64, vp, vp, vp, vp], ci),
        "ipm_reduce_segmented": ([ci, ci, vp, i64, i64, i64, vp, vp, vp, vp], ci),
        "ipm_reduce_ragged": ([ci, ci, vp, vp, i64, vp, vp, vp, vp], ci),
        "ipm_ragged_scratch_bytes": ([ci, i64, i64], sz),
        "ipm_reduce_ragged_marked": ([ci, ci, vp, i64, vp, i64, vp, vp, vp, vp, sz, vp], ci),
        "ipm_reduce_partials": ([ci, ci, vp, i64, vp, ci, ctypes.POINTER(ci), vp], ci),
        "ipm_finalize_partials": ([ci, ci, vp, ci, vp, vp, vp], ci),
        "ipm_reduce_2d": ([ci, ci, vp, i64, i64, i64, vp, vp, vp], ci),
        "ipm_reduce_2d_async": ([ci, ci, vp, i64, i64, i64, vp, vp, vp, vp], ci),
        "ipm_fused_nvars": ([ci], ci),
        "ipm_reduce_fused": ([ci, ci, vp, vp, i64, vp, vp, vp], ci),
        "ipm_reduce_fused_async": ([ci, ci, vp, vp, i64, vp, vp, vp, vp], ci),
        "ipm_reduce_host": ([ci, ci, vp, i64, vp, vp, vp], ci),
        "ipm_release_staging": ([], ci),
        "ipm_set_option": ([ci, i64], ci),
        "ipm_profile_enable": ([ci], ci),
        "ipm_profile_read": ([vp, vp, ci, ctypes.POINTER(ci)], ci),
        "ipm_profile_disable": ([], ci),
        "ipm_flat_geometry": ([ci, i64, ctypes.POINTER(ci), ctypes.POINTER(ci)], ci),
        "ipm_flat_schedule": ([ci, i64, ctypes.POINTER(ci)], ci),
        "ipm_identity": ([ci, ci, vp], ci),
        "ipm_comm_id_bytes": ([], sz),
        "ipm_comm_unique_id": ([vp], ci),
        "ipm_comm_init": ([ctypes.POINTER(vp), ci, ci, vp, ci], ci),
        "ipm_comm_destroy": ([vp], ci),
        "ipm_comm_init_group": ([vp, ci, ci], ci),
        "ipm_comm_ipc_handle_bytes": ([], sz),
        "ipm_comm_create_ipc": ([ctypes.POINTER(vp), ci, ci, ci, vp], ci),
        "ipm_comm_attach_ipc": ([vp, vp], ci),
        "ipm_shard_range": ([i64, ci, ci, ctypes.POINTER(i64), ctypes.POINTER(i64)], ci),
        "ipm_comm_uses_peer_memory": ([vp], ci),
        "ipm_comm_error": ([vp, ctypes.POINTER(ci)], ci),
        "ipm_reduce_host_dist": ([vp, ci, ci, vp, i64, vp, vp, vp], ci),
        "ipm_reduce_dist": ([vp, ci, ci, vp, i64, vp, vp, vp], ci),
        "ipm_reduce_dist_async": ([vp, ci, ci, vp, i64, vp, vp, vp, vp], ci),
    }
    for name, (args, res) in sigs.items():
        if "IPM_LIB" in os.environ and not hasattr(L, name):
            continue  # an older build loaded for a same-box A/B (tools/ab_lib.py): calls it lacks fail when used
        f = getattr(L, name)  # AttributeError if the library does not export it: fail loudly
        f.argtypes = args
        f.restype = res
    return L


lib = _load()
EXPORTED = ("ipm_status_str ipm_last_error_message ipm_op_legal ipm_dtype_size ipm_version ipm_set_allocator "
            "ipm_copyin ipm_create ipm_present ipm_update_device ipm_update_host ipm_copyout ipm_delete "
            "ipm_present_count ipm_workspace_bytes ipm_workspace_init ipm_reduce ipm_reduce_async "
            "ipm_reduce_segmented ipm_reduce_ragged ipm_ragged_scratch_bytes ipm_reduce_ragged_marked ipm_reduce_partials ipm_finalize_partials ipm_reduce_2d ipm_reduce_2d_async ipm_fused_nvars ipm_reduce_fused ipm_reduce_fused_async ipm_reduce_host ipm_release_staging ipm_set_option ipm_profile_enable ipm_profile_read "
            "ipm_profile_disable ipm_flat_geometry ipm_flat_schedule ipm_identity ipm_comm_id_bytes "
            "ipm_comm_unique_id ipm_comm_init ipm_comm_destroy ipm_comm_init_group ipm_comm_ipc_handle_bytes "
            "ipm_comm_create_ipc ipm_comm_attach_ipc ipm_shard_range ipm_comm_uses_peer_memory ipm_comm_error "
            "ipm_reduce_host_dist ipm_reduce_dist "
            "ipm_reduce_dist_async").split()


def _check(code: int, where: str):
    if code != 0:
        raise IpmError(code, where, lib.ipm_last_error_message().decode(errors="replace"))


# ------------------------------------------------------------------ allocator hook: PyTorch's caching allocator
_ALLOC_T = ctypes.CFUNCTYPE(ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_void_p)
_FREE_T = ctypes.CFUNCTYPE(None, ctypes.c_void_p, ctypes.c_void_p, ctypes.c_void_p)


class _CAllocator(ctypes.Structure):
    _fields_ = [("alloc", _ALLOC_T), ("free", _FREE_T), ("ctx", ctypes.c_void_p)]


def _torch_alloc(nbytes, stream, ctx):
    try:
        return torch.cuda.caching_allocator_alloc(int(nbytes), torch.cuda.current_device(), stream or 0)
    except Exception:  # out of memory -> NULL -> IPM_E_CUDA on the C side
        return None


def _torch_free(p, stream, ctx):
    torch.cuda.caching_allocator_delete(p)


_alloc_cb = _ALLOC_T(_torch_alloc)
_free_cb = _FREE_T(_torch_free)
_allocator = _CAllocator(_alloc_cb, _free_cb, None)
_check(lib.ipm_set_allocator(ctypes.byref(_allocator)), "ipm_set_allocator")


# ------------------------------------------------------------------ helpers
def op_code(op: str) -> int:
    try:
        return OPS[op]
    except KeyError:
        raise ValueError(f"unknown reduction operator {op!r}; one of {list(OPS)}") from None


def dtype_code(dt) -> int:
    if isinstance(dt, torch.dtype):
        return DTYPES[dt]
    return DTYPES[{np.int32: torch.int32, np.int64: torch.int64, np.float32: torch.float32,
                   np.float64: torch.float64}[np.dtype(dt).type]]


def legal(op: str, dtype) -> bool:
    return bool(lib.ipm_op_legal(op_code(op), dtype_code(dtype)))


_raw_stream = getattr(torch._C, "_cuda_getCurrentRawStream", None)


def _stream(stream=None) -> int:
    if stream is None:
        # torch's current stream of the current device; the raw accessor avoids building a Stream object
        # (~3 us per call, measured by tools/py_overhead.py)
        if _raw_stream is not None:
            return _raw_stream(torch.cuda.current_device())
        return torch.cuda.current_stream().cuda_stream
    return stream.cuda_stream if hasattr(stream, "cuda_stream") else int(stream)


def _sync(stream=None) -> None:
    """Wait for `stream` (None = torch's current stream) before reading results on the host."""
    if stream is None:
        torch.cuda.current_stream().synchronize()
    elif hasattr(stream, "synchronize"):
        stream.synchronize()
    else:
        torch.cuda.ExternalStream(int(stream)).synchronize()


def _scalar(dt: int, value):
    """a 1-element numpy buffer holding `value` in element type dt (None -> None)"""
    if value is None:
        return None
    return np.array([value], dtype=NP_OF[dt])


WS_BYTES = lib.ipm_workspace_bytes()
_ws_cache: dict = {}
_ws_lock = threading.Lock()


def workspace(stream=None, device=None) -> torch.Tensor:
    """The per-(device, stream) zero-initialised workspace used when none is passed explicitly."""
    dev = torch.cuda.current_device() if device is None else device
    s = stream if isinstance(stream, int) else _stream(stream)
    with _ws_lock:
        ws = _ws_cache.get((dev, s))
        if ws is None:
            ws = torch.empty(WS_BYTES, dtype=torch.uint8, device=f"cuda:{dev}")
            # zeroed ON the stream the library will use it on (ipm_workspace_init), so the first kernel's
            # tickets and counter cannot race with a memset queued on another stream
            with torch.cuda.device(dev):
                _check(lib.ipm_workspace_init(ws.data_ptr(), s), "ipm_workspace_init")
            _ws_cache[(dev, s)] = ws
    return ws


def _check_out(out: torch.Tensor, like: torch.Tensor, count: int, what: str = "out") -> None:
    """A caller-supplied result tensor must match the input's dtype and device, be contiguous and hold at least
    `count` elements (the library writes count elements of the input's type there)."""
    if not out.is_cuda or out.device != like.device:
        raise ValueError(f"{what} must be a CUDA tensor on {like.device}")
    if out.dtype != like.dtype:
        raise ValueError(f"{what} has dtype {out.dtype}, expected {like.dtype}")
    if not out.is_contiguous() or out.numel() < count:
        raise ValueError(f"{what} must be contiguous with at least {count} elements")


def _check_region(t: torch.Tensor, rows: int, cols: int, row_stride: int) -> None:
    """rows x cols elements at row_stride must lie inside t's storage from t's first element"""
    if rows < 0 or cols < 0 or row_stride < cols:
        raise ValueError("need rows >= 0, cols >= 0, row_stride >= cols")
    if rows and cols:
        span = (rows - 1) * row_stride + cols
        avail = t.untyped_storage().nbytes() // t.element_size() - t.storage_offset()
        if span > avail:
            raise ValueError(f"region of {rows} x {cols} at stride {row_stride} ({span} elements) exceeds the "
                             f"tensor's storage ({avail} elements from its start)")


def _flat_arg(t: torch.Tensor):
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor (use reduce_host for host arrays)")
    if not t.is_contiguous():
        raise ValueError("expected a contiguous tensor")
    return t.data_ptr(), t.numel(), DTYPES[t.dtype]


# ------------------------------------------------------------------ reductions
def reduce(op: str, t: torch.Tensor, init=None, ws: torch.Tensor | None = None, stream=None):
    """`reduction(op:var)` over all elements of a CUDA tensor; returns init ⊕ fold as a numpy scalar.
    Blocks until the result is on the host (ipm_reduce). A non-contiguous 2-D view whose rows are contiguous
    (e.g. ``big[:, a:b]``) is reduced in place as a strided 2-D region (ipm_reduce_2d)."""
    if t.is_cuda and not t.is_contiguous() and t.dim() == 2 and (t.shape[1] <= 1 or t.stride(1) == 1):
        return reduce_2d(op, t, init=init, ws=ws, stream=stream)
    ptr, n, dt = _flat_arg(t)
    s = _stream(stream)
    ws = workspace(s) if ws is None else ws
    # no original value: start from the identity, which leaves the fold unchanged
    box = _scalar(dt, identity_value(op, dt) if init is None else init)
    _check(lib.ipm_reduce(op_code(op), dt, ptr, n, box.ctypes.data, ws.data_ptr(), s), "ipm_reduce")
    return box[0]


def reduce_async(op: str, t: torch.Tensor, init=None, out: torch.Tensor | None = None,
                 ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Asynchronous form: returns (or fills) a 1-element CUDA tensor written in stream order."""
    ptr, n, dt = _flat_arg(t)
    if out is None:
        out = torch.empty(1, dtype=t.dtype, device=t.device)
    else:
        _check_out(out, t, 1)
    ws = workspace(stream) if ws is None else ws
    box = _scalar(dt, init)
    _check(lib.ipm_reduce_async(op_code(op), dt, ptr, n, None if box is None else box.ctypes.data, out.data_ptr(),
                                ws.data_ptr(), _stream(stream)), "ipm_reduce_async")
    return out


def reduce_segmented(op: str, t: torch.Tensor, rows: int | None = None, cols: int | None = None,
                     row_stride: int | None = None, init=None, out: torch.Tensor | None = None,
                     ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Nested gang-outer / vector-inner clause: out[r] = init ⊕ fold_j t[r*row_stride + j], j < cols.
    With a 2-D tensor, rows/cols/row_stride default to its shape and row stride."""
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    dt = DTYPES[t.dtype]
    if t.dim() == 2 and rows is None:
        rows, cols = t.shape
        row_stride = t.stride(0)
        if t.stride(1) != 1:
            raise ValueError("rows must be contiguous")
    elif rows is None or cols is None:
        raise ValueError("rows and cols are required for a flat tensor")
    row_stride = cols if row_stride is None else row_stride
    _check_region(t, rows, cols, row_stride)
    if out is None:
        out = torch.empty(rows, dtype=t.dtype, device=t.device)
    else:
        _check_out(out, t, rows)
    ws = workspace(stream) if ws is None else ws
    box = _scalar(dt, init)
    _check(lib.ipm_reduce_segmented(op_code(op), dt, t.data_ptr(), rows, cols, row_stride,
                                    None if box is None else box.ctypes.data, out.data_ptr(), ws.data_ptr(),
                                    _stream(stream)), "ipm_reduce_segmented")
    return out


def reduce_ragged(op: str, values: torch.Tensor, offsets: torch.Tensor, init=None,
                  out: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Ragged (CSR) rows: out[r] = init ⊕ fold values[offsets[r]:offsets[r+1]] (offsets: int64 CUDA tensor of
    rows+1 non-decreasing indices)."""
    if not (values.is_cuda and offsets.is_cuda) or offsets.dtype != torch.int64 or not offsets.is_contiguous():
        raise ValueError("values and offsets must be CUDA tensors, offsets contiguous int64")
    ptr, _, dt = _flat_arg(values)
    rows = offsets.numel() - 1
    if out is None:
        out = torch.empty(max(rows, 0), dtype=values.dtype, device=values.device)
    else:
        _check_out(out, values, rows)
    ws = workspace(stream) if ws is None else ws
    box = _scalar(dt, init)
    if _ragged_marked[0]:  # two passes over scratch from torch's caching allocator (ipm_reduce_ragged_marked)
        nvalues = values.numel()
        scratch = torch.empty(lib.ipm_ragged_scratch_bytes(dt, nvalues, rows), dtype=torch.uint8,
                              device=values.device)
        s = _stream(stream)
        _check(lib.ipm_reduce_ragged_marked(op_code(op), dt, ptr, nvalues, offsets.data_ptr(), rows,
                                            None if box is None else box.ctypes.data, out.data_ptr(), ws.data_ptr(),
                                            scratch.data_ptr(), scratch.numel(), s),
               "ipm_reduce_ragged_marked")
        if stream is not None:
            # the scratch was allocated on torch's current stream; the kernels run on `stream`: keep the block out
            # of the caching allocator's pool until that stream's work so far has completed
            scratch.record_stream(stream if isinstance(stream, torch.cuda.Stream)
                                  else torch.cuda.ExternalStream(s, device=values.device))
        return out
    _check(lib.ipm_reduce_ragged(op_code(op), dt, ptr, offsets.data_ptr(), rows,
                                 None if box is None else box.ctypes.data, out.data_ptr(), ws.data_ptr(),
                                 _stream(stream)), "ipm_reduce_ragged")
    return out


def reduce_partials(op: str, t: torch.Tensor, out: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """The paper's first level alone: one accumulator-typed partial per thread block (8-byte slots, returned as
    a uint8 tensor view of int64 slots). See ipm.h for the slot format."""
    ptr, n, dt = _flat_arg(t)
    g, _ = flat_geometry(t.dtype, n)
    if out is None:
        out = torch.empty(g, dtype=torch.int64, device=t.device)
    cnt = ctypes.c_int()
    _check(lib.ipm_reduce_partials(op_code(op), dt, ptr, n, out.data_ptr(), out.numel(), ctypes.byref(cnt),
                                   _stream(stream)), "ipm_reduce_partials")
    return out[:cnt.value]


def finalize_partials(op: str, dtype, partials: torch.Tensor, init=None, out: torch.Tensor | None = None,
                      stream=None) -> torch.Tensor:
    """The second level on the GPU (one warp): init ⊕ fold of the slots, in index order."""
    dt = dtype_code(dtype)
    if out is None:
        out = torch.empty(1, dtype=TORCH_OF[dt], device=partials.device)
    box = _scalar(dt, init)
    _check(lib.ipm_finalize_partials(op_code(op), dt, partials.data_ptr(), partials.numel(),
                                     None if box is None else box.ctypes.data, out.data_ptr(), _stream(stream)),
           "ipm_finalize_partials")
    return out


def reduce_2d(op: str, t: torch.Tensor, rows: int | None = None, cols: int | None = None,
              row_stride: int | None = None, init=None, ws: torch.Tensor | None = None, stream=None):
    """One scalar over a strided 2-D region: init ⊕ fold_{r,j} t[r*row_stride + j] (a 2-D tensor view with
    unit column stride works directly, e.g. ``big[:, 10:500]``). Returns a numpy scalar."""
    if not t.is_cuda:
        raise ValueError("expected a CUDA tensor")
    dt = DTYPES[t.dtype]
    if t.dim() == 2 and rows is None:
        rows, cols = t.shape
        row_stride = t.stride(0) if rows > 1 else cols
        if cols > 1 and t.stride(1) != 1:
            raise ValueError("columns must be contiguous")
    elif rows is None or cols is None:
        raise ValueError("rows and cols are required for a flat tensor")
    row_stride = cols if row_stride is None else row_stride
    _check_region(t, rows, cols, row_stride)
    s = _stream(stream)
    ws = workspace(s) if ws is None else ws
    box = _scalar(dt, identity_value(op, dt) if init is None else init)
    _check(lib.ipm_reduce_2d(op_code(op), dt, t.data_ptr(), rows, cols, row_stride, box.ctypes.data, ws.data_ptr(), s),
           "ipm_reduce_2d")
    return box[0]


FUSED = {"sum_sumsq": 0, "dot": 1, "minmax": 2, "stats": 3}


def reduce_fused_async(sig: str, x: torch.Tensor, y: torch.Tensor | None = None, init=None,
                       out: torch.Tensor | None = None, ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
    """Several reduction variables in one pass (ipm_reduce_fused_async): sum_sumsq -> [Σx, Σx²], dot -> [Σxy],
    minmax -> [min, max], stats -> [Σx, Σx², min, max]; returns a CUDA tensor of the variables."""
    f = FUSED[sig]
    ptr, n, dt = _flat_arg(x)
    yp = 0
    if f == FUSED["dot"]:
        if y is None or y.numel() != n or y.dtype != x.dtype or y.device != x.device:
            raise ValueError("dot needs y with the same length, dtype and device")
        yp = _flat_arg(y)[0]
    nv = lib.ipm_fused_nvars(f)
    if out is None:
        out = torch.empty(nv, dtype=x.dtype, device=x.device)
    else:
        _check_out(out, x, nv)
    if init is not None and np.size(init) != nv:
        raise ValueError(f"{sig} carries {nv} variables: init needs {nv} values")
    ws = workspace(stream) if ws is None else ws
    box = None if init is None else np.ascontiguousarray(init, dtype=NP_OF[dt])
    _check(lib.ipm_reduce_fused_async(f, dt, ptr, yp or None, n, None if box is None else box.ctypes.data,
                                      out.data_ptr(), ws.data_ptr(), _stream(stream)), "ipm_reduce_fused_async")
    return out


def reduce_fused(sig: str, x: torch.Tensor, y: torch.Tensor | None = None, init=None,
                 ws: torch.Tensor | None = None, stream=None) -> np.ndarray:
    """Blocking form: returns the variables as a numpy array (init: one value per variable, or None)."""
    if init is None:
        out = reduce_fused_async(sig, x, y, None, ws=ws, stream=stream)
        _sync(stream)
        return out.cpu().numpy()
    f = FUSED[sig]
    ptr, n, dt = _flat_arg(x)
    yp = None
    if f == FUSED["dot"]:
        if y is None or y.numel() != n or y.dtype != x.dtype or y.device != x.device:
            raise ValueError("dot needs y with the same length, dtype and device")
        yp = _flat_arg(y)[0]
    nv = lib.ipm_fused_nvars(f)
    box = np.array(init, dtype=NP_OF[dt]).reshape(-1).copy()
    if box.size != nv:
        raise ValueError(f"{sig} carries {nv} variables: init needs {nv} values")
    ws = workspace(stream) if ws is None else ws
    _check(lib.ipm_reduce_fused(f, dt, ptr, yp, n, box.ctypes.data, ws.data_ptr(), _stream(stream)),
           "ipm_reduce_fused")
    return box


def reduce_host(op: str, a, init=None, ws: torch.Tensor | None = None, stream=None):
    """End-to-end clause over a HOST array (numpy array or CPU tensor, pinned is fastest): copyin fused with
    the reduction, chunked H2D overlapped with the kernels; returns the result as a numpy scalar."""
    if isinstance(a, torch.Tensor):
        if a.is_cuda:
            raise ValueError("reduce_host takes a host array")
        a = a.contiguous()
        ptr, n, dt = a.data_ptr(), a.numel(), DTYPES[a.dtype]
        keep = a
    else:
        keep = np.ascontiguousarray(a)
        ptr, n, dt = keep.ctypes.data, keep.size, dtype_code(keep.dtype)
    ws = workspace(stream) if ws is None else ws
    box = _scalar(dt, init)
    if box is None:
        box = _scalar(dt, identity_value(op, dt))
    _check(lib.ipm_reduce_host(op_code(op), dt, ptr, n, box.ctypes.data, ws.data_ptr(), _stream(stream)),
           "ipm_reduce_host")
    del keep
    return box[0]


@functools.lru_cache(maxsize=None)
def identity_value(op: str, dt: int):
    """The identity of op on element type dt, from the library (ipm_identity): the value the synchronous calls
    start from when the variable has no original value."""
    box = np.zeros(1, dtype=NP_OF[dt])
    _check(lib.ipm_identity(op_code(op), dt, box.ctypes.data), "ipm_identity")
    return box[0]


OPTIONS = {"flat_ctas_per_sm": 0, "seg_kernel": 1, "deterministic": 2, "dist_mode": 3, "dist_timeout_ms": 4,
           "ragged_kernel": 5}
RAGGED_KERNELS = {"auto": 0, "warp": 1, "tile": 2, "rank": 3, "lpr": 4}
# "marked": reduce_ragged calls ipm_reduce_ragged_marked (two passes over scratch) instead of ipm_reduce_ragged
_ragged_marked = [False]
DIST_MODES = {"auto": 0, "p2p": 0, "nccl": 1}
SEG_KERNELS = {"auto": 0, "warp": 1, "ldg": 1, "tma": 2}


def set_option(key: str, value) -> None:
    """Process-wide tuning option (ipm_set_option): flat_ctas_per_sm (1..8, -1 default), seg_kernel
    ('auto' | 'warp' | 'tma'), ragged_kernel ('auto' | 'warp' | 'tile' | 'rank' | 'lpr', or 'marked': reduce_ragged
    then calls ipm_reduce_ragged_marked with scratch from torch's caching allocator)."""
    if key == "seg_kernel" and isinstance(value, str):
        value = SEG_KERNELS[value]
    if key == "dist_mode" and isinstance(value, str):
        value = DIST_MODES[value]
    if key == "ragged_kernel" and isinstance(value, str):
        _ragged_marked[0] = value == "marked"
        value = RAGGED_KERNELS.get(value, 0)
    _check(lib.ipm_set_option(OPTIONS[key], int(value)), "ipm_set_option")


def flat_geometry(dtype, n: int):
    g, b = ctypes.c_int(), ctypes.c_int()
    _check(lib.ipm_flat_geometry(dtype_code(dtype), n, ctypes.byref(g), ctypes.byref(b)), "ipm_flat_geometry")
    return g.value, b.value


SCHEDULES = {-1: "none", 0: "static", 1: "guided", 2: "dynamic"}


def flat_schedule(dtype, n: int) -> str:
    """Which flat kernel the library launches for n elements under the current options (ipm_flat_schedule):
    'static' (k_flat grid-stride), 'guided' (k_flat_guided), 'dynamic' (k_flat with a tile counter), 'none'."""
    s = ctypes.c_int()
    _check(lib.ipm_flat_schedule(dtype_code(dtype), n, ctypes.byref(s)), "ipm_flat_schedule")
    return SCHEDULES[s.value]


class KernelTimer:
    """Per-launch device time of the library's reduction kernels (CUDA events recorded by libipm on the
    launch stream around each kernel): ``with KernelTimer(1000) as kt: ...; kt.ms -> list of floats``."""

    def __init__(self, max_records: int = 4096):
        self.max_records = max_records
        self.ms: list[float] = []
        self.kinds: list[int] = []

    def __enter__(self):
        _check(lib.ipm_profile_enable(self.max_records), "ipm_profile_enable")
        return self

    def read(self):
        ms = np.zeros(self.max_records, np.float32)
        kinds = np.zeros(self.max_records, np.int32)
        cnt = ctypes.c_int()
        _check(lib.ipm_profile_read(ms.ctypes.data, kinds.ctypes.data, self.max_records, ctypes.byref(cnt)),
               "ipm_profile_read")
        n = min(cnt.value, self.max_records)
        self.ms, self.kinds = [float(x) for x in ms[:n]], [int(k) for k in kinds[:n]]
        return self.ms

    def __exit__(self, *exc):
        try:
            self.read()
        finally:
            lib.ipm_profile_disable()
        return False


# ------------------------------------------------------------------ data environment
def copyin(host: np.ndarray, stream=None) -> int:
    """acc `copyin(host[0:n])`: returns the device address (present-or semantics)."""
    d = ctypes.c_void_p()
    _check(lib.ipm_copyin(host.ctypes.data, host.nbytes, ctypes.byref(d), _stream(stream)), "ipm_copyin")
    return d.value


def create(host: np.ndarray, stream=None) -> int:
    d = ctypes.c_void_p()
    _check(lib.ipm_create(host.ctypes.data, host.nbytes, ctypes.byref(d), _stream(stream)), "ipm_create")
    return d.value


def present(host: np.ndarray) -> int:
    d = ctypes.c_void_p()
    _check(lib.ipm_present(host.ctypes.data, host.nbytes, ctypes.byref(d)), "ipm_present")
    return d.value


def update_device(host: np.ndarray, stream=None):
    _check(lib.ipm_update_device(host.ctypes.data, host.nbytes, _stream(stream)), "ipm_update_device")


def update_host(host: np.ndarray, stream=None):
    _check(lib.ipm_update_host(host.ctypes.data, host.nbytes, _stream(stream)), "ipm_update_host")


def copyout(host: np.ndarray, stream=None):
    _check(lib.ipm_copyout(host.ctypes.data, host.nbytes, _stream(stream)), "ipm_copyout")


def delete(host: np.ndarray, stream=None):
    _check(lib.ipm_delete(host.ctypes.data, _stream(stream)), "ipm_delete")


def present_count() -> int:
    return lib.ipm_present_count()


def as_tensor(dev_ptr: int, n: int, dtype: torch.dtype) -> torch.Tensor:
    """View a device address from the present table as a CUDA tensor (no copy, not owning)."""
    class _Holder:
        __cuda_array_interface__ = {"shape": (n,), "typestr": np.dtype(NP_OF[DTYPES[dtype]]).str,
                                    "data": (dev_ptr, False), "version": 3}
    return torch.as_tensor(_Holder(), device="cuda")


# ------------------------------------------------------------------ multi-GPU
def shard_range(n: int, rank: int, world: int):
    lo, hi = ctypes.c_int64(), ctypes.c_int64()
    _check(lib.ipm_shard_range(n, rank, world, ctypes.byref(lo), ctypes.byref(hi)), "ipm_shard_range")
    return lo.value, hi.value


class _StdoutToStderr:
    """NCCL prints its version banner on the C-level stdout during init; keep stdout for the caller's output."""

    def __enter__(self):
        import sys
        sys.stdout.flush()
        self._saved = os.dup(1)
        os.dup2(2, 1)
        return self

    def __exit__(self, *exc):
        os.dup2(self._saved, 1)
        os.close(self._saved)
        return False


class Comm:
    """One NCCL communicator per process/GPU, bootstrapped through the torch.distributed store."""

    @classmethod
    def group(cls, world: int, device: int | None = None) -> list["Comm"]:
        """`world` ranks in this process on one device (ipm_comm_init_group): fused exchange only."""
        device = torch.cuda.current_device() if device is None else device
        arr = (ctypes.c_void_p * world)()
        _check(lib.ipm_comm_init_group(arr, world, device), "ipm_comm_init_group")
        out = []
        for r in range(world):
            c = cls.__new__(cls)
            c._h = ctypes.c_void_p(arr[r])
            c.rank, c.world, c.device = r, world, device
            out.append(c)
        return out

    @classmethod
    def ipc(cls, rank: int, world: int, device: int, store, key: str = "ipm_ipc") -> "Comm":
        """Bootstrap WITHOUT NCCL (ipm_comm_create_ipc / ipm_comm_attach_ipc): the slot-buffer IPC handles travel
        through `store` (any torch.distributed Store). Fused exchange only. Every rank learns whether every other
        rank mapped all peers; if any failed, all raise."""
        torch.cuda.set_device(device)
        hb = lib.ipm_comm_ipc_handle_bytes()
        mine = ctypes.create_string_buffer(hb)
        c = cls.__new__(cls)
        c._h = ctypes.c_void_p()
        c.rank, c.world, c.device = rank, world, device
        _check(lib.ipm_comm_create_ipc(ctypes.byref(c._h), rank, world, device, mine), "ipm_comm_create_ipc")
        store.set(f"{key}/handle/{rank}", bytes(mine.raw))
        allh = b"".join(store.get(f"{key}/handle/{q}") for q in range(world))
        buf = ctypes.create_string_buffer(allh, hb * world)
        code = lib.ipm_comm_attach_ipc(c._h, buf)
        msg = lib.ipm_last_error_message().decode(errors="replace") if code else ""
        store.set(f"{key}/ok/{rank}", b"1" if code == 0 else b"0")
        oks = [store.get(f"{key}/ok/{q}") == b"1" for q in range(world)]
        if not all(oks):
            c.close()
            raise IpmError(code or 10, "Comm.ipc", msg or f"ranks {[q for q, o in enumerate(oks) if not o]} "
                                                          "could not map every peer")
        return c

    @staticmethod
    def bootstrap_id(rank: int, store, key: str = "ipm_nccl_id") -> bytes:
        """Rank 0 makes the NCCL unique id (ipm_comm_unique_id) and publishes it in `store`; every rank returns the
        same ipm_comm_id_bytes() bytes (host-only: no GPU is touched, so CPU tests drive it with gloo)."""
        nb = lib.ipm_comm_id_bytes()
        if rank == 0:
            buf = ctypes.create_string_buffer(nb)
            _check(lib.ipm_comm_unique_id(buf), "ipm_comm_unique_id")
            store.set(key, bytes(buf.raw))
        uid = store.get(key)
        if len(uid) != nb:
            raise IpmError(10, "Comm", "bad NCCL id from store")
        return uid

    def __init__(self, rank: int, world: int, device: int, store=None, key: str = "ipm_nccl_id"):
        if store is None:
            import torch.distributed as dist
            store = dist.distributed_c10d._get_default_store()
        uid = self.bootstrap_id(rank, store, key)
        self._id = ctypes.create_string_buffer(uid, len(uid))
        self._h = ctypes.c_void_p()
        torch.cuda.set_device(device)
        with _StdoutToStderr():
            _check(lib.ipm_comm_init(ctypes.byref(self._h), rank, world, self._id, device), "ipm_comm_init")
        self.rank, self.world, self.device = rank, world, device

    @property
    def fused(self) -> bool:
        """True when reduce() exchanges partials inside the reduction kernel over peer memory (no NCCL)."""
        return bool(lib.ipm_comm_uses_peer_memory(self._h))

    def close(self):
        if self._h:
            _check(lib.ipm_comm_destroy(self._h), "ipm_comm_destroy")
            self._h = ctypes.c_void_p()

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    def reduce(self, op: str, shard: torch.Tensor, init=None, ws: torch.Tensor | None = None, stream=None):
        """Every rank passes its shard and the same init; every rank returns the global result."""
        ptr, n, dt = _flat_arg(shard)
        ws = workspace(stream) if ws is None else ws
        box = _scalar(dt, identity_value(op, dt) if init is None else init)
        _check(lib.ipm_reduce_dist(self._h, op_code(op), dt, ptr, n, box.ctypes.data, ws.data_ptr(),
                                   _stream(stream)), "ipm_reduce_dist")
        return box[0]

    def reduce_host(self, op: str, host_shard, init=None, ws: torch.Tensor | None = None, stream=None):
        """End to end: this rank's HOST shard (numpy array or CPU tensor, pinned fastest) is streamed to the GPU,
        reduced and exchanged (ipm_reduce_host_dist); every rank returns the global result."""
        if isinstance(host_shard, torch.Tensor):
            if host_shard.is_cuda:
                raise ValueError("reduce_host takes a host array")
            keep = host_shard.contiguous()
            ptr, n, dt = keep.data_ptr(), keep.numel(), DTYPES[keep.dtype]
        else:
            keep = np.ascontiguousarray(host_shard)
            ptr, n, dt = keep.ctypes.data, keep.size, dtype_code(keep.dtype)
        ws = workspace(stream) if ws is None else ws
        box = _scalar(dt, init)
        if box is None:
            box = _scalar(dt, identity_value(op, dt))
        _check(lib.ipm_reduce_host_dist(self._h, op_code(op), dt, ptr, n, box.ctypes.data, ws.data_ptr(),
                                        _stream(stream)), "ipm_reduce_host_dist")
        del keep
        return box[0]

    def reduce_async(self, op: str, shard: torch.Tensor, init=None, out: torch.Tensor | None = None,
                     ws: torch.Tensor | None = None, stream=None) -> torch.Tensor:
        ptr, n, dt = _flat_arg(shard)
        if out is None:
            out = torch.empty(1, dtype=shard.dtype, device=shard.device)
        else:
            _check_out(out, shard, 1)
        ws = workspace(stream) if ws is None else ws
        box = _scalar(dt, init)
        _check(lib.ipm_reduce_dist_async(self._h, op_code(op), dt, ptr, n, None if box is None else box.ctypes.data,
                                         out.data_ptr(), ws.data_ptr(), _stream(stream)), "ipm_reduce_dist_async")
        return out
