"""CPU-side checks of the C-ABI boundary: libipm loads, exports every symbol include/ipm.h declares, and its
host-only logic (legality table, validation before any CUDA call, shard ranges) behaves as documented."""
import ctypes
import os
import re

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def ipm():
    from tools import build
    build.build_ipm()
    from paper_1412_1127_b200 import ipm as m
    return m


def header_functions():
    src = open(os.path.join(ROOT, "include", "ipm.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(ipm_[a-z_0-9]+)\s*\(", src)))


def test_exports_every_declared_symbol(ipm):
    names = header_functions()
    assert len(names) >= 28
    nm = os.popen(f"nm -D --defined-only {ipm.LIB_PATH}").read()
    exported = set(re.findall(r"\bT (ipm_[a-z_0-9]+)", nm))
    missing = [n for n in names if n not in exported]
    assert not missing, missing
    assert set(ipm.EXPORTED) == set(names)


def test_no_oracle_in_product():
    # the product path shares no code with the oracle and never loads it
    nm = os.popen(f"nm -D {os.path.join(ROOT, 'paper_1412_1127_b200', 'libipm.so')}").read()
    assert "ora_" not in nm
    for f in os.listdir(os.path.join(ROOT, "paper_1412_1127_b200")):
        if f.endswith(".py"):
            txt = open(os.path.join(ROOT, "paper_1412_1127_b200", f)).read()
            assert "import oracle" not in txt and "from oracle" not in txt
    for f in os.listdir(os.path.join(ROOT, "paper_1412_1127_b200", "csrc")):
        txt = open(os.path.join(ROOT, "paper_1412_1127_b200", "csrc", f)).read()
        assert "oracle" not in txt.lower()


def test_legality_table(ipm):
    import torch
    legal = [(op, dt) for op in ipm.OPS for dt in ipm.DTYPES if ipm.legal(op, dt)]
    assert len(legal) == 30
    for op in "&|^":
        assert not ipm.legal(op, torch.float32) and not ipm.legal(op, torch.float64)
        assert ipm.legal(op, torch.int32) and ipm.legal(op, torch.int64)


def test_status_strings(ipm):
    for i, s in enumerate(ipm.STATUS):
        assert ipm.lib.ipm_status_str(i).decode() == s


def test_validation_before_cuda(ipm):
    """argument errors are reported without touching the GPU (fake non-NULL pointers are never dereferenced)"""
    L = ipm.lib
    ws = ctypes.c_void_p(0x10000)  # 256-aligned fake address
    dev = ctypes.c_void_p(0x20000)
    out = ctypes.c_void_p(0x30000)
    box = (ctypes.c_int32 * 1)(0)
    assert L.ipm_reduce_async(4, 2, dev, 10, None, out, ws, None) == 1        # & on float32: IPM_E_REDOP
    assert L.ipm_reduce_async(9, 0, dev, 10, None, out, ws, None) == 1        # unknown op
    assert L.ipm_reduce_async(0, 7, dev, 10, None, out, ws, None) == 2        # unknown dtype
    assert L.ipm_reduce_async(0, 0, None, 10, None, out, ws, None) == 3       # NULL array, n > 0
    assert L.ipm_reduce_async(0, 0, dev, -1, None, out, ws, None) == 4        # negative n
    assert L.ipm_reduce_async(0, 0, ctypes.c_void_p(0x20001), 10, None, out, ws, None) == 6  # misaligned
    assert L.ipm_reduce_async(0, 0, dev, 10, None, out, ctypes.c_void_p(0x10010), None) == 7  # ws alignment
    assert L.ipm_reduce_async(0, 0, dev, 10, None, out, None, None) == 7
    assert L.ipm_reduce(0, 0, dev, 10, None, ws, None) == 3                   # NULL inout
    assert L.ipm_reduce_segmented(0, 0, dev, 5, 10, 9, None, out, ws, None) == 4   # row_stride < cols
    assert L.ipm_reduce_segmented(5, 3, dev, 5, 10, 10, None, out, ws, None) == 1  # | on float64
    assert L.ipm_reduce_host(0, 0, None, 10, box, ws, None) == 3
    assert "illegal" in L.ipm_last_error_message().decode() or L.ipm_last_error_message()
    # marked ragged rows: scratch size from the element count (bitmap bit per element + a count per chunk)
    offs, scr = ctypes.c_void_p(0x40000), ctypes.c_void_p(0x50000)
    need = L.ipm_ragged_scratch_bytes(2, 1 << 20, 100)
    assert (1 << 20) // 8 < need <= (1 << 20) // 8 + (1 << 20) // 256 * 4 + 1024
    assert need % 256 == 0 and L.ipm_ragged_scratch_bytes(3, 1 << 20, 100) > need  # 8-byte types: half-size chunks
    assert L.ipm_ragged_scratch_bytes(2, 1 << 20, 1 << 20) >= need + (1 << 20) // 8  # + a bit per row
    assert L.ipm_reduce_ragged_marked(0, 2, dev, 1 << 20, offs, 100, None, out, ws, scr, need - 256, None) == 7
    assert L.ipm_reduce_ragged_marked(0, 2, dev, 1 << 20, offs, 100, None, out, ws, ctypes.c_void_p(0x50010),
                                      need, None) == 6                        # scratch alignment
    assert L.ipm_reduce_ragged_marked(4, 2, dev, 1 << 20, offs, 100, None, out, ws, scr, need, None) == 1
    assert L.ipm_reduce_ragged_marked(0, 2, dev, 1 << 20, None, 100, None, out, ws, scr, need, None) == 3
    assert L.ipm_reduce_ragged_marked(0, 2, dev, -1, offs, 100, None, out, ws, scr, need, None) == 4
    assert L.ipm_reduce_ragged_marked(0, 2, dev, 1 << 20, offs, 0, None, out, ws, scr, need, None) == 0  # no rows


def test_present_table_errors(ipm):
    import numpy as np
    a = np.zeros(16, np.float32)
    with pytest.raises(ipm.IpmError) as e:
        ipm.present(a)
    assert e.value.status == "IPM_E_PRESENT"
    with pytest.raises(ipm.IpmError):
        ipm.copyout(a, stream=0)
    with pytest.raises(ipm.IpmError):
        ipm.delete(a, stream=0)
    assert ipm.present_count() == 0


def test_shard_ranges(ipm):
    for n in [0, 1, 7, 8, 1000, 2**34, 2**34 + 3, 2**62]:
        for P in [1, 2, 3, 4, 8, 64]:
            rs = [ipm.shard_range(n, r, P) for r in range(P)]
            assert rs[0][0] == 0 and rs[-1][1] == n
            assert all(rs[i][1] == rs[i + 1][0] for i in range(P - 1))          # contiguous, no overlap
            sizes = [hi - lo for lo, hi in rs]
            assert max(sizes) - min(sizes) <= 1                                   # balanced
            assert all(lo == (n * r) // P for r, (lo, _) in enumerate(rs))        # the documented formula
    with pytest.raises(ipm.IpmError):
        ipm.shard_range(10, 3, 3)
    with pytest.raises(ipm.IpmError):
        ipm.shard_range(-1, 0, 1)


def test_workspace_layout(ipm):
    assert ipm.WS_BYTES >= 8192 + 8 * 4096
    assert ipm.lib.ipm_comm_id_bytes() == 128


def test_identity_matches_oracle(ipm):
    """ipm_identity (the start value of the synchronous calls when the variable has none) equals the oracle's
    empty fold for all 30 legal pairs, bit for bit; illegal pairs are refused."""
    import numpy as np
    import oracle
    NP = {"int32": np.int32, "int64": np.int64, "float32": np.float32, "float64": np.float64}
    U = {"int32": np.uint32, "int64": np.uint64, "float32": np.uint32, "float64": np.uint64}
    n = 0
    for op in ipm.OPS:
        for dt in NP:
            code = {"int32": 0, "int64": 1, "float32": 2, "float64": 3}[dt]
            box = np.zeros(1, NP[dt])
            rc = ipm.lib.ipm_identity(ipm.OPS[op], code, box.ctypes.data)
            if not oracle.legal(op, dt):
                assert rc == 1  # IPM_E_REDOP
                continue
            assert rc == 0
            want = np.array([oracle.identity(op, dt)], NP[dt])
            assert box.view(U[dt])[0] == want.view(U[dt])[0], (op, dt, box, want)
            n += 1
    assert n == 30
    assert ipm.lib.ipm_identity(0, 0, None) == 3


def test_flat_schedule_query(ipm):
    import torch
    assert ipm.flat_schedule(torch.float32, 0) == "none"
    assert ipm.flat_schedule(torch.float32, 1 << 24) == "static"
    assert ipm.flat_schedule(torch.float32, (1 << 24) + 1) == "guided"
    ipm.set_option("deterministic", 0)
    try:
        assert ipm.flat_schedule(torch.int64, 1 << 30) == "dynamic"
        ipm.set_option("deterministic", 2)
        assert ipm.flat_schedule(torch.int64, 1 << 30) == "static"
    finally:
        ipm.set_option("deterministic", 1)
