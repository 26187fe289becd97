"""GPU parity at the sizes where the PRODUCTION schedules run (VERDICT r01 "parity sweeps stop below the size where
the production schedule starts"): the flat clause above 64 MiB goes through k_flat_guided (about 90 % of the tiles
dealt statically, the rest in dynamically claimed chunks plus one remainder chunk); IPM_OPT_DETERMINISTIC 0 / 2
select the dynamic / static k_flat; the strided 2-D kernel and the several-variables kernel step through more
than one round of work items; the paper's two-level pieces (ipm_reduce_partials + ipm_finalize_partials,
PAPER.md:205) are compared with the oracle for all 30 (op, dtype) pairs. Every case asserts which schedule ran
(ipm_flat_schedule, the same decision function the launch uses). Oracle = the plain left fold (oracle/), compared
bit-exactly for exact ops and within 1e-5 / 1e-12 for float + * (BASELINE.json north_star)."""
import numpy as np
import pytest
import torch

import ipmgen
import oracle
from test_gpu_parity import DTS, LEGAL, NPT, TD, TOL, bits, check, device_input, workload

pytestmark = pytest.mark.gpu

BIG = {"int32": 20_000_005, "float32": 20_000_005, "int64": 10_000_007, "float64": 10_000_007}  # 80 MB > 64 MiB


@pytest.fixture(scope="module")
def ipm():
    from paper_1412_1127_b200 import ipm as m
    return m


def guided_layout(ipm, t: torch.Tensor):
    """Element ranges of k_flat_guided's schedule for tensor t (ipm_kernels.cuh k_flat_guided): the static part,
    the dynamic chunks and the remainder chunk (vectors past the last whole tile + head + tail scalars)."""
    n, es = t.numel(), t.element_size()
    vw = 32 // es
    g, block = ipm.flat_geometry(t.dtype, n)
    head = min(n, ((32 - (t.data_ptr() & 31)) & 31) // es)
    nv = (n - head) // vw
    tile = block * 2 * vw  # elements per tile (BLOCK threads x U = 2 vectors)
    ntiles = nv // (block * 2)
    dyn0 = (ntiles - ntiles // 10) // g * g
    return {"static": (head, head + dyn0 * tile), "dynamic": (head + dyn0 * tile, head + ntiles * tile),
            "remainder": (head + ntiles * tile, n), "head": head, "grid": g}


@pytest.mark.parametrize("op,dt", LEGAL)
def test_guided_parity_every_pair(ipm, op, dt):
    """> 64 MiB, misaligned start, init != identity: the guided schedule's static tiles, dynamic chunks and
    remainder chunk all contribute."""
    n = BIG[dt]
    spec = workload(op, dt, n, seed=77)
    x = device_input(spec, offset=3)
    assert ipm.flat_schedule(x.dtype, n) == "guided"
    lay = guided_layout(ipm, x)
    assert lay["dynamic"][1] > lay["dynamic"][0] and lay["remainder"][1] > lay["remainder"][0] and lay["head"] > 0
    init = NPT[dt](5)
    got = ipm.reduce(op, x, init=init)
    want_t, want_ld = oracle.reduce(op, ipmgen.fill_host(spec), init=init)
    check(op, dt, got, want_t, want_ld)
    # repeated runs give identical bits (the guided schedule fixes every fold order)
    assert bits(ipm.reduce(op, x, init=init), dt) == bits(got, dt)


def _upload(a: np.ndarray, offset: int) -> torch.Tensor:
    buf = torch.empty(a.size + offset + 1, dtype=TD[a.dtype.name], device="cuda")
    v = buf[offset:offset + a.size]
    v.copy_(torch.from_numpy(a))
    return v


@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_guided_float_edges_in_dynamic_and_remainder(ipm, dt):
    """NaN and -0 planted inside a dynamically claimed chunk and inside the remainder chunk (R10, R5)."""
    n = BIG[dt]
    NaN, negz = NPT[dt](np.nan), NPT[dt](-0.0)
    base_neg = -np.abs(ipmgen.fill_host(ipmgen.Spec(dt, n, "signed", seed=5))) - NPT[dt](1)   # all < 0
    base_pos = -base_neg                                                                           # all > 0
    probe = _upload(base_neg, 5)
    lay = guided_layout(ipm, probe)
    d_mid = (lay["dynamic"][0] + lay["dynamic"][1]) // 2
    r_mid = (lay["remainder"][0] + lay["remainder"][1]) // 2
    del probe
    cases = []
    # max over negatives: -0 in a dynamic chunk is the maximum; a +0 in the remainder beats it; NaN absorbs
    a = base_neg.copy(); a[d_mid] = negz; cases.append(("max", a))
    a = base_neg.copy(); a[d_mid] = negz; a[r_mid] = NPT[dt](0.0); cases.append(("max", a))
    a = base_neg.copy(); a[r_mid] = NaN; cases.append(("max", a))
    a = base_neg.copy(); a[d_mid] = NaN; cases.append(("max", a))
    # min over positives: +0 in the remainder, -0 in a dynamic chunk below it, NaN in either
    a = base_pos.copy(); a[r_mid] = NPT[dt](0.0); cases.append(("min", a))
    a = base_pos.copy(); a[r_mid] = NPT[dt](0.0); a[d_mid] = negz; cases.append(("min", a))
    a = base_pos.copy(); a[d_mid] = NaN; cases.append(("min", a))
    a = base_pos.copy(); a[r_mid] = NaN; cases.append(("min", a))
    # &&: -0 is false (in a dynamic chunk / in the remainder); NaN is true
    a = base_pos.copy(); a[d_mid] = negz; cases.append(("&&", a))
    a = base_pos.copy(); a[r_mid] = negz; cases.append(("&&", a))
    a = base_pos.copy(); a[d_mid] = NaN; cases.append(("&&", a))
    # ||: all zeros with -0s stays false; one NaN (dynamic / remainder) makes it true
    z = np.zeros(n, NPT[dt]); z[::7] = negz
    cases.append(("||", z.copy()))
    a = z.copy(); a[r_mid] = NaN; cases.append(("||", a))
    a = z.copy(); a[d_mid] = NaN; cases.append(("||", a))
    for op, a in cases:
        x = _upload(a, 5)
        assert guided_layout(ipm, x)["dynamic"] == lay["dynamic"]   # same alignment -> same layout
        assert ipm.flat_schedule(x.dtype, n) == "guided"
        got = ipm.reduce(op, x)
        want = oracle.reduce(op, a)[0]
        assert bits(got, dt) == bits(want, dt), (op, got, want)
        del x


@pytest.mark.parametrize("det,sched", [(0, "dynamic"), (1, "guided"), (2, "static")])
@pytest.mark.parametrize("cps", [1, 2, 8])
def test_options_reach_their_kernels(ipm, det, sched, cps):
    """IPM_OPT_DETERMINISTIC 0 / 1 / 2 and IPM_OPT_FLAT_CTAS_PER_SM above 64 MiB: the schedule they name runs
    and the results equal the oracle's."""
    ipm.set_option("flat_ctas_per_sm", cps)
    ipm.set_option("deterministic", det)
    try:
        for op, dt, n in [("+", "float64", 10_000_011), ("^", "int32", 20_000_001), ("max", "float32", 17_777_777),
                          ("*", "int64", 9_000_001), ("+", "float32", 20_000_037)]:
            spec = workload(op, dt, n, seed=cps * 10 + det)
            x = device_input(spec, offset=1)
            assert ipm.flat_schedule(x.dtype, n) == sched
            want_t, want_ld = oracle.reduce(op, ipmgen.fill_host(spec), init=NPT[dt](2))
            check(op, dt, ipm.reduce(op, x, init=NPT[dt](2)), want_t, want_ld)
            if det != 0:  # deterministic schedules: identical bits run to run
                assert bits(ipm.reduce(op, x, init=NPT[dt](2)), dt) == bits(ipm.reduce(op, x, init=NPT[dt](2)), dt)
    finally:
        ipm.set_option("flat_ctas_per_sm", -1)
        ipm.set_option("deterministic", 1)


def test_small_inputs_take_the_static_schedule(ipm):
    assert ipm.flat_schedule(torch.float32, 0) == "none"
    assert ipm.flat_schedule(torch.float32, 1 << 20) == "static"
    assert ipm.flat_schedule(torch.float32, 1 << 24) == "static"        # exactly 64 MiB
    assert ipm.flat_schedule(torch.float32, (1 << 24) + 1) == "guided"
    assert ipm.flat_schedule(torch.float64, (1 << 23) + 1) == "guided"


# --------------------------------------------------------------------------- the paper's two levels, all pairs

@pytest.mark.parametrize("op,dt", LEGAL)
def test_partials_then_finalize_parity(ipm, op, dt):
    """ipm_reduce_partials (one partial per thread block, the paper's GPU level) + ipm_finalize_partials (the
    second level, here one warp on the GPU instead of the paper's host loop) == the oracle."""
    for k, n in enumerate([0, 1, 1000, (1 << 20) + 3, BIG[dt]]):
        spec = workload(op, dt, n, seed=k + 40)
        x = device_input(spec, offset=k % 4)
        parts = ipm.reduce_partials(op, x)
        assert parts.numel() == ipm.flat_geometry(x.dtype, n)[0]
        init = NPT[dt](3)
        got = ipm.finalize_partials(op, x.dtype, parts, init=init).cpu().numpy()[0]
        want_t, want_ld = oracle.reduce(op, ipmgen.fill_host(spec), init=init)
        check(op, dt, got, want_t, want_ld)
        # without init: the identity start
        got0 = ipm.finalize_partials(op, x.dtype, parts).cpu().numpy()[0]
        want_t0, want_ld0 = oracle.reduce(op, ipmgen.fill_host(spec))
        check(op, dt, got0, want_t0, want_ld0)


# --------------------------------------------------------------------------- strided 2-D, several rounds

def _region(h, rows, cols, stride):
    return np.ascontiguousarray(np.lib.stride_tricks.as_strided(h, shape=(rows, cols),
                                                                strides=(stride * h.itemsize, h.itemsize))).ravel()


@pytest.mark.parametrize("op,dt", LEGAL)
def test_2d_multi_round_parity(ipm, op, dt):
    """More (row, chunk) work items than resident warps (148 SMs x 3-4 CTAs x 8 warps), so every warp steps
    through several items: long rows split into many chunks, and many short rows with one item each."""
    for k, (rows, cols, stride) in enumerate([(3000, 5000, 5003), (100_000, 33, 40), (700, 20_001, 20_009)]):
        total = (rows - 1) * stride + cols
        spec = workload(op, dt, total, seed=k + 60)
        x = device_input(spec, offset=k + 1)
        init = NPT[dt](2)
        got = ipm.reduce_2d(op, x, rows=rows, cols=cols, row_stride=stride, init=init)
        want_t, want_ld = oracle.reduce(op, _region(ipmgen.fill_host(spec), rows, cols, stride), init=init)
        check(op, dt, got, want_t, want_ld)


@pytest.mark.slow
def test_2d_bench_window(ipm):
    """The bench suite's 16384 x 16000 window of a 16384 x 16384 float32 image, against the oracle."""
    rows, cols, stride = 16384, 16000, 16384
    for op, dt in [("+", "float32"), ("max", "float32"), ("^", "int32")]:
        spec = workload(op, dt, rows * stride, seed=1)
        x = device_input(spec)
        got = ipm.reduce_2d(op, x, rows=rows, cols=cols, row_stride=stride)
        want_t, want_ld = oracle.reduce(op, _region(ipmgen.fill_host(spec), rows, cols, stride))
        check(op, dt, got, want_t, want_ld)
        del x
        torch.cuda.empty_cache()


# --------------------------------------------------------------------------- several variables, several rounds

@pytest.mark.parametrize("dt", DTS)
@pytest.mark.parametrize("sig", ["sum_sumsq", "dot", "minmax", "stats"])
def test_fused_multi_round_parity(ipm, sig, dt):
    """n well above one grid-wide round of k_fused's tiles (4 rounds for 4-byte, 8 for 8-byte elements)."""
    n = 10_000_003
    kind = "signed" if sig in ("minmax", "stats") else "random"
    sx = ipmgen.Spec(dt, n, kind, seed=91)
    sy = ipmgen.Spec(dt, n, kind, seed=92)
    hx, hy = ipmgen.fill_host(sx), ipmgen.fill_host(sy)
    nv = {"sum_sumsq": 2, "dot": 1, "minmax": 2, "stats": 4}[sig]
    ops = {"sum_sumsq": ["+", "+"], "dot": ["+"], "minmax": ["min", "max"], "stats": ["+", "+", "min", "max"]}[sig]
    init = np.arange(1, nv + 1).astype(NPT[dt])
    want_t, want_ld = oracle.reduce_fused(sig, hx, hy if sig == "dot" else None, init=init)
    for offx, offy in [(0, 0), (3, 3), (1, 2)]:
        x = device_input(sx, offx)
        y = device_input(sy, offy)
        got = ipm.reduce_fused(sig, x, y if sig == "dot" else None, init=init)
        for v, op in enumerate(ops):
            check(op, dt, got[v], want_t[v], want_ld[v])


@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_float_edges_segmented_and_2d(ipm, dt):
    """IEEE maximum / minimum and C truthiness (R10, R5) through the row kernels and the 2-D kernel: rows of
    negatives with a -0 / +0 / NaN planted at varying lanes and positions, against the oracle row by row."""
    rows, cols, stride = 300, 1000, 1003
    base = -np.abs(ipmgen.fill_host(ipmgen.Spec(dt, rows * stride, "signed", seed=8))) - NPT[dt](1)
    rng = np.random.default_rng(3)
    for op in ("max", "min", "&&", "||"):
        a = base.copy() if op != "min" else -base
        if op == "||":
            a = np.zeros_like(base)
            a[::3] = NPT[dt](-0.0)
        r_idx = rng.integers(0, rows, 60)
        c_idx = rng.integers(0, cols, 60)
        for j, (r, c) in enumerate(zip(r_idx, c_idx)):
            v = [NPT[dt](-0.0), NPT[dt](0.0), NPT[dt](np.nan)][j % 3]
            a[r * stride + c] = v
        x = _upload(a, 1)
        for kern in ("warp", "tma"):
            ipm.set_option("seg_kernel", kern)
            got = ipm.reduce_segmented(op, x, rows=rows, cols=cols, row_stride=stride).cpu().numpy()
            want, _ = oracle.reduce_segmented(op, a, rows, cols, stride)
            assert got.tobytes() == want.tobytes(), (op, kern)
        ipm.set_option("seg_kernel", "auto")
        got = ipm.reduce_2d(op, x, rows=rows, cols=cols, row_stride=stride)
        want = oracle.reduce(op, _region(a, rows, cols, stride))[0]
        assert bits(got, dt) == bits(want, dt), op
