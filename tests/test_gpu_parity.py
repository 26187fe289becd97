"""GPU parity: the CUDA path (through the C ABI) against the CPU oracle, element by element on the same seeded
inputs. Bit-exact for integer, bitwise, logical, max and min; |g - o| <= tol*|o| for float + and * with
tol = 1e-5 (float32) / 1e-12 (float64) against the oracle's long double value (BASELINE.json north_star)."""
import ctypes
import os
import time

import numpy as np
import pytest
import torch

import ipmgen
import oracle

pytestmark = pytest.mark.gpu

OPS = ["+", "*", "max", "min", "&", "|", "^", "&&", "||"]
DTS = ["int32", "int64", "float32", "float64"]
TD = {"int32": torch.int32, "int64": torch.int64, "float32": torch.float32, "float64": torch.float64}
NPT = {"int32": np.int32, "int64": np.int64, "float32": np.float32, "float64": np.float64}
TOL = {"float32": 1e-5, "float64": 1e-12}
LEGAL = [(o, d) for o in OPS for d in DTS if not (d.startswith("float") and o in "&|^")]


@pytest.fixture(scope="module")
def ipm():
    from paper_1412_1127_b200 import ipm as m
    return m


def workload(op, dt, n, seed):
    """the input recipe of DESIGN.md for each op (values where the op is well conditioned and non-degenerate)"""
    if op == "*":
        if dt.startswith("float"):
            return ipmgen.Spec(dt, n, "signs", seed=seed, plant="factor", nplant=64)
        return ipmgen.Spec(dt, n, "odd", seed=seed)
    if op in ("max", "min"):
        return ipmgen.Spec(dt, n, "signed", seed=seed)
    if op == "&":
        return ipmgen.Spec(dt, n, "allbits", seed=seed, plant="clearbit", nplant=8)
    if op == "|":
        return ipmgen.Spec(dt, n, "const", param=0, seed=seed, plant="setbit", nplant=8)
    if op == "&&":
        return ipmgen.Spec(dt, n, "nonzero", seed=seed, plant="value", nplant=1 if seed % 2 else 0, plant_param=0)
    if op == "||":
        return ipmgen.Spec(dt, n, "const", param=0, seed=seed, plant="value", nplant=1 if seed % 2 else 0,
                           plant_param=3)
    return ipmgen.Spec(dt, n, "random", seed=seed)


def device_input(spec, offset=0):
    """the spec's elements in a fresh CUDA buffer starting `offset` elements past a 256-byte boundary"""
    buf = torch.empty(spec.n + offset + 1, dtype=TD[spec.dtype], device="cuda")
    view = buf[offset:offset + spec.n]
    if spec.n:
        ipmgen.fill_device(spec, view.data_ptr(), 0, spec.n, torch.cuda.current_stream().cuda_stream)
    return view


def bits(x, dt):
    return np.array([x], dtype=NPT[dt]).view(np.uint32 if dt.endswith("32") else np.uint64)[0]


def check(op, dt, got, want_t, want_ld):
    if dt.startswith("float") and op in ("+", "*"):
        g = np.longdouble(got)
        assert abs(g - want_ld) <= TOL[dt] * abs(want_ld) or g == want_ld, (op, dt, got, want_ld)
    else:
        assert bits(got, dt) == bits(want_t, dt), (op, dt, got, want_t)


# --------------------------------------------------------------------------- generator: device == host

@pytest.mark.parametrize("dt", DTS)
@pytest.mark.parametrize("kind", ["random", "signed", "odd", "iota", "mod", "signs", "allbits", "nonzero"])
def test_generator_device_equals_host(dt, kind):
    spec = ipmgen.Spec(dt, 1_000_003, kind, seed=17, param=1024 if kind == "mod" else 5,
                       plant="factor" if dt.startswith("float") else "clearbit", nplant=33)
    d = device_input(spec).cpu().numpy()
    h = ipmgen.fill_host(spec)
    assert d.tobytes() == h.tobytes()
    # a sub-range fill (lo > 0), as the sharded path uses
    lo = 123_457
    part = torch.empty(5000, dtype=TD[dt], device="cuda")
    ipmgen.fill_device(spec, part.data_ptr(), lo, 5000, torch.cuda.current_stream().cuda_stream)
    assert part.cpu().numpy().tobytes() == h[lo:lo + 5000].tobytes()


# --------------------------------------------------------------------------- flat clause, every (op, dtype)

SIZES = [0, 1, 2, 3, 7, 8, 9, 31, 32, 33, 255, 256, 257, 1000, 1023, 1024, 1025, 4095, 4096, 4097, 65_537,
         (1 << 20) + 3]


@pytest.mark.parametrize("op,dt", LEGAL)
def test_flat_parity_sizes(ipm, op, dt):
    for i, n in enumerate(SIZES):
        spec = workload(op, dt, n, seed=i + 1)
        x = device_input(spec, offset=i % 8)  # misaligned starts exercise the head/tail peel
        init = NPT[dt](3)
        got = ipm.reduce(op, x, init=init)
        want_t, want_ld = oracle.reduce(op, ipmgen.fill_host(spec), init=init)
        check(op, dt, got, want_t, want_ld)


@pytest.mark.parametrize("op,dt", LEGAL)
def test_flat_no_init_is_identity_start(ipm, op, dt):
    spec = workload(op, dt, 100_000, seed=5)
    x = device_input(spec)
    got = ipm.reduce(op, x)
    want_t, want_ld = oracle.reduce(op, ipmgen.fill_host(spec))
    check(op, dt, got, want_t, want_ld)
    # the identity itself (n = 0, no init): the library's finalize kernel, the synchronous call (which starts
    # from the binding's host-side identity table) and that table all agree with the oracle
    want = bits(oracle.identity(op, dt), dt)
    assert bits(ipm.reduce_async(op, x[:0]).cpu().numpy()[0], dt) == want
    assert bits(ipm.reduce(op, x[:0]), dt) == want
    assert bits(ipm.identity_value(op, ipm.dtype_code(TD[dt])), dt) == want


@pytest.mark.parametrize("dt", DTS)
def test_flat_seeds_and_determinism(ipm, dt):
    # 30 seeds; run twice -> identical bits (fixed fold order)
    for seed in range(30):
        spec = workload("+", dt, 4096 + 37 * seed, seed)
        x = device_input(spec)
        a = ipm.reduce("+", x)
        b = ipm.reduce("+", x)
        assert bits(a, dt) == bits(b, dt)
        want_t, want_ld = oracle.reduce("+", ipmgen.fill_host(spec))
        check("+", dt, a, want_t, want_ld)


def test_spec_worked_examples(ipm):
    x = torch.arange(1, 1025, dtype=torch.int32, device="cuda")
    assert ipm.reduce("+", x, init=np.int32(0)) == 524800
    assert ipm.reduce("max", torch.tensor([3, -1, 7], dtype=torch.int32, device="cuda")) == 7


@pytest.mark.parametrize("dt", ["float32", "float64"])
def test_float_edge_semantics(ipm, dt):
    T = TD[dt]
    t = lambda v: torch.tensor(v, dtype=T, device="cuda")
    for vals in ([-0.0, 0.0], [0.0, -0.0], [-0.0, -0.0, -1.0], [1.0, float("nan"), 2.0], [float("-inf")],
                 [-float("nan"), -5.0], [0.0] * 100 + [-0.0] * 100):
        a = np.array(vals, NPT[dt])
        for op in ("max", "min", "&&", "||"):
            got = ipm.reduce(op, t(vals))
            want, _ = oracle.reduce(op, a)
            assert bits(got, dt) == bits(want, dt), (op, vals, got, want)
    # NaN / -0 anywhere in a long array, every lane position
    for pos in [0, 5, 31, 32, 1000, 99_999]:
        a = ipmgen.fill_host(ipmgen.Spec(dt, 100_000, "signed", seed=pos))
        a[pos] = np.nan
        for op in ("max", "min", "&&", "||"):
            assert bits(ipm.reduce(op, torch.from_numpy(a).cuda()), dt) == bits(oracle.reduce(op, a)[0], dt)


@pytest.mark.parametrize("dt", ["int32", "int64"])
def test_int_edges(ipm, dt):
    info = np.iinfo(NPT[dt])
    for vals in ([info.min, info.min], [info.max] * 3, [-1, 5, -7], [1 << 31 if dt == "int64" else 1, 0]):
        a = np.array(vals, NPT[dt])
        for op in ("max", "min", "&&", "||", "+", "*", "&", "|", "^"):
            assert bits(ipm.reduce(op, torch.from_numpy(a).cuda()), dt) == bits(oracle.reduce(op, a)[0], dt)
    if dt == "int64":  # truthiness of high bits (a 32-bit truncation would get these wrong)
        a = np.array([1 << 32, 1 << 63 if False else -(1 << 63), 1 << 40], np.int64)
        assert ipm.reduce("&&", torch.from_numpy(a).cuda()) == 1
        z = np.zeros(1000, np.int64); z[777] = 1 << 33
        assert ipm.reduce("||", torch.from_numpy(z).cuda()) == 1


def test_exactly_once(ipm):
    # Σ 1 = n and Σ h(i) mod 2^64 over the iteration space: a dropped or duplicated element changes them
    for n in [1, 255, 256, 257, 1000, 1024, (1 << 22) + 5, 10_000_019]:
        ones = torch.ones(n, dtype=torch.int64, device="cuda")
        assert ipm.reduce("+", ones) == n
        spec = ipmgen.Spec("int64", n, "random", seed=n)
        got = ipm.reduce("+", device_input(spec, offset=3))
        assert bits(got, "int64") == bits(oracle.reduce("+", ipmgen.fill_host(spec))[0], "int64")


def test_async_and_workspace_reuse(ipm):
    spec = ipmgen.Spec("float32", 3_000_001, "random", seed=9)
    x = device_input(spec)
    ws = torch.zeros(ipm.WS_BYTES, dtype=torch.uint8, device="cuda")
    outs = [ipm.reduce_async("+", x, init=np.float32(1.0), ws=ws) for _ in range(5)]
    vals = {bits(o.cpu().numpy()[0], "float32") for o in outs}
    assert len(vals) == 1
    _, want = oracle.reduce("+", ipmgen.fill_host(spec), init=np.float32(1.0))
    check("+", "float32", outs[0].cpu().numpy()[0], None, want)
    assert ws[:4096].view(torch.int32).abs().sum().item() == 0   # tickets left at zero


def test_cuda_graph_capture(ipm):
    spec = ipmgen.Spec("int32", 5_000_000, "random", seed=4)
    x = device_input(spec)
    s = torch.cuda.Stream()
    ws = torch.zeros(ipm.WS_BYTES, dtype=torch.uint8, device="cuda")
    out = torch.empty(1, dtype=torch.int32, device="cuda")
    with torch.cuda.stream(s):
        ipm.reduce_async("^", x, out=out, ws=ws, stream=s)  # warm
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        ipm.reduce_async("^", x, out=out, ws=ws, stream=s)
    want = oracle.reduce("^", ipmgen.fill_host(spec))[0]
    for _ in range(3):
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        assert out.item() == want


# --------------------------------------------------------------------------- segmented (nested) clause

SEG_SHAPES = [(0, 5), (1, 0), (7, 0), (1, 1), (7, 3), (1000, 1), (1000, 3), (1000, 31), (1000, 32), (1000, 33),
              (257, 4095), (257, 4096), (65, 4097), (3, 1 << 20), (1, (1 << 21) + 5), (40, 70_001),
              (700, 1025), (1200, 4099), (65536, 3), (65536, 33), (65536, 0),
              # more rows than one resident wave of warps: the CTA count is chosen to divide the rows evenly
              (9473, 40), (50000, 36)]


@pytest.fixture(params=["auto", "warp", "tma"])
def seg_kernel(request, ipm):
    ipm.set_option("seg_kernel", request.param)
    yield request.param
    ipm.set_option("seg_kernel", "auto")


@pytest.mark.parametrize("op,dt", LEGAL)
def test_segmented_parity(ipm, op, dt, seg_kernel):
    for k, (rows, cols) in enumerate(SEG_SHAPES):
        stride = cols + (k % 3) * 5  # row_stride >= cols, also non-multiples of the vector width
        total = max(0, (rows - 1) * stride + cols) if rows else 0
        spec = workload(op, dt, total, seed=k + 11)
        x = device_input(spec, offset=k % 4)
        init = NPT[dt](2)
        out = ipm.reduce_segmented(op, x, rows=rows, cols=cols, row_stride=stride, init=init).cpu().numpy()
        want_t, want_ld = oracle.reduce_segmented(op, ipmgen.fill_host(spec), rows, cols, stride, init=init)
        if dt.startswith("float") and op in ("+", "*"):
            err = np.abs(out.astype(np.longdouble) - want_ld)
            assert np.all((err <= TOL[dt] * np.abs(want_ld)) | (err == 0)), (op, dt, rows, cols)
        else:
            assert out.tobytes() == want_t.tobytes(), (op, dt, rows, cols)


def test_segmented_row_constant_closed_form(ipm, seg_kernel):
    rows, cols = 4096, 4096
    spec = ipmgen.Spec("float32", rows * cols, "const", param=0)
    x = device_input(spec)
    x.view(rows, cols).copy_((torch.arange(rows, device="cuda") % 1024).float()[:, None].expand(rows, cols))
    out = ipm.reduce_segmented("+", x.view(rows, cols)).cpu().numpy()
    assert np.array_equal(out, (cols * (np.arange(rows) % 1024)).astype(np.float32))


# --------------------------------------------------------------------------- data environment + host path

def test_data_clauses_and_host_path(ipm):
    h = ipmgen.fill_host(ipmgen.Spec("float64", 1_000_000, "random", seed=3))
    d = ipm.copyin(h)
    assert ipm.present(h) == d and ipm.present_count() == 1
    assert ipm.present(h[1000:2000]) == d + 8000          # sub-range lookup
    assert ipm.copyin(h) == d                              # present-or: ref++ only
    t = ipm.as_tensor(d, h.size, torch.float64)
    got = ipm.reduce("+", t)
    _, want = oracle.reduce("+", h)
    check("+", "float64", got, None, want)
    ipm.delete(h)
    ipm.copyout(h)
    assert ipm.present_count() == 0
    # fused copyin + reduce over a host array (pageable and pinned), chunked through staging buffers
    for pin in (False, True):
        src = torch.from_numpy(h).pin_memory() if pin else h
        got = ipm.reduce_host("+", src, init=np.float64(1.0))
        _, want = oracle.reduce("+", h, init=np.float64(1.0))
        check("+", "float64", got, None, want)
    big = ipmgen.fill_host(ipmgen.Spec("int32", 40_000_003, "random", seed=8))  # > one 64 MiB chunk
    assert ipm.reduce_host("^", big) == oracle.reduce("^", big)[0]


# --------------------------------------------------------------------------- multi-GPU code path at world 1

@pytest.mark.parametrize("mode", ["p2p", "nccl"])
def test_dist_world1(ipm, mode):
    import torch.distributed as dist
    ipm.set_option("dist_mode", mode)
    try:
        comm = ipm.Comm(0, 1, torch.cuda.current_device(), store=dist.HashStore())
        assert comm.fused == (mode == "p2p")
        for op, dt in [("+", "float32"), ("^", "int64"), ("max", "float64"), ("&&", "int32"), ("*", "float64"),
                       ("min", "int32")]:
            spec = workload(op, dt, 1_000_003, seed=2)
            x = device_input(spec)
            want_t, want_ld = oracle.reduce(op, ipmgen.fill_host(spec), init=NPT[dt](1))
            for _ in range(3):  # repeated calls: the fused path's epochs / parities
                check(op, dt, comm.reduce(op, x, init=NPT[dt](1)), want_t, want_ld)
            # back-to-back asynchronous calls, then one sync
            outs = [comm.reduce_async(op, x, init=NPT[dt](1)) for _ in range(5)]
            for o in outs:
                check(op, dt, o.cpu().numpy()[0], want_t, want_ld)
            # an empty shard contributes the identity
            check(op, dt, comm.reduce(op, x[:0], init=NPT[dt](1)), *oracle.reduce(op, x[:0].cpu().numpy(),
                                                                                 init=NPT[dt](1)))
            # end to end from a host shard (copyin fused with the reduction, then the exchange)
            check(op, dt, comm.reduce_host(op, ipmgen.fill_host(spec), init=NPT[dt](1)), want_t, want_ld)
        comm.close()
    finally:
        ipm.set_option("dist_mode", "auto")


def test_dist_fused_graph_capture(ipm):
    import torch.distributed as dist
    comm = ipm.Comm(0, 1, torch.cuda.current_device(), store=dist.HashStore())
    spec = ipmgen.Spec("float32", 3_000_017, "random", seed=5)
    x = device_input(spec)
    s = torch.cuda.Stream()
    ws = torch.zeros(ipm.WS_BYTES, dtype=torch.uint8, device="cuda")
    out = torch.empty(1, dtype=torch.float32, device="cuda")
    with torch.cuda.stream(s):
        comm.reduce_async("+", x, out=out, ws=ws, stream=s)
    torch.cuda.synchronize()
    g = torch.cuda.CUDAGraph()
    with torch.cuda.graph(g, stream=s):
        comm.reduce_async("+", x, out=out, ws=ws, stream=s)
    _, want = oracle.reduce("+", ipmgen.fill_host(spec))
    for _ in range(4):  # the device-side epoch advances on every replay
        out.zero_()
        g.replay()
        torch.cuda.synchronize()
        check("+", "float32", out.cpu().numpy()[0], None, want)
    comm.close()


# --------------------------------------------------------------------------- several variables, one pass

FSIGS = ["sum_sumsq", "dot", "minmax", "stats"]


@pytest.mark.parametrize("dt", DTS)
@pytest.mark.parametrize("sig", FSIGS)
def test_fused_parity(ipm, sig, dt):
    for i, n in enumerate([0, 1, 5, 33, 1000, 4097, 65_537, (1 << 20) + 3]):
        kind = "signed" if sig in ("minmax", "stats") else "random"
        sx = ipmgen.Spec(dt, n, kind, seed=i + 1)
        sy = ipmgen.Spec(dt, n, kind, seed=i + 101)
        for offx, offy in [(0, 0), (i % 8, i % 8), (1, 2)]:    # same and different alignment (DOT)
            x = device_input(sx, offx)
            y = device_input(sy, offy)
            nv = {"sum_sumsq": 2, "dot": 1, "minmax": 2, "stats": 4}[sig]
            init = np.arange(1, nv + 1).astype(NPT[dt])
            got = ipm.reduce_fused(sig, x, y if sig == "dot" else None, init=init)
            want_t, want_ld = oracle.reduce_fused(sig, ipmgen.fill_host(sx),
                                                  ipmgen.fill_host(sy) if sig == "dot" else None, init=init)
            ops = {"sum_sumsq": ["+", "+"], "dot": ["+"], "minmax": ["min", "max"],
                   "stats": ["+", "+", "min", "max"]}[sig]
            for v, op in enumerate(ops):
                check(op, dt, got[v], want_t[v], want_ld[v])


def test_fused_srad_statistics_closed_form(ipm):
    # SRAD-style image statistics: a_i = i mod 1024 -> Σ and Σ² in closed form, exact
    n = 1 << 24
    x = torch.arange(n, device="cuda", dtype=torch.int64).remainder(1024).to(torch.float32)
    s, s2, lo, hi = ipm.reduce_fused("stats", x)
    k = n // 1024
    assert s == k * 523776 and s2 == k * sum(i * i for i in range(1024)) and lo == 0 and hi == 1023


# --------------------------------------------------------------------------- strided 2-D region -> one scalar

@pytest.mark.parametrize("op,dt", LEGAL)
def test_2d_collapse_parity(ipm, op, dt):
    shapes = [(0, 5, 5), (3, 0, 4), (1, 1, 1), (7, 3, 5), (100, 33, 40), (5, 5000, 5003), (3, 300_001, 300_010),
              (2000, 257, 300), (64, 4096, 4096), (4096, 1, 3)]
    for k, (rows, cols, stride) in enumerate(shapes):
        total = max(0, (rows - 1) * stride + cols) if rows else 0
        spec = workload(op, dt, total, seed=k + 3)
        x = device_input(spec, offset=k % 8)
        init = NPT[dt](2)
        got = ipm.reduce_2d(op, x, rows=rows, cols=cols, row_stride=stride, init=init)
        h = ipmgen.fill_host(spec)
        region = np.concatenate([h[r * stride:r * stride + cols] for r in range(rows)]) if rows and cols else h[:0]
        want_t, want_ld = oracle.reduce(op, region, init=init)   # the plain fold over the region, row-major
        check(op, dt, got, want_t, want_ld)


def test_2d_view_api(ipm):
    big = torch.arange(1000 * 700, dtype=torch.int64, device="cuda").view(1000, 700)
    sub = big[10:900, 33:650]
    assert ipm.reduce_2d("+", sub) == int(sub.sum())
    assert ipm.reduce_2d("max", sub) == int(sub.max())
    assert ipm.reduce("^", sub) == int(np.bitwise_xor.reduce(sub.cpu().numpy().ravel()))   # reduce() dispatches


# --------------------------------------------------------------------------- ragged (CSR) rows

def ragged_cases():
    yield "tiny", np.array([0, 1, 1, 3], np.int64)
    yield "all_empty", np.array([4] * 6, np.int64)
    yield "one_row", np.array([0, 1000], np.int64)
    yield "const", ipmgen.offsets_from_degrees(ipmgen.degrees(2000, kind="const", mean=33))
    yield "uniform_off3", ipmgen.offsets_from_degrees(ipmgen.degrees(5000, kind="uniform", mean=20, seed=2), 3)
    yield "powerlaw", ipmgen.offsets_from_degrees(ipmgen.degrees(20_000, seed=3))
    d = np.zeros(300, np.int64); d[[0, 150, 299]] = [100_000, 1_000_000, 7]
    yield "huge_rows", ipmgen.offsets_from_degrees(d)
    # > 512 elements per warp at 148 x 32 warps: whole chunks in which no row starts (the flag-free path),
    # long rows next to runs of short and empty ones, empty rows after the last element
    d = ipmgen.degrees(1500, kind="const", mean=4096)
    d[100:400] = np.arange(300) % 5
    d[-3:] = 0
    yield "long_rows", ipmgen.offsets_from_degrees(d, 1)
    # thousands of empty rows inside one tile (the per-tile row window repeats), rows of one element, a row
    # spanning many CTAs, rows ending exactly where others start
    d = np.ones(200_000, np.int64)
    d[5000:15000] = 0
    d[50_000] = 3_000_000
    d[60_000:60_100] = 4096
    d[-5000:] = 0
    yield "empties_and_giant", ipmgen.offsets_from_degrees(d, 7)


@pytest.fixture(params=["auto", "tile", "warp", "rank", "lpr", "marked"])
def ragged_kernel(request, ipm):
    ipm.set_option("ragged_kernel", request.param)
    yield request.param
    ipm.set_option("ragged_kernel", "auto")


@pytest.mark.parametrize("op,dt", LEGAL)
def test_ragged_parity(ipm, op, dt, ragged_kernel):
    for k, (name, off) in enumerate(ragged_cases()):
        n = int(off[-1]) + 5
        spec = workload(op, dt, n, seed=k + 21)
        x = device_input(spec, offset=k % 4)
        offs = torch.from_numpy(off).cuda()
        init = NPT[dt](2)
        got = ipm.reduce_ragged(op, x, offs, init=init).cpu().numpy()
        want_t, want_ld = oracle.reduce_ragged(op, ipmgen.fill_host(spec), off, init=init)
        if dt.startswith("float") and op in ("+", "*"):
            err = np.abs(got.astype(np.longdouble) - want_ld)
            assert np.all((err <= TOL[dt] * np.abs(want_ld)) | (err == 0)), (op, dt, name)
        else:
            assert got.tobytes() == want_t.tobytes(), (op, dt, name)


def test_ragged_big_powerlaw_deterministic(ipm, ragged_kernel):
    off = ipmgen.offsets_from_degrees(ipmgen.degrees(1 << 20, seed=7))
    spec = ipmgen.Spec("float32", int(off[-1]), "random", seed=7)
    x = device_input(spec)
    offs = torch.from_numpy(off).cuda()
    a = ipm.reduce_ragged("+", x, offs).cpu().numpy()
    b = ipm.reduce_ragged("+", x, offs).cpu().numpy()
    assert a.tobytes() == b.tobytes()
    _, want = oracle.reduce_ragged("+", ipmgen.fill_host(spec), off)
    # dyadic data: row sums are exact in fp64 -> correctly rounded per row
    assert np.array_equal(a, want.astype(np.float32))


def test_ragged_marked_side_stream(ipm):
    """The two-pass path on a caller stream other than torch's current one: its scratch (from torch's caching
    allocator, allocated on the current stream) must not be handed out again while the kernels still use it —
    allocations and writes on the current stream right after each call, result checked against the oracle."""
    off = ipmgen.offsets_from_degrees(ipmgen.degrees(1 << 18, seed=11))
    spec = ipmgen.Spec("int32", int(off[-1]), "random", seed=11)
    x = device_input(spec)
    offs = torch.from_numpy(off).cuda()
    want, _ = oracle.reduce_ragged("^", ipmgen.fill_host(spec), off)
    side = torch.cuda.Stream()
    side.wait_stream(torch.cuda.current_stream())
    ipm.set_option("ragged_kernel", "marked")
    try:
        outs = []
        for _ in range(4):
            o = torch.empty(off.size - 1, dtype=torch.int32, device="cuda")
            o.record_stream(side)
            outs.append(ipm.reduce_ragged("^", x, offs, out=o, stream=side))
            junk = torch.empty(ipm.lib.ipm_ragged_scratch_bytes(0, x.numel(), off.size - 1), dtype=torch.uint8,
                               device="cuda")
            junk.fill_(0xFF)  # on the current stream, while the side stream may still be running
        side.synchronize()
    finally:
        ipm.set_option("ragged_kernel", "auto")
    for o in outs:
        assert o.cpu().numpy().tobytes() == want.tobytes()


def test_ragged_marked_offsets_beyond_nvalues_stay_in_scratch(ipm):
    """Outside the contract (off[rows] > nvalues, the bound the scratch is sized from) the results are undefined,
    but the two-pass kernels must not write past the scratch: canary bytes after it stay intact."""
    L = ipm.lib
    nvalues = 1000
    x = torch.ones(1 << 20, dtype=torch.float32, device="cuda")  # the kernels may read past nvalues, not past x
    off = torch.tensor([0, 10, 500_000, 900_000], dtype=torch.int64, device="cuda")
    need = L.ipm_ragged_scratch_bytes(2, nvalues, 3)
    scratch = torch.full((need + 4096,), 0xAB, dtype=torch.uint8, device="cuda")
    out = torch.zeros(3, dtype=torch.float32, device="cuda")
    ws = ipm.workspace()
    rc = L.ipm_reduce_ragged_marked(0, 2, x.data_ptr(), nvalues, off.data_ptr(), 3, None, out.data_ptr(),
                                    ws.data_ptr(), scratch.data_ptr(), need, ipm._stream())
    torch.cuda.synchronize()
    assert rc == 0
    assert bool((scratch[need:] == 0xAB).all())


def test_nondeterministic_mode_parity(ipm):
    ipm.set_option("deterministic", 0)
    try:
        for dt in ("float32", "float64"):
            for n in [1, 1000, 4_000_037]:
                spec = workload("+", dt, n, seed=n)
                x = device_input(spec)
                want_t, want_ld = oracle.reduce("+", ipmgen.fill_host(spec))
                check("+", dt, ipm.reduce("+", x), want_t, want_ld)
    finally:
        ipm.set_option("deterministic", 1)


@pytest.mark.parametrize("world", [2, 3, 8])
def test_dist_fused_multirank_one_gpu(ipm, world):
    """world ranks in one process on one GPU (ipm_comm_init_group): each rank's kernel runs on its own stream and
    exchanges its partial through the other ranks' slot buffers — the fused multi-GPU code path with world > 1."""
    comms = ipm.Comm.group(world)
    streams = [torch.cuda.Stream() for _ in range(world)]
    wss = [torch.zeros(ipm.WS_BYTES, dtype=torch.uint8, device="cuda") for _ in range(world)]
    for op, dt, n in [("+", "float32", 10_000_019), ("^", "int64", 1_000_003), ("max", "float64", 777),
                      ("&&", "int32", 5), ("min", "int32", 0)]:
        spec = workload(op, dt, n, seed=world)
        x = device_input(spec)
        torch.cuda.synchronize()
        h = ipmgen.fill_host(spec)
        for rep in range(3):  # repeated, back-to-back asynchronous calls per rank (epochs / parities)
            init = NPT[dt](rep + 1)  # a different init per call: a stale slot would give a wrong result
            want_t, want_ld = oracle.reduce(op, h, init=init)
            outs = []
            t0 = time.perf_counter()
            for r, c in enumerate(comms):
                lo, hi = ipm.shard_range(n, r, world)
                with torch.cuda.stream(streams[r]):
                    o = torch.empty(1, dtype=TD[dt], device="cuda")
                    outs.append(c.reduce_async(op, x[lo:hi], init=init, out=o, ws=wss[r], stream=streams[r]))
            torch.cuda.synchronize()
            assert time.perf_counter() - t0 < 2.0                    # no rank waited for a timeout
            for c in comms:
                e = ctypes.c_int(0)
                ipm.lib.ipm_comm_error(c._h, ctypes.byref(e))
                assert e.value == 0
            vals = [o.cpu().numpy()[0] for o in outs]
            assert len({bits(v, dt) for v in vals}) == 1, vals      # every rank gets the same bits
            check(op, dt, vals[0], want_t, want_ld)
    for c in comms:
        c.close()


@pytest.mark.parametrize("world", [2, 3])
def test_dist_ipc_processes_one_gpu(ipm, world, tmp_path):
    """world PROCESSES on one GPU bootstrapped without NCCL (ipm_comm_create_ipc / ipm_comm_attach_ipc: the slot
    buffers' CUDA IPC handles travel through a FileStore): the cross-process peer mapping + fused exchange, device
    and host shards, every rank's bits equal and equal to the oracle's answer."""
    import json
    import subprocess
    import sys

    import ipc_worker
    store = str(tmp_path / "store")
    worker = os.path.join(os.path.dirname(os.path.abspath(__file__)), "ipc_worker.py")
    procs = [subprocess.Popen([sys.executable, worker, str(r), str(world), store], stdout=subprocess.PIPE,
                              stderr=subprocess.PIPE, text=True) for r in range(world)]
    outs = []
    for p in procs:
        out, err = p.communicate(timeout=300)
        assert p.returncode == 0, err[-2000:]
        outs.append([json.loads(l) for l in out.splitlines() if l.startswith("{")])
    per_case = len(ipc_worker.CASES) * (len(ipc_worker.INITS) + 1)
    assert all(len(o) == per_case for o in outs)
    for i in range(per_case):
        rows = [o[i] for o in outs]
        assert len({r["bits"] for r in rows}) == 1, rows         # every rank the same bits
        r0 = rows[0]
        case = next(c for c in ipc_worker.CASES if c[0] == r0["op"] and c[1] == r0["dt"])
        op, dt, kind, n = case
        h = ipmgen.fill_host(ipmgen.Spec(dt, n, kind, seed=ipc_worker.SEED))
        want_t, want_ld = oracle.reduce(op, h, init=NPT[dt](r0["init"]))
        got = np.frombuffer(bytes.fromhex(r0["bits"]), dtype=dt)[0]
        check(op, dt, got, want_t, want_ld)


# --------------------------------------------------------------------------- options, data clauses, host path edges

@pytest.mark.parametrize("cps", [1, 2, 8])
@pytest.mark.parametrize("det", [0, 1, 2])
def test_flat_options_keep_results(ipm, cps, det):
    ipm.set_option("flat_ctas_per_sm", cps)
    ipm.set_option("deterministic", det)
    try:
        for op, dt, n in [("+", "float64", 5_000_011), ("^", "int32", 3_000_001), ("max", "float32", 777_777)]:
            spec = workload(op, dt, n, seed=cps * 10 + det)
            want_t, want_ld = oracle.reduce(op, ipmgen.fill_host(spec), init=NPT[dt](2))
            check(op, dt, ipm.reduce(op, device_input(spec, offset=1), init=NPT[dt](2)), want_t, want_ld)
    finally:
        ipm.set_option("flat_ctas_per_sm", -1)
        ipm.set_option("deterministic", 1)


def test_update_clauses_and_host_edges(ipm):
    h = np.arange(10_000, dtype=np.int64)
    d = ipm.copyin(h)
    t = ipm.as_tensor(d, h.size, torch.int64)
    assert ipm.reduce("+", t) == h.sum()
    h[:] = 2                                   # acc update device(h)
    ipm.update_device(h)
    assert ipm.reduce("+", t) == 20_000
    t.fill_(3)                                 # acc update host(h)
    torch.cuda.synchronize()
    ipm.update_host(h)
    assert np.all(h == 3)
    ipm.copyout(h)
    assert ipm.present_count() == 0
    # the fused host path: empty, one element, a size that is not a multiple of the 64 MiB staging chunk
    assert ipm.reduce_host("+", np.zeros(0, np.float32), init=np.float32(1.5)) == np.float32(1.5)
    assert ipm.reduce_host("max", np.array([7], np.int32)) == 7
    big = ipmgen.fill_host(ipmgen.Spec("float32", (1 << 24) * 3 + 17, "random", seed=4))
    _, want = oracle.reduce("+", big)
    check("+", "float32", ipm.reduce_host("+", torch.from_numpy(big).pin_memory()), None, want)
    ipm.lib.ipm_release_staging()
