"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ipmgen  # noqa: E402
from paper_1412_1127_b200 import ipm  # noqa: E402

TD = {"int32": torch.int32, "int64": torch.int64, "float32": torch.float32, "float64": torch.float64}
for dt in TD:
    for n in [0, 1, 7, 33, 1000, 70_001, 300_007]:
        for off in (0, 3):
            buf = torch.empty(n + off + 1, dtype=TD[dt], device="cuda")
            x = buf[off:off + n]
            if n:
                ipmgen.fill_device(ipmgen.Spec(dt, n, "random", seed=n), x.data_ptr(), 0, n,
                                   torch.cuda.current_stream().cuda_stream)
            for op in ["+", "max", "&&"] + (["^"] if dt.startswith("int") else []):
                ipm.reduce(op, x, init=np.array(1, dtype=x.cpu().numpy().dtype)[()])
    for kern in ("ldg", "tma"):
        ipm.set_option("seg_kernel", kern)
        for rows, cols, stride in [(5, 3, 4), (33, 100, 103), (9, 4097, 4100), (2, 40_000, 40_001), (300, 64, 64),
                                  (6000, 40, 40)]:  # more rows than one resident wave of warps
            x = torch.empty((rows - 1) * stride + cols + 3, dtype=TD[dt], device="cuda")
            ipmgen.fill_device(ipmgen.Spec(dt, x.numel(), "random", seed=1), x.data_ptr(), 0, x.numel(),
                               torch.cuda.current_stream().cuda_stream)
            ipm.reduce_segmented("+", x[1:], rows=rows, cols=cols, row_stride=stride)
    ipm.set_option("seg_kernel", "auto")
h = np.arange(100_000, dtype=np.int64)
ipm.reduce_host("+", h)
torch.cuda.synchronize()
print("sanitize_run: ok")
# ragged rows (all three kernels), several variables, 2-D region, the fused multi-rank exchange (2 ranks, one GPU)


def ragged_all(op, x, off):
    for kern in ("auto", "warp", "tile", "rank", "lpr", "marked"):
        ipm.set_option("ragged_kernel", kern)
        ipm.reduce_ragged(op, x, off)
    ipm.set_option("ragged_kernel", "auto")


for dt in TD:
    off = np.array([0, 3, 3, 40, 41, 300, 300, 5000], np.int64) + 2
    x = torch.empty(int(off[-1]) + 3, dtype=TD[dt], device="cuda")
    ipmgen.fill_device(ipmgen.Spec(dt, x.numel(), "random", seed=2), x.data_ptr(), 0, x.numel(),
                       torch.cuda.current_stream().cuda_stream)
    ragged_all("+", x, torch.from_numpy(off).cuda())
    for sig in ("sum_sumsq", "dot", "minmax", "stats"):
        ipm.reduce_fused(sig, x[1:2001], x[3:2003] if sig == "dot" else None)
    ipm.reduce_2d("max", x, rows=7, cols=300, row_stride=700)
    # a power-law graph: short rows packed several per lane (shared-memory parked segments), rows split across
    # warps (head/tail records + fix-up), empty rows
    off2 = ipmgen.offsets_from_degrees(ipmgen.degrees(1 << 14, seed=4, mean=6.0))
    z = torch.empty(int(off2[-1]) + 1, dtype=TD[dt], device="cuda")
    ipmgen.fill_device(ipmgen.Spec(dt, z.numel(), "random", seed=4), z.data_ptr(), 0, z.numel(),
                       torch.cuda.current_stream().cuda_stream)
    ragged_all("max", z[1:], torch.from_numpy(off2).cuda())
    # > 512 elements per warp: whole chunks in which no row starts (the flag-free path), rows across many warps
    off3 = np.array([0, 1_500_000, 1_500_003, 3_000_000, 3_000_000, 3_000_017, 4_600_000], np.int64) + 1
    z = torch.empty(int(off3[-1]) + 2, dtype=TD[dt], device="cuda")
    ipmgen.fill_device(ipmgen.Spec(dt, z.numel(), "random", seed=6), z.data_ptr(), 0, z.numel(),
                       torch.cuda.current_stream().cuda_stream)
    ragged_all("+", z, torch.from_numpy(off3).cuda())
    # thousands of empty rows inside one chunk (jumps in the offset ring), more than 64 rows per chunk
    d4 = np.ones(20_000, np.int64)
    d4[100:6000] = 0
    d4[7000] = 50_000
    off4 = ipmgen.offsets_from_degrees(d4)
    z = torch.empty(int(off4[-1]) + 1, dtype=TD[dt], device="cuda")
    ragged_all("+", z, torch.from_numpy(off4).cuda())
    for rows, cols, stride in [(33, 1000, 1024), (5, 4099, 4101), (200, 31, 37)]:
        w = torch.empty(rows * stride + 1, dtype=TD[dt], device="cuda")
        ipmgen.fill_device(ipmgen.Spec(dt, w.numel(), "random", seed=5), w.data_ptr(), 0, w.numel(),
                           torch.cuda.current_stream().cuda_stream)
        ipm.reduce_2d("+", w[1:], rows=rows, cols=cols, row_stride=stride)
ipm.set_option("dist_timeout_ms", 3000)  # the sanitizer may serialise the two ranks' kernels
comms = ipm.Comm.group(2)
y = torch.arange(100_003, dtype=torch.float64, device="cuda")
ss = [torch.cuda.Stream() for _ in range(2)]
wss = [torch.zeros(ipm.WS_BYTES, dtype=torch.uint8, device="cuda") for _ in range(2)]
for r, c in enumerate(comms):
    lo, hi = ipm.shard_range(y.numel(), r, 2)
    c.reduce_async("+", y[lo:hi], ws=wss[r], stream=ss[r])
torch.cuda.synchronize()
for c in comms:
    c.close()
print("sanitize_run (extended): ok")
for dt in TD:  # one CTA per row (long rows, many of them)
    x = torch.empty(600 * 1100 + 5, dtype=TD[dt], device="cuda")
    ipmgen.fill_device(ipmgen.Spec(dt, x.numel(), "random", seed=3), x.data_ptr(), 0, x.numel(),
                       torch.cuda.current_stream().cuda_stream)
    ipm.reduce_segmented("+", x[1:], rows=600, cols=1100, row_stride=1100)
torch.cuda.synchronize()
print("sanitize_run (seg cta): ok")
# the production flat schedule above 64 MiB: k_flat_guided (static tiles, dynamic chunks, remainder chunk), and
# the dynamic / static k_flat selected by IPM_OPT_DETERMINISTIC, on misaligned inputs
for dt, n in (("int32", 20_000_005), ("float32", 17_000_003), ("int64", 9_000_007), ("float64", 8_500_001)):
    buf = torch.empty(n + 4, dtype=TD[dt], device="cuda")
    x = buf[3:3 + n]
    ipmgen.fill_device(ipmgen.Spec(dt, n, "random", seed=9), x.data_ptr(), 0, n, torch.cuda.current_stream().cuda_stream)
    for det in (1, 0, 2):
        ipm.set_option("deterministic", det)
        assert ipm.flat_schedule(x.dtype, n) == {1: "guided", 0: "dynamic", 2: "static"}[det]
        for op in ["+", "max"] + (["^"] if dt.startswith("int") else ["&&"]):
            ipm.reduce(op, x, init=np.array(1, dtype=x.cpu()[:1].numpy().dtype)[()])
    ipm.set_option("deterministic", 1)
    del buf, x
torch.cuda.synchronize()
print("sanitize_run (guided > 64 MiB): ok")
