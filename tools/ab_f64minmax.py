"""Same-box A/B: the flat clause on 2^28 float64 for + max min && and 2^30 int64 for & && max (device time per
launch, library events, interleaved rounds); IPM_LIB selects the library build (tools/ab_lib.py pattern)."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ipmgen
from paper_1412_1127_b200 import ipm

CASES = [("float64", 1 << 28, op, kind) for op, kind in (("+", "random"), ("max", "signed"), ("min", "signed"),
                                                          ("&&", "nonzero"))] + \
        [("int64", 1 << 30, op, kind) for op, kind in (("&", "allbits"), ("&&", "nonzero"), ("max", "random"))]
res = {}
bufs = {}
for dt, n, op, kind in CASES:
    key = (dt, n, kind)
    if key not in bufs:
        x = torch.empty(n, dtype=getattr(torch, dt), device="cuda")
        ipmgen.fill_tensor(ipmgen.Spec(dt, n, kind, seed=1), x)
        bufs[key] = x
r = torch.empty(1, dtype=torch.float64, device="cuda")
t0 = time.perf_counter()
while time.perf_counter() - t0 < 0.3:
    ipm.reduce_async("+", bufs[("float64", 1 << 28, "random")])
    torch.cuda.synchronize()
for rnd in range(5):
    for dt, n, op, kind in CASES:
        x = bufs[(dt, n, kind)]
        with ipm.KernelTimer(20) as kt:
            for _ in range(20):
                ipm.reduce_async(op, x)
            torch.cuda.synchronize()
        res.setdefault((dt, op), []).extend(kt.ms)
for (dt, op), v in res.items():
    n = 1 << 28 if dt == "float64" else 1 << 30
    print(f"{dt:8s} {op:3s} {n * 8 / statistics.median(v) / 1e6:7.1f} GB/s  median {statistics.median(v)*1e3:8.1f} us")
