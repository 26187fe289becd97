"""A/B of the flat kernel's tile schedules on ONE box, interleaved rounds (box-to-box HBM speed varies ~3%):
guided (default, deterministic), dynamic, static — C5 (2^34 float32) and C2 sizes."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ipmgen
from paper_1412_1127_b200 import ipm

MODES = {"guided": 1, "dynamic": 0, "static": 2}
for n, dt, tdt in [(1 << 34, "float32", torch.float32), (1 << 28, "float32", torch.float32),
                   (1 << 30, "int32", torch.int32)]:
    x = torch.empty(n, dtype=tdt, device="cuda")
    ipmgen.fill_tensor(ipmgen.Spec(dt, n, "random", seed=1), x)
    r = torch.empty(1, dtype=tdt, device="cuda")
    op = "+" if dt == "float32" else "^"
    res = {m: [] for m in MODES}
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.3:
        ipm.reduce_async(op, x, out=r)
        torch.cuda.synchronize()
    reps = 10 if n >= (1 << 34) else 40
    for rnd in range(4):
        for m, v in MODES.items():
            ipm.set_option("deterministic", v)
            for _ in range(2):
                ipm.reduce_async(op, x, out=r)
            with ipm.KernelTimer(reps) as kt:
                for _ in range(reps):
                    ipm.reduce_async(op, x, out=r)
                torch.cuda.synchronize()
            res[m] += kt.ms
    ipm.set_option("deterministic", 1)
    nb = n * x.element_size()
    print(f"n=2^{n.bit_length()-1} {dt} {op}: " + "  ".join(
        f"{m} {nb / statistics.median(v) / 1e6:7.1f} GB/s (min-time {nb / min(v) / 1e6:7.1f})" for m, v in res.items()),
        flush=True)
    del x
    torch.cuda.empty_cache()
