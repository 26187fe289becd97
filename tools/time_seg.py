"""Segmented rows: one CTA per row vs one warp per row vs TMA ring, interleaved on one box."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ipmgen
from paper_1412_1127_b200 import ipm
for rows, cols in [(65536, 4096), (16384, 16384), (262144, 1024), (4096, 65536)]:
    x = torch.empty(rows * cols, dtype=torch.float32, device="cuda")
    ipmgen.fill_tensor(ipmgen.Spec("float32", rows * cols, "random", seed=1), x)
    o = torch.empty(rows, dtype=torch.float32, device="cuda")
    res = {}
    for rnd in range(3):
        for k in ("auto", "warp", "tma"):
            ipm.set_option("seg_kernel", k)
            t0 = time.perf_counter()
            while time.perf_counter() - t0 < 0.1:
                ipm.reduce_segmented("+", x.view(rows, cols), out=o)
            torch.cuda.synchronize()
            with ipm.KernelTimer(20) as kt:
                for _ in range(20):
                    ipm.reduce_segmented("+", x.view(rows, cols), out=o)
                torch.cuda.synchronize()
            res.setdefault(k, []).extend(kt.ms)
    ipm.set_option("seg_kernel", "auto")
    nb = rows * cols * 4 + rows * 4
    print(f"{rows}x{cols}: " + "  ".join(f"{k} {nb / statistics.median(v) / 1e6:7.1f} GB/s" for k, v in res.items()),
          flush=True)
    del x
