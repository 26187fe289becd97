"""Kernel-time floor: the flat clause at n = 1, 2^12, 2^16, 2^20 (int32), events around each launch."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ipmgen
from paper_1412_1127_b200 import ipm
for det in (1, 2):
    ipm.set_option("deterministic", det)
    for lg in (0, 12, 16, 20, 22):
        n = 1 << lg
        x = torch.ones(n, dtype=torch.int32, device="cuda")
        r = torch.empty(1, dtype=torch.int32, device="cuda")
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 0.1:
            ipm.reduce_async("+", x, out=r)
        torch.cuda.synchronize()
        with ipm.KernelTimer(50) as kt:
            for _ in range(50):
                ipm.reduce_async("+", x, out=r)
            torch.cuda.synchronize()
        print(f"det={det} n=2^{lg}: median {statistics.median(kt.ms)*1e3:.2f} us grid={ipm.flat_geometry(torch.int32, n)[0]}",
              flush=True)
