"""C1 (2^20 int32, 4 MiB) latency: static vs guided schedule, L2 flushed before each launch."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ipmgen
from paper_1412_1127_b200 import ipm
n = 1 << 20
x = torch.empty(n, dtype=torch.int32, device="cuda")
ipmgen.fill_tensor(ipmgen.Spec("int32", n, "iota", param=1), x)
scratch = torch.empty(1 << 27, dtype=torch.float32, device="cuda")
r = torch.empty(1, dtype=torch.int32, device="cuda")
for mode, v in [("guided", 1), ("static", 2), ("dynamic", 0)]:
    ipm.set_option("deterministic", v)
    for flush in (True, False):
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 0.2:
            ipm.reduce_async("+", x, out=r)
        torch.cuda.synchronize()
        ms = []
        for _ in range(50):
            if flush:
                scratch.fill_(1.0)
            with ipm.KernelTimer(2) as kt:
                ipm.reduce_async("+", x, out=r)
                torch.cuda.synchronize()
            ms += kt.ms
        print(f"{mode:8s} flush={flush}: median {statistics.median(ms)*1e3:.2f} us  min {min(ms)*1e3:.2f} us  result {r.item()}")
