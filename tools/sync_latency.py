"""Host latency of the synchronous clause call (ipm.reduce: launch, kernel, result into the caller's variable) on
BASELINE config 1 (2^20 int32 +) and on 2^24 float32 +, back to back, L2-warm. Run under IPM_LIB=... for an A/B."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
from paper_1412_1127_b200 import ipm

for n, dt in ((1 << 20, torch.int32), (1 << 24, torch.float32)):
    x = torch.ones(n, dtype=dt, device="cuda")
    for _ in range(2000):
        ipm.reduce("+", x)
    reps = []
    for _ in range(7):
        t0 = time.perf_counter()
        for _ in range(500):
            v = ipm.reduce("+", x)
        reps.append((time.perf_counter() - t0) / 500 * 1e6)
    print(f"{os.path.basename(os.environ.get('IPM_LIB', 'libipm.so'))} n={n} {dt}: median {statistics.median(reps):.2f} us "
          f"min {min(reps):.2f} us result {v}", flush=True)
