"""Probe: int64 `&&` runs 2-20 % slower than `& | ^ ||` in the bench suite (profiles/r01_bench_*.json). Is it
the op (unsigned 64-bit min) or the data (random nonzero words)? Times each op on each data kind, twice."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ipmgen  # noqa: E402
from paper_1412_1127_b200 import ipm  # noqa: E402


def t(op, x, reps=10):
    r = torch.empty(1, dtype=x.dtype, device="cuda")
    for _ in range(5):
        ipm.reduce_async(op, x, out=r)
    torch.cuda.synchronize()
    with ipm.KernelTimer(reps) as kt:
        for _ in range(reps):
            ipm.reduce_async(op, x, out=r)
        torch.cuda.synchronize()
    ms = sorted(kt.ms)
    med = statistics.median(ms)
    return f"med {med:.4f} ms min {ms[0]:.4f} max {ms[-1]:.4f} {x.numel() * x.element_size() / med / 1e6:7.1f} GB/s"


n = 1 << 30
for dt, tdt in (("int64", torch.int64), ("int32", torch.int32)):
    x = torch.empty(n, dtype=tdt, device="cuda")
    for kind in ["nonzero", "random", "allbits"]:
        ipmgen.fill_tensor(ipmgen.Spec(dt, n, kind, seed=1), x)
        for rep in range(2):
            for op in ["^", "&&", "||", "min", "max", "&"]:
                print(dt, kind, rep, f"{op:3s}", t(op, x), flush=True)
    del x
    torch.cuda.empty_cache()
