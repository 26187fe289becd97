"""Probe: why do 4-byte-element reductions over 4 GiB run slower in the bench suite than in the sweep?
Times the library's flat kernel on int32 / int64 / float32 with different data and allocation orders."""
import os
import statistics
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch  # noqa: E402

import ipmgen  # noqa: E402
from paper_1412_1127_b200 import ipm  # noqa: E402


def t(op, x, reps=10):
    r = torch.empty(1, dtype=x.dtype, device="cuda")
    for _ in range(3):
        ipm.reduce_async(op, x, out=r)
    torch.cuda.synchronize()
    with ipm.KernelTimer(reps) as kt:
        for _ in range(reps):
            ipm.reduce_async(op, x, out=r)
        torch.cuda.synchronize()
    med = statistics.median(kt.ms)
    return f"{med:.4f} ms {x.numel() * x.element_size() / med / 1e6:7.1f} GB/s"


for dt, tdt, n in [("int32", torch.int32, 1 << 30), ("int64", torch.int64, 1 << 29), ("int32", torch.int32, 1 << 31),
                   ("float32", torch.float32, 1 << 30)]:
    x = torch.empty(n, dtype=tdt, device="cuda")
    for kind in ["random", "const", "allbits"]:
        ipmgen.fill_tensor(ipmgen.Spec(dt, n, kind, seed=1, param=0), x)
        for op in (["^", "|", "+"] if dt.startswith("int") else ["+", "max"]):
            print(dt, n, kind, op, t(op, x), flush=True)
    x.fill_(1)
    print(dt, n, "fill_1", "^" if dt.startswith("int") else "+", t("^" if dt.startswith("int") else "+", x))
    for cps in (1, 2, 4, 8):
        ipm.set_option("flat_ctas_per_sm", cps)
        print(dt, n, "cps", cps, t("^" if dt.startswith("int") else "+", x))
    ipm.set_option("flat_ctas_per_sm", -1)
    del x
    torch.cuda.empty_cache()
