"""Device time of ipm_reduce_ragged on the DESIGN.md ragged recipes (CUDA events on the launch stream)."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import ipmgen
from paper_1412_1127_b200 import ipm

CASES = [("powerlaw", 1 << 24, 16.0), ("const", 1 << 22, 64.0), ("uniform", 1 << 24, 16.0),
         ("const", 1 << 16, 4096.0), ("const", 1 << 25, 4.0)]
OPS = [("+", "float32"), ("max", "float32"), ("+", "float64"), ("^", "int32"), ("max", "float64")]
KERNELS = os.environ.get("KERNELS", "warp,tile,rank").split(",")
if os.environ.get("CASES"):  # e.g. CASES="const:262144:1024,powerlaw:16777216:16"
    CASES = [(c.split(":")[0], int(c.split(":")[1]), float(c.split(":")[2])) for c in os.environ["CASES"].split(",")]
if len(sys.argv) > 1 and sys.argv[1] == "quick":
    OPS = OPS[:1]
if os.environ.get("OPS"):  # e.g. OPS="+:float32,^:int32"
    OPS = [tuple(o.split(":")) for o in os.environ["OPS"].split(",")]
for kind, rows, mean in CASES:
    off = ipmgen.offsets_from_degrees(ipmgen.degrees(rows, seed=1, kind=kind, mean=mean))
    nnz = int(off[-1])
    offs = torch.from_numpy(off).cuda()
    for op, dt in OPS:
        tdt = getattr(torch, dt)
        vals = torch.empty(nnz, dtype=tdt, device="cuda")
        ipmgen.fill_tensor(ipmgen.Spec(dt, nnz, "random", seed=1), vals)
        o = torch.empty(rows, dtype=tdt, device="cuda")
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 0.2:
            ipm.reduce_ragged(op, vals, offs, out=o)
            torch.cuda.synchronize()
        for kern in KERNELS:
            ipm.set_option("ragged_kernel", kern)
            ipm.reduce_ragged(op, vals, offs, out=o)
            torch.cuda.synchronize()
            with ipm.KernelTimer(20) as kt:
                for _ in range(20):
                    ipm.reduce_ragged(op, vals, offs, out=o)
                torch.cuda.synchronize()
            med = statistics.median(kt.ms)
            w = vals.element_size()
            nbytes = nnz * w + off.size * 8 + rows * w
            print(f"{kern:5s} {kind:8s} rows={rows:9d} mean={mean:6.0f} {op:3s} {dt:7s} nnz={nnz} "
                  f"max={int(np.diff(off).max())}: {med:.3f} ms {nbytes/med/1e6:7.1f} GB/s", flush=True)
        ipm.set_option("ragged_kernel", "auto")
        del vals, o
