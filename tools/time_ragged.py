import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, torch
import ipmgen
from paper_1412_1127_b200 import ipm
for kind, rows, mean in [("powerlaw", 1 << 24, 16.0), ("const", 1 << 22, 64.0), ("uniform", 1 << 24, 16.0),
                         ("const", 1 << 16, 4096.0)]:
    off = ipmgen.offsets_from_degrees(ipmgen.degrees(rows, seed=1, kind=kind, mean=mean))
    nnz = int(off[-1])
    vals = torch.empty(nnz, dtype=torch.float32, device="cuda")
    ipmgen.fill_tensor(ipmgen.Spec("float32", nnz, "random", seed=1), vals)
    offs = torch.from_numpy(off).cuda()
    o = torch.empty(rows, dtype=torch.float32, device="cuda")
    t0 = time.perf_counter()
    while time.perf_counter() - t0 < 0.2:
        ipm.reduce_ragged("+", vals, offs, out=o)
        torch.cuda.synchronize()
    with ipm.KernelTimer(20) as kt:
        for _ in range(20):
            ipm.reduce_ragged("+", vals, offs, out=o)
        torch.cuda.synchronize()
    med = statistics.median(kt.ms)
    nbytes = nnz * 4 + off.size * 8 + rows * 4
    print(f"{kind} rows={rows} mean={mean} nnz={nnz} max={int(np.diff(off).max())}: {med:.3f} ms {nbytes/med/1e6:.1f} GB/s",
          flush=True)
