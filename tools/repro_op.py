import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ipmgen
from paper_1412_1127_b200 import ipm
op, dt, n = sys.argv[1], sys.argv[2], int(sys.argv[3])
tdt = {"int32": torch.int32, "int64": torch.int64, "float32": torch.float32, "float64": torch.float64}[dt]
x = torch.empty(n, dtype=tdt, device="cuda")
ipmgen.fill_tensor(ipmgen.Spec(dt, n, "random", seed=1), x)
try:
    r = ipm.reduce(op, x)
    torch.cuda.synchronize()
    print(op, dt, "ok", r)
except Exception as e:
    print(op, dt, "FAIL", str(e)[:80])
