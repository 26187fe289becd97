import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ipmgen
from paper_1412_1127_b200 import ipm
n = int(sys.argv[1]) if len(sys.argv) > 1 else (1 << 30)
ws = ipm.workspace()
for op in ["&", "|", "^", "|", "&", "+", "max", "|"]:
    x = torch.empty(n, dtype=torch.int32, device="cuda")
    ipmgen.fill_tensor(ipmgen.Spec("int32", n, "random", seed=1), x)
    torch.cuda.synchronize()
    print("before", op, "counter", ws[4288:4296].view(torch.int64).item(), "ticket", ws[0:4].view(torch.int32).item(),
          flush=True)
    r = ipm.reduce(op, x)
    torch.cuda.synchronize()
    print("after", op, r, "counter", ws[4288:4296].view(torch.int64).item(), "ticket",
          ws[0:4].view(torch.int32).item(), flush=True)
print("ok")
