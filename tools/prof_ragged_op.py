"""One ragged call per kernel option on the power-law recipe for a given op / dtype, for ncu.
usage: KERNELS=marked,warp python tools/prof_ragged_op.py OP DTYPE"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ipmgen
from paper_1412_1127_b200 import ipm

op, dt = sys.argv[1], sys.argv[2]
off = ipmgen.offsets_from_degrees(ipmgen.degrees(1 << 24, seed=1, mean=16.0))
nnz = int(off[-1])
offs = torch.from_numpy(off).cuda()
vals = torch.empty(nnz, dtype=getattr(torch, dt), device="cuda")
ipmgen.fill_tensor(ipmgen.Spec(dt, nnz, "random", seed=1), vals)
for kern in os.environ.get("KERNELS", "warp,marked").split(","):
    ipm.set_option("ragged_kernel", kern)
    for _ in range(2):
        ipm.reduce_ragged(op, vals, offs)
    torch.cuda.synchronize()
ipm.set_option("ragged_kernel", "auto")
print("prof_ragged_op: ok")
