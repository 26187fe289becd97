"""ncu driver: the ragged (CSR) clause, 3 calls. usage: prof_ragged.py [tile|warp] [powerlaw|const4096] [op] [dtype]
Default: the suite's power-law graph (2^24 rows, mean degree 16), float32 +, the default kernel."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ipmgen
from paper_1412_1127_b200 import ipm
kern = sys.argv[1] if len(sys.argv) > 1 else "auto"
graph = sys.argv[2] if len(sys.argv) > 2 else "powerlaw"
op = sys.argv[3] if len(sys.argv) > 3 else "+"
dt = sys.argv[4] if len(sys.argv) > 4 else "float32"
ipm.set_option("ragged_kernel", kern)
if graph == "powerlaw":
    off = ipmgen.offsets_from_degrees(ipmgen.degrees(1 << 24, seed=1, mean=16.0))
else:
    off = ipmgen.offsets_from_degrees(ipmgen.degrees(1 << 16, seed=1, kind="const", mean=4096.0))
vals = torch.empty(int(off[-1]), dtype=getattr(torch, dt), device="cuda")
ipmgen.fill_tensor(ipmgen.Spec(dt, vals.numel(), "random", seed=1), vals)
offs = torch.from_numpy(off).cuda()
for _ in range(3):
    ipm.reduce_ragged(op, vals, offs)
torch.cuda.synchronize()
print("done")
