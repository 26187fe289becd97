"""One marked-ragged call (and one warp-kernel call) on the power-law recipe, for an ncu launch list / capture.
usage: python tools/prof_marked.py [kind rows mean]"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ipmgen
from paper_1412_1127_b200 import ipm

kind, rows, mean = (sys.argv[1], int(sys.argv[2]), float(sys.argv[3])) if len(sys.argv) > 3 else ("powerlaw", 1 << 24, 16.0)
off = ipmgen.offsets_from_degrees(ipmgen.degrees(rows, seed=1, kind=kind, mean=mean))
nnz = int(off[-1])
offs = torch.from_numpy(off).cuda()
vals = torch.empty(nnz, dtype=torch.float32, device="cuda")
ipmgen.fill_tensor(ipmgen.Spec("float32", nnz, "random", seed=1), vals)
o = torch.empty(rows, dtype=torch.float32, device="cuda")
for kern in os.environ.get("KERNELS", "warp,marked").split(","):
    ipm.set_option("ragged_kernel", kern)
    for _ in range(2):
        ipm.reduce_ragged("+", vals, offs, out=o)
    torch.cuda.synchronize()
ipm.set_option("ragged_kernel", "auto")
print("prof_marked: ok")
