"""ncu driver: the ragged (CSR) clause on the suite's power-law graph (2^24 rows, mean degree 16), 3 calls."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import ipmgen
from paper_1412_1127_b200 import ipm
off = ipmgen.offsets_from_degrees(ipmgen.degrees(1 << 24, seed=1, mean=16.0))
vals = torch.empty(int(off[-1]), dtype=torch.float32, device="cuda")
ipmgen.fill_tensor(ipmgen.Spec("float32", vals.numel(), "random", seed=1), vals)
offs = torch.from_numpy(off).cuda()
for _ in range(3):
    ipm.reduce_ragged("+", vals, offs)
torch.cuda.synchronize()
print("done")
