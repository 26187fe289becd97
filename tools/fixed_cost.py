"""Fixed per-call cost of the flat clause: device time (library events) against size, 2^24..2^32 float32 `+`,
and a least-squares line T = a + bytes / BW over the sizes >= 2^27 (a = the per-call cost that makes 1 GiB
inputs run below the 64 GiB rate). Also an empty-kernel launch floor measured the same way (a 1-element reduce)."""
import os, statistics, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import ipmgen
from paper_1412_1127_b200 import ipm

dt = sys.argv[1] if len(sys.argv) > 1 else "float32"
tdt = getattr(torch, dt)
big = torch.empty(1 << 32, dtype=tdt, device="cuda")
ipmgen.fill_tensor(ipmgen.Spec(dt, big.numel(), "random", seed=1), big)
r = torch.empty(1, dtype=tdt, device="cuda")
t0 = time.perf_counter()
while time.perf_counter() - t0 < 0.5:
    ipm.reduce_async("+", big, out=r)
    torch.cuda.synchronize()
pts = []
for e in [0] + list(range(24, 33)):
    n = 1 << e if e else 1
    x = big[:n]
    for _ in range(3):
        ipm.reduce_async("+", x, out=r)
    with ipm.KernelTimer(30) as kt:
        for _ in range(30):
            ipm.reduce_async("+", x, out=r)
        torch.cuda.synchronize()
    med = statistics.median(kt.ms)
    nb = n * big.element_size()
    pts.append((e, nb, med))
    print(f"n=2^{e:2d} {nb/2**20:9.1f} MiB  {med*1e3:9.2f} us  {nb/med/1e6:8.1f} GB/s  sched={ipm.flat_schedule(tdt, n)}",
          flush=True)
X = np.array([p[1] for p in pts if p[0] >= 27], float)
Y = np.array([p[2] for p in pts if p[0] >= 27], float) * 1e-3
A = np.vstack([np.ones_like(X), X]).T
(a, b), *_ = np.linalg.lstsq(A, Y, rcond=None)
print(f"fit over 2^27..2^32: fixed {a*1e6:.2f} us + bytes / {1/b/1e9:.1f} GB/s")
