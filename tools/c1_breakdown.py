"""Where the C1 kernel time goes: device time of the library's flat kernel on 2^20 int32
with and without the cross-CTA finish, and of the smallest launch, each with L2 flushed before every call (a
512 MiB write, outside the timed kernel) and L2-warm. Events are the library's own (ipm_profile) on the launch
stream, around the kernel only.
  full      ipm_reduce_async: loads, CTA reduce, partial store, ticket, last CTA folds the partials, result store
  partials  ipm_reduce_partials: the same grid without the finish (partials only: the paper's first level)
  n=1       ipm_reduce_async on one element: a one-CTA launch with the finish (launch + chain floor)"""
import os, statistics, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
from paper_1412_1127_b200 import ipm

flush = torch.empty(512 << 20, dtype=torch.uint8, device="cuda")
x = torch.ones(1 << 20, dtype=torch.int32, device="cuda")
x1 = torch.ones(1, dtype=torch.int32, device="cuda")
r = torch.empty(1, dtype=torch.int32, device="cuda")
parts = torch.empty(4096, dtype=torch.int64, device="cuda")
calls = {
    "full": lambda: ipm.reduce_async("+", x, out=r),
    "partials": lambda: ipm.reduce_partials("+", x, out=parts),
    "n=1": lambda: ipm.reduce_async("+", x1, out=r),
}
for _ in range(200):
    for f in calls.values():
        f()
torch.cuda.synchronize()
for warm in (False, True):
    for name, f in calls.items():
        ms = []
        for _ in range(60):
            if not warm:
                flush.fill_(1)
            with ipm.KernelTimer(4) as kt:
                f()
                torch.cuda.synchronize()
            ms += kt.ms
        ms = ms[10:]
        print(f"{'L2-warm ' if warm else 'L2-flush'} {name:9s} median {statistics.median(ms)*1e3:6.2f} us  "
              f"min {min(ms)*1e3:6.2f} us  (n={len(ms)})", flush=True)
