"""Small invocations of every kernel family for compute-sanitizer (memcheck / racecheck / synccheck)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ipmgen  # noqa: E402
from paper_1412_1127_b200 import ipm  # noqa: E402

TD = {"int32": torch.int32, "int64": torch.int64, "float32": torch.float32, "float64": torch.float64}
for dt in TD:
    for n in [0, 1, 7, 33, 1000, 70_001, 300_007]:
        for off in (0, 3):
            buf = torch.empty(n + off + 1, dtype=TD[dt], device="cuda")
            x = buf[off:off + n]
            if n:
                ipmgen.fill_device(ipmgen.Spec(dt, n, "random", seed=n), x.data_ptr(), 0, n,
                                   torch.cuda.current_stream().cuda_stream)
            for op in ["+", "max", "&&"] + (["^"] if dt.startswith("int") else []):
                ipm.reduce(op, x, init=np.array(1, dtype=x.cpu().numpy().dtype)[()])
    for kern in ("ldg", "tma"):
        ipm.set_option("seg_kernel", kern)
        for rows, cols, stride in [(5, 3, 4), (33, 100, 103), (9, 4097, 4100), (2, 40_000, 40_001), (300, 64, 64)]:
            x = torch.empty((rows - 1) * stride + cols + 3, dtype=TD[dt], device="cuda")
            ipmgen.fill_device(ipmgen.Spec(dt, x.numel(), "random", seed=1), x.data_ptr(), 0, x.numel(),
                               torch.cuda.current_stream().cuda_stream)
            ipm.reduce_segmented("+", x[1:], rows=rows, cols=cols, row_stride=stride)
    ipm.set_option("seg_kernel", "auto")
h = np.arange(100_000, dtype=np.int64)
ipm.reduce_host("+", h)
torch.cuda.synchronize()
print("sanitize_run: ok")
