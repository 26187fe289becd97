"""Per-piece host overhead of the Python synchronous call path (GPU box)."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import time, torch, numpy as np, ctypes
from paper_1412_1127_b200 import ipm
x = torch.arange(1, (1<<20)+1, dtype=torch.int32, device="cuda")
def t(name, f, n=5000):
    for _ in range(200): f()
    t0=time.perf_counter()
    for _ in range(n): f()
    print(f"{name:40s} {(time.perf_counter()-t0)/n*1e6:7.2f} us")
t("torch.cuda.current_stream()", lambda: torch.cuda.current_stream())
t("current_stream().cuda_stream", lambda: torch.cuda.current_stream().cuda_stream)
t("torch._C._cuda_getCurrentRawStream(0)", lambda: torch._C._cuda_getCurrentRawStream(0))
t("torch.cuda.current_device()", lambda: torch.cuda.current_device())
t("ipm.workspace()", lambda: ipm.workspace())
t("_flat_arg", lambda: ipm._flat_arg(x))
t("np.array box", lambda: np.array([0], dtype=np.int32))
t("x.data_ptr()", lambda: x.data_ptr())
t("op_code", lambda: ipm.op_code("+"))
ws = ipm.workspace(); box = np.array([0], dtype=np.int32); s = torch.cuda.current_stream().cuda_stream
t("raw lib.ipm_reduce", lambda: ipm.lib.ipm_reduce(0, 0, x.data_ptr(), x.numel(), box.ctypes.data, ws.data_ptr(), s))
t("ipm.reduce(init=0)", lambda: ipm.reduce("+", x, init=np.int32(0)))
t("ipm.reduce()", lambda: ipm.reduce("+", x))
