"""Minimal driver for ncu captures: generate one config's input on the device, then launch the reduction a few
times (no oracle, no timing). Example:
    ncu --set full --clock-control none --import-source on -k regex:k_flat -s 2 -c 1 -o gpurun_out/prof \
        python tools/prof_run.py --config c5 --reps 3
"""
import argparse
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

import torch  # noqa: E402

import ipmgen  # noqa: E402
from paper_1412_1127_b200 import ipm  # noqa: E402

TD = {"int32": torch.int32, "int64": torch.int64, "float32": torch.float32, "float64": torch.float64}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="c5", choices=["c1", "c2", "c3", "c4", "c5", "stats", "dot", "2d"])
    ap.add_argument("--op", default="+")
    ap.add_argument("--dtype", default="float32")
    ap.add_argument("--reps", type=int, default=3)
    ap.add_argument("--log2n", type=int, default=None)
    ap.add_argument("--seg-kernel", default="auto", choices=["auto", "warp", "tma"])
    a = ap.parse_args()
    ipm.set_option("seg_kernel", a.seg_kernel)
    n = {"c1": 1 << 20, "c2": 1 << 28, "c3": 65536 * 4096, "c4": 1 << 30, "c5": 1 << 34, "stats": 1 << 28,
         "dot": 1 << 29, "2d": 16384 * 16384}[a.config]
    if a.log2n:
        n = 1 << a.log2n
    kind = {"+": "random", "*": "signs", "max": "signed", "min": "signed", "&": "allbits", "|": "random",
            "^": "random", "&&": "nonzero", "||": "random"}[a.op]
    spec = ipmgen.Spec(a.dtype, n, kind, seed=1)
    x = torch.empty(n, dtype=TD[a.dtype], device="cuda")
    ipmgen.fill_tensor(spec, x)
    torch.cuda.synchronize()
    for _ in range(a.reps):
        if a.config == "c3":
            ipm.reduce_segmented(a.op, x.view(65536, 4096))
        elif a.config == "stats":  # the suite's fused row: [sum, sum of squares, min, max] in one pass
            ipm.reduce_fused_async("stats", x)
        elif a.config == "dot":    # two streams of 2^28
            ipm.reduce_fused_async("dot", x[: 1 << 28], x[1 << 28:])
        elif a.config == "2d":     # a 16384 x 16000 window of a 16384 x 16384 image
            ipm.reduce_2d(a.op, x.view(16384, 16384)[:, :16000])
        else:
            ipm.reduce_async(a.op, x)
    torch.cuda.synchronize()
    print("done", n)


if __name__ == "__main__":
    main()
