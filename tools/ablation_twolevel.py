"""Ablation of the gang-level merge: the paper's design point vs the one-launch path.

PAPER.md:205 (SRAD): IPMACC reduces "along threads of thread block on GPU and ... along thread block on CPU"
(a D2H copy of the per-block partials, then a host loop), while the CUDA version it compares against reduces
"by multiple serial kernel launches, all on the GPU". libipm does both levels in ONE kernel (last-CTA finish).
This tool times the three on B200, with the paper's statistic (harmonic mean of 30 runs) and its
time split (kernel / memory transfer / launch+host):

  one_launch   ipm_reduce: k_flat (both levels) + 4-byte D2H
  paper_2lvl   ipm_reduce_partials (level 1 on the GPU) + D2H of G 8-byte partials + host fold (level 2)
  multi_launch ipm_reduce_partials + ipm_finalize_partials (level 2 on the GPU, second launch) + 4-byte D2H

The host fold here is the ablation's own code (this file), not part of libipm.
    python tools/ablation_twolevel.py [--out profiles/r01_ablation_twolevel.json]
"""
import argparse
import json
import os
import statistics
import sys
import time

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import ipmgen  # noqa: E402
from paper_1412_1127_b200 import ipm  # noqa: E402


def hmean(xs):
    return len(xs) / sum(1.0 / x for x in xs)


def run_case(name, dt, n, reps=30):
    tdt = {"float32": torch.float32, "int32": torch.int32}[dt]
    x = torch.empty(n, dtype=tdt, device="cuda")
    ipmgen.fill_tensor(ipmgen.Spec(dt, n, "random", seed=1), x)
    scratch = torch.empty(1 << 27, dtype=torch.float32, device="cuda")  # 512 MiB: evicts L2 between reps
    acc_np = np.float64 if dt == "float32" else np.uint32
    init = np.array(0, dtype=dt)[()]
    res = {}

    def timeit(fn):
        walls, kerns, mems = [], [], []
        for i in range(reps + 3):
            scratch.fill_(1.0)
            torch.cuda.synchronize()
            with ipm.KernelTimer(8) as kt:
                t0 = time.perf_counter()
                val, mem_ms = fn()
                wall = (time.perf_counter() - t0) * 1e3
            if i >= 3:
                walls.append(wall)
                kerns.append(sum(kt.ms))
                mems.append(mem_ms)
        return val, {"wall_ms_hmean": hmean(walls), "wall_ms_median": statistics.median(walls),
                     "kernel_ms_hmean": hmean(kerns), "memcpy_ms_median": statistics.median(mems),
                     "host_and_launch_ms": statistics.median(walls) - statistics.median(kerns) -
                     statistics.median(mems)}

    ev0, ev1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)

    def one_launch():
        return ipm.reduce("+", x, init=init), 0.0

    def paper_two_level():
        parts = ipm.reduce_partials("+", x)
        ev0.record()
        h = parts.cpu()                    # D2H of the per-block partials ("copying intermediate data")
        ev1.record()
        ev1.synchronize()
        a = h.numpy().view(np.uint64)
        # the host loop over thread-block partials, as compiled host code would run it (vectorised numpy)
        if acc_np is np.float64:
            s = float(init) + float(np.add.reduce(a.view(np.float64)))
        else:
            s = np.uint32((int(init) + int(np.add.reduce((a & 0xFFFFFFFF).astype(np.uint32), dtype=np.uint32)))
                          & 0xFFFFFFFF)
        return (np.float32(s) if dt == "float32" else np.int32(np.uint32(s).view(np.int32))), ev0.elapsed_time(ev1)

    def multi_launch():
        parts = ipm.reduce_partials("+", x)
        out = ipm.finalize_partials("+", tdt, parts, init=init)
        ev0.record()
        v = out.cpu()
        ev1.record()
        ev1.synchronize()
        return v.numpy()[0], ev0.elapsed_time(ev1)

    vals = {}
    for label, fn in [("one_launch", one_launch), ("paper_2lvl", paper_two_level), ("multi_launch", multi_launch)]:
        vals[label], res[label] = timeit(fn)
    g, _ = ipm.flat_geometry(tdt, n)
    res["partials"] = g
    res["values_agree"] = bool(all(abs(float(vals[k]) - float(vals["one_launch"])) <=
                                   1e-6 * abs(float(vals["one_launch"])) for k in vals))
    res["n"] = n
    res["dtype"] = dt
    return name, res


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--out", default="gpurun_out/ablation_twolevel.json")
    a = ap.parse_args()
    out = {"note": "PAPER.md:205 two-level scheme vs GPU-only merges; harmonic mean of 30 runs (PAPER.md:122); "
                   "L2 flushed before every run"}
    for name, dt, n in [("SRAD-like image 2048x2048 float32", "float32", 2048 * 2048),
                        ("C1 2^20 int32", "int32", 1 << 20), ("C2 2^28 float32", "float32", 1 << 28)]:
        k, v = run_case(name, dt, n)
        out[k] = v
        print(k, json.dumps(v))
    json.dump(out, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
