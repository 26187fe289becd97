"""A/B of two builds of libipm on ONE box: each round runs this script's child mode under IPM_LIB=<lib> for
every lib, interleaved (box-to-box HBM speed varies ~3 %). usage: python tools/ab_lib.py LIB_A LIB_B [rounds]"""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
CASES = [("flat", "float32", "+", 1 << 28), ("flat", "float64", "max", 1 << 28), ("flat", "int64", "&&", 1 << 30),
         ("seg", "float32", "+", 65536 * 4096), ("2d", "float32", "+", 16384 * 16384),
         ("stats", "float32", "+", 1 << 28), ("sum_sumsq", "float32", "+", 1 << 28), ("minmax", "float32", "+", 1 << 28),
         ("dot", "float32", "+", 1 << 29), ("stats", "float64", "+", 1 << 28), ("2d", "float32", "max", 16384 * 16384), ("2d", "int32", "^", 16384 * 16384),
         ("2d", "float64", "+", 16384 * 16384), ("seg", "float32", "max", 65536 * 4096),
         ("seg", "float64", "+", 65536 * 4096), ("seg", "int32", "^", 65536 * 4096), ("seg", "int64", "min", 65536 * 4096),
         ("2d", "int32", "+", 16384 * 16384), ("2d", "int64", "+", 8192 * 16384), ("2d", "int64", "max", 8192 * 16384),
         ("2d", "float64", "max", 8192 * 16384), ("2d", "float32", "&&", 16384 * 16384), ("2d", "int32", "*", 16384 * 16384),
         ("flat", "float64", "+", 1 << 28), ("flat", "float64", "min", 1 << 28), ("flat", "int64", "max", 1 << 30),
         ("flat", "int64", "*", 1 << 30), ("flat", "float32", "max", 1 << 28)]
if os.environ.get("AB_CASES"):  # e.g. AB_CASES=2d: only cases of that kind
    CASES = [c for c in CASES if c[0] in os.environ["AB_CASES"].split(",")]


def child():
    import statistics
    import time
    sys.path.insert(0, ROOT)
    import torch
    import ipmgen
    from paper_1412_1127_b200 import ipm
    TD = {"float32": torch.float32, "float64": torch.float64, "int64": torch.int64, "int32": torch.int32}
    out = {}
    for kind, dt, op, n in CASES:
        x = torch.empty(n, dtype=TD[dt], device="cuda")
        ipmgen.fill_tensor(ipmgen.Spec(dt, n, "random", seed=1), x)
        r = torch.empty(1, dtype=TD[dt], device="cuda")

        def call():
            if kind == "flat":
                ipm.reduce_async(op, x, out=r)
            elif kind == "seg":
                ipm.reduce_segmented(op, x.view(65536, 4096))
            elif kind == "2d":
                ipm.reduce_2d(op, x.view(-1, 16384)[:, :16000])
            elif kind == "dot":
                ipm.reduce_fused_async("dot", x[: n // 2], x[n // 2:])
            else:
                ipm.reduce_fused_async(kind, x)
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 0.2:
            call()
        torch.cuda.synchronize()
        with ipm.KernelTimer(64) as kt:
            for _ in range(30):
                call()
            torch.cuda.synchronize()
        nbytes = n * x.element_size() * (16000 / 16384 if kind == "2d" else 1)
        out[f"{kind} {dt} {op}"] = nbytes / statistics.median(kt.ms) / 1e6
        del x
    print(json.dumps(out))


if __name__ == "__main__":
    if sys.argv[1] == "--child":
        child()
        sys.exit(0)
    libs = [a for a in sys.argv[1:] if not a.isdigit()]
    rounds = next((int(a) for a in sys.argv[1:] if a.isdigit()), 3)
    res = {lib: [] for lib in libs}
    for _ in range(rounds):
        for lib in libs:
            path, *envs = lib.split("::")  # LIB::VAR=VALUE::... sets extra environment for that build's runs
            env = dict(os.environ, IPM_LIB=path, **dict(e.split("=", 1) for e in envs))
            p = subprocess.run([sys.executable, __file__, "--child"], env=env, capture_output=True, text=True)
            res[lib].append(json.loads(p.stdout.strip().splitlines()[-1]))
    for k in res[libs[0]][0]:
        print(f"{k:24s} " + "  ".join(f"{os.path.basename(lib)[:24]}: " + " ".join(f"{r[k]:7.1f}" for r in res[lib])
                                       for lib in libs) + "  GB/s")
