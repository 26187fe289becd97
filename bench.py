"""bench.py — the headline benchmark: `reduction(+:sum)` sharded over 2^34 float32 (BASELINE.json config 5) on N GPUs.

    python bench.py [--gpus N] [--steps K] [--warmup W] [--impl ours|reference] [--no-suite] [--no-e2e]
    torchrun --nproc-per-node N bench.py --gpus N ...        (one process per GPU, NCCL)
    python bench.py --gpus N ...   without a launcher re-launches itself under torch.distributed.run (N ranks);
                                   under a launcher WORLD_SIZE must equal --gpus (else exit 2)
    python bench.py --gpus N --dry-run   the N-rank wiring on CPU (gloo): shards, id bootstrap, path decision

One step = one execution of the clause over the whole 2^34-element iteration space: every rank runs the flat
reduction kernel over its contiguous shard (rows a1-a6 of SURVEY.md §8(a)); the kernel's last CTA exchanges the
8-byte accumulator partials with the other ranks over NVLink peer memory and folds them in rank order (a9), result
left in device memory — one launch per rank per step (fallback if peer mapping fails: ncclAllGather + a one-warp
fold kernel).
Inputs are generated on the device (ipmgen) before timing and are larger than L2 (64/N GiB per GPU), so no
flush is needed between steps. Timed with CUDA events between two barriers, max over ranks.

Rank 0 prints ONE JSON line. Besides the contract keys it carries:
  roofline      the flat kernel's HBM roofline: algorithmic bytes per launch / its live per-launch event time
  cpu_baseline  the CPU oracle (test infrastructure, tests/ + here only) timed on a bounded sample, 1 core
  e2e           the same metric through ipm_reduce_host_dist: pinned host shards -> devices + the rank exchange,
                with the box's plain pinned H2D bandwidth as its roofline
  result_check  the timed steps' result against the oracle's fold of the whole 2^34-element input (host cores)
  per_gpu       `value` is the whole-job aggregate (bench contract); the metric's per-GPU figures are here
  suite         (N=1) the other BASELINE configs device-timed: C1 latency, C2 per op, C3 segmented, C4 per op,
                the NEXT rows (fused, 2-D, ragged), and torch / CUB reductions on the same shapes as context
`--impl reference` times the CPU oracle as the reference arm on the same metric (no GPU work).
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

N_TOTAL = 1 << 34          # config 5: 2^34 float32 = 64 GiB
ELEM = 4
METRIC = "reduction GB/s per GPU (% of B200 HBM peak) and elements/s at 1/2/4/8 GPUs"
WORKLOAD = "C5: sharded reduction(+:sum) over 2^34 float32 (dyadic uniform [0,1024), seed 1), fp64 accumulation"


def peaks():
    p = os.path.join(ROOT, "MEASURED_PEAKS.json")
    try:
        d = json.load(open(p))
        return float(d["hbm_gbs"]), "measured (MEASURED_PEAKS.json hbm_gbs: torch copy, read+write bytes)"
    except Exception:
        return 6650.0, "fallback (B200_PROFILING.md 6.65 TB/s)"


def host_cores():
    try:
        return len(os.sched_getaffinity(0))
    except Exception:
        return os.cpu_count()


def host_cpu_model():
    try:
        for line in open("/proc/cpuinfo"):
            if line.startswith("model name"):
                return line.split(":", 1)[1].strip()
    except Exception:
        pass
    return "unknown"


class Clocks:
    """Sample SM clock and throttle reasons with NVML during the timed region."""
    REASONS = {0x1: "gpu_idle", 0x2: "applications_clocks_setting", 0x4: "sw_power_cap", 0x8: "hw_slowdown",
               0x20: "sw_thermal_slowdown", 0x40: "hw_thermal_slowdown", 0x80: "hw_power_brake_slowdown",
               0x100: "display_clock_setting"}

    def __init__(self, device_index: int):
        self.samples, self.reasons, self.ok = [], set(), False
        try:
            import pynvml
            pynvml.nvmlInit()
            self.nv = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(device_index)
            self.max_mhz = pynvml.nvmlDeviceGetMaxClockInfo(self.h, pynvml.NVML_CLOCK_SM)
            self.ok = True
        except Exception as e:  # pragma: no cover
            self.err = str(e)
        self._stop = threading.Event()

    def _run(self):
        while not self._stop.is_set():
            try:
                self.samples.append(self.nv.nvmlDeviceGetClockInfo(self.h, self.nv.NVML_CLOCK_SM))
                r = self.nv.nvmlDeviceGetCurrentClocksEventReasons(self.h)
                for bit, name in self.REASONS.items():
                    if r & bit and name != "gpu_idle":
                        self.reasons.add(name)
            except Exception:
                pass
            time.sleep(0.01)

    def __enter__(self):
        if self.ok:
            self.t = threading.Thread(target=self._run, daemon=True)
            self.t.start()
        return self

    def __exit__(self, *a):
        if self.ok:
            self._stop.set()
            self.t.join()

    def summary(self):
        if not self.ok or not self.samples:
            return {"sm_mhz": None, "sm_max_mhz": None, "reasons": ["unavailable"]}
        return {"sm_mhz": statistics.median(self.samples), "sm_max_mhz": self.max_mhz,
                "reasons": sorted(self.reasons), "samples": len(self.samples)}


def harmonic(xs):
    return len(xs) / sum(1.0 / x for x in xs) if xs and all(x > 0 for x in xs) else None


# --------------------------------------------------------------------------------------------- reference arm
def run_reference(args, rank, world):
    """The CPU oracle as the reference arm: each step folds a bounded sample of the C5 input on 1 host core."""
    if rank != 0:
        return
    import numpy as np

    import ipmgen
    import oracle
    sample = 1 << 27  # elements per step (512 MiB of float32): about 1 s per step on one core
    spec = ipmgen.Spec("float32", N_TOTAL, "random", seed=1)
    a = ipmgen.fill_host(spec, 0, sample)
    times = []
    for i in range(args.warmup + args.steps):
        t0 = time.perf_counter()
        oracle.reduce("+", a)
        dt = time.perf_counter() - t0
        if i >= args.warmup:
            times.append(dt)
    per_step = sum(times) / len(times)
    gbs = sample * ELEM / per_step / 1e9
    line = {"impl": "reference", "metric": METRIC, "value": gbs, "unit": "GB/s", "n_gpus": args.gpus,
            "steps": args.steps, "warmup": args.warmup, "ms_per_step": per_step * 1e3, "higher_is_better": True,
            "scaling": "strong", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n_total": N_TOTAL, "sample_elements_per_step": sample},
            "cpu_baseline": {"value": gbs, "unit": "GB/s", "cores": 1, "kind": "oracle",
                             "sample": f"first 2^27 elements of the C5 input per step (host array), "
                                       f"long double Neumaier fold; host has {host_cores()} cores",
                             "cpu_model": host_cpu_model()},
            "e2e": {"value": gbs, "unit": "GB/s", "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0},
            "elements_per_s": sample / per_step, "gpu_launches": 0}
    print(json.dumps(line), file=OUT, flush=True)
    del np


# --------------------------------------------------------------------------------------------- our arm
def cpu_baseline_oracle(x_dev, seconds_target=10.0):
    """The oracle, as it stands, timed on the host over a bounded prefix of this rank's input."""
    import numpy as np

    import oracle
    n = min(x_dev.numel(), 1 << 30)
    a = x_dev[:n].cpu().numpy()
    # time a small piece first to size the sample to ~seconds_target
    t0 = time.perf_counter()
    oracle.reduce("+", a[: 1 << 22])
    per = (time.perf_counter() - t0) / (1 << 22)
    m = int(min(n, max(1 << 22, seconds_target / max(per, 1e-12))))
    t0 = time.perf_counter()
    oracle.reduce("+", a[:m])
    dt = time.perf_counter() - t0
    del np
    return {"value": m * ELEM / dt / 1e9, "unit": "GB/s", "cores": 1, "kind": "oracle",
            "sample": f"first {m} elements of rank 0's C5 shard (host copy), long double Neumaier fold, "
                      f"{dt:.1f} s; host has {host_cores()} cores", "elements_per_s": m / dt,
            "cpu_model": host_cpu_model()}


def cpu_native_omp(x_dev, reps=3):
    """BASELINE.md's CPU native baseline: OpenMP `parallel for simd reduction(+:s)` in the input's native precision
    (float32 accumulators) on all host cores (tools/cpu_omp.c), over the same bounded prefix as the oracle."""
    import ctypes

    lib_path = os.path.join(ROOT, "tools", "bin", "libcpu_omp.so")
    if not os.path.exists(lib_path):
        return {"value": None, "unit": "GB/s", "kind": "openmp", "error": "tools/bin/libcpu_omp.so not built"}
    L = ctypes.CDLL(lib_path)
    L.cpu_omp_sum_f32.restype = ctypes.c_float
    L.cpu_omp_sum_f32.argtypes = [ctypes.c_void_p, ctypes.c_int64]
    n = min(x_dev.numel(), 1 << 30)
    a = x_dev[:n].cpu().numpy()
    L.cpu_omp_sum_f32(a.ctypes.data, n)  # warm (first touch of the threads)
    best, res = None, None
    for _ in range(reps):
        t0 = time.perf_counter()
        res = L.cpu_omp_sum_f32(a.ctypes.data, n)
        dt = time.perf_counter() - t0
        best = dt if best is None else min(best, dt)
    return {"value": n * ELEM / best / 1e9, "unit": "GB/s", "cores": int(L.cpu_omp_threads()), "kind": "openmp",
            "sample": f"first {n} elements of rank 0's C5 shard (host copy), float32 accumulators, best of {reps}",
            "result": float(res), "elements_per_s": n / best, "cpu_model": host_cpu_model()}


def suite(ipm, torch, ipmgen, peak):
    """The other BASELINE configs, device-timed with the library's per-kernel events (rank 0, N=1)."""
    out = {}
    ws = ipm.workspace()

    def timed(fn, reps=20, flush=None):
        t0 = time.perf_counter()
        while True:  # clock spin-up: at least 3 calls and 0.1 s of back-to-back work before timing
            for _ in range(3):
                fn()
            torch.cuda.synchronize()
            if time.perf_counter() - t0 > 0.1:
                break
        with ipm.KernelTimer(4 * reps) as kt:
            for _ in range(reps):
                if flush is not None:
                    flush()
                fn()
            torch.cuda.synchronize()
        return kt.ms

    # C1: 2^20 int32 (+), L2-resident: flush L2 (write 512 MiB) before each rep; report latency
    n = 1 << 20
    x = torch.empty(n, dtype=torch.int32, device="cuda")
    ipmgen.fill_tensor(ipmgen.Spec("int32", n, "iota", param=1), x)
    scratch = torch.empty(1 << 27, dtype=torch.float32, device="cuda")
    res = torch.empty(1, dtype=torch.int32, device="cuda")
    ms = timed(lambda: ipm.reduce_async("+", x, out=res, ws=ws), flush=lambda: scratch.fill_(1.0))
    ok = int(res.item()) == 524288
    t0 = time.perf_counter()
    for _ in range(50):
        ipm.reduce("+", x, init=0)
    host_us = (time.perf_counter() - t0) / 50 * 1e6
    out["C1_int32_add_2^20"] = {"kernel_us_median": statistics.median(ms) * 1e3, "kernel_us_min": min(ms) * 1e3,
                                "sync_call_us": host_us, "GB/s": n * 4 / statistics.median(ms) / 1e6,
                                "closed_form_ok": ok, "note": "L2 flushed before each rep; latency-bound"}
    del x, scratch
    # C2: 2^28 float32 / float64, + * max min
    for dt, tdt in (("float32", torch.float32), ("float64", torch.float64)):
        n = 1 << 28
        for op in ("+", "*", "max", "min"):
            kind = {"+": "random", "*": "signs", "max": "signed", "min": "signed"}[op]
            spec = ipmgen.Spec(dt, n, kind, seed=1, plant="factor" if op == "*" else "none",
                               nplant=64 if op == "*" else 0)
            x = torch.empty(n, dtype=tdt, device="cuda")
            ipmgen.fill_tensor(spec, x)
            r = torch.empty(1, dtype=tdt, device="cuda")
            ms = timed(lambda: ipm.reduce_async(op, x, out=r, ws=ws))
            med = statistics.median(ms)
            gbs = x.numel() * x.element_size() / med / 1e6
            out[f"C2_{dt}_{op}_2^28"] = {"kernel_ms_median": med, "GB/s": gbs, "frac": gbs / peak}
            del x
    # C3: 65536 x 4096 float32 row sums (segmented)
    rows, cols = 65536, 4096
    x = torch.empty(rows * cols, dtype=torch.float32, device="cuda")
    ipmgen.fill_tensor(ipmgen.Spec("float32", rows * cols, "random", seed=1), x)
    o = torch.empty(rows, dtype=torch.float32, device="cuda")
    ms = timed(lambda: ipm.reduce_segmented("+", x.view(rows, cols), out=o, ws=ws))
    med = statistics.median(ms)
    gbs = (rows * cols * 4 + rows * 4) / med / 1e6
    out["C3_float32_segmented_65536x4096"] = {"kernel_ms_median": med, "GB/s": gbs, "frac": gbs / peak}
    del x, o
    # C4: 2^30 int32 / int64, & | ^ && ||
    for dt, tdt in (("int32", torch.int32), ("int64", torch.int64)):
        n = 1 << 30
        x = torch.empty(n, dtype=tdt, device="cuda")
        for op in ("&", "|", "^", "&&", "||"):
            spec = {"&": ipmgen.Spec(dt, n, "allbits", seed=1, plant="clearbit", nplant=8),
                    "|": ipmgen.Spec(dt, n, "const", param=0, seed=1, plant="setbit", nplant=8),
                    "^": ipmgen.Spec(dt, n, "random", seed=1),
                    "&&": ipmgen.Spec(dt, n, "nonzero", seed=1, plant="value", nplant=1, plant_param=0),
                    "||": ipmgen.Spec(dt, n, "const", param=0, seed=1, plant="value", nplant=1, plant_param=3)}[op]
            ipmgen.fill_tensor(spec, x)
            r = torch.empty(1, dtype=tdt, device="cuda")
            ms = timed(lambda: ipm.reduce_async(op, x, out=r, ws=ws), reps=10)
            med = statistics.median(ms)
            gbs = x.numel() * x.element_size() / med / 1e6
            out[f"C4_{dt}_{op}_2^30"] = {"kernel_ms_median": med, "GB/s": gbs, "frac": gbs / peak}
        del x
    # library context (not targets): torch's own reductions on the same shapes, CUDA events on torch's stream
    def torch_timed(fn, reps=20):
        t0 = time.perf_counter()
        while time.perf_counter() - t0 < 0.1:
            fn()
            torch.cuda.synchronize()
        evs = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(reps)]
        for a, b in evs:
            a.record()
            fn()
            b.record()
        torch.cuda.synchronize()
        return statistics.median([a.elapsed_time(b) for a, b in evs])
    ctx = {}
    for dt, tdt, n in (("float32", torch.float32, 1 << 28), ("float64", torch.float64, 1 << 28),
                       ("int32", torch.int32, 1 << 30)):
        x = torch.empty(n, dtype=tdt, device="cuda")
        ipmgen.fill_tensor(ipmgen.Spec(dt, n, "random", seed=1), x)
        for name, fn in (("torch.sum", lambda: x.sum()), ("torch.amax", lambda: x.amax())):
            ms = torch_timed(fn)
            ctx[f"{name}_{dt}_2^{n.bit_length() - 1}"] = {"ms": ms, "GB/s": n * x.element_size() / ms / 1e6}
        del x
    out["library_context_torch"] = ctx

    # NEXT rows: several variables in one pass (SRAD statistics, dot) and a strided 2-D region
    n = 1 << 28
    x = torch.empty(n, dtype=torch.float32, device="cuda")
    ipmgen.fill_tensor(ipmgen.Spec("float32", n, "random", seed=1), x)
    y = torch.empty(n, dtype=torch.float32, device="cuda")
    ipmgen.fill_tensor(ipmgen.Spec("float32", n, "random", seed=2), y)
    r = torch.empty(4, dtype=torch.float32, device="cuda")
    for sig, nbytes in (("stats", n * 4), ("dot", 2 * n * 4)):
        ms = timed(lambda: ipm.reduce_fused_async(sig, x, y if sig == "dot" else None, out=r, ws=ws))
        med = statistics.median(ms)
        out[f"fused_{sig}_float32_2^28"] = {"kernel_ms_median": med, "GB/s": nbytes / med / 1e6,
                                            "frac": nbytes / med / 1e6 / peak}
    del y
    rows, cols, stride = 16384, 16000, 16384  # a 16384 x 16000 window of a 16384 x 16384 float32 image
    x2 = x[: rows * stride]
    r1 = torch.empty(1, dtype=torch.float32, device="cuda")
    ms = timed(lambda: ipm.lib.ipm_reduce_2d_async(0, 2, x2.data_ptr(), rows, cols, stride, None, r1.data_ptr(),
                                                   ws.data_ptr(), torch.cuda.current_stream().cuda_stream))
    med = statistics.median(ms)
    out["2d_float32_16384x16000_stride16384"] = {"kernel_ms_median": med, "GB/s": rows * cols * 4 / med / 1e6,
                                                 "frac": rows * cols * 4 / med / 1e6 / peak}
    del x, x2
    # NEXT row 2: ragged (CSR) rows — power-law degree graph, 2^24 rows, mean degree 16 (BFS-style)
    import numpy as np
    off = ipmgen.offsets_from_degrees(ipmgen.degrees(1 << 24, seed=1, mean=16.0))
    nnz = int(off[-1])
    vals = torch.empty(nnz, dtype=torch.float32, device="cuda")
    ipmgen.fill_tensor(ipmgen.Spec("float32", nnz, "random", seed=1), vals)
    offs = torch.from_numpy(off).cuda()
    o = torch.empty(1 << 24, dtype=torch.float32, device="cuda")
    ms = timed(lambda: ipm.reduce_ragged("+", vals, offs, out=o, ws=ws))
    med = statistics.median(ms)  # one record per call, covering all of its kernels
    nbytes = nnz * 4 + off.size * 8 + (1 << 24) * 4
    out["ragged_float32_powerlaw_2^24rows"] = {"nnz": nnz, "max_degree": int(np.diff(off).max()),
                                               "ms_median": med, "GB/s": nbytes / med / 1e6,
                                               "frac": nbytes / med / 1e6 / peak, "kernel": "auto",
                                               "kernels_per_call": 3,
                                               "kernels_note": "k_ragged_vec (runs: mean row length 16 < 256), "
                                                               "k_ragged_lpr (returns after its gate), k_ragged_fix"}
    # the same graph through the two-pass path (ipm_reduce_ragged_marked, scratch from torch's allocator)
    ipm.set_option("ragged_kernel", "marked")
    try:
        ms = timed(lambda: ipm.reduce_ragged("+", vals, offs, out=o, ws=ws))
    finally:
        ipm.set_option("ragged_kernel", "auto")
    med = statistics.median(ms)
    out["ragged_float32_powerlaw_2^24rows_marked"] = {
        "ms_median": med, "GB/s": nbytes / med / 1e6, "frac": nbytes / med / 1e6 / peak, "kernel": "marked",
        "kernels_per_call": 4, "kernels_note": "memset of the scratch, k_ragged_mark, k_ragged_mk, k_ragged_fix"}
    del vals, offs, o
    torch.cuda.empty_cache()
    # library context: CUB's DeviceReduce / DeviceSegmentedReduce on the same shapes, including this ragged graph
    # (tools/cub_context.cu, a separate process; skipped if it was not built)
    cub = os.path.join(ROOT, "tools", "bin", "cub_context")
    if os.path.exists(cub):
        import tempfile
        torch.cuda.synchronize()
        with tempfile.NamedTemporaryFile(suffix=".bin") as f:
            off.astype(np.int64).tofile(f.name)
            try:
                r = subprocess.run([cub, f.name], capture_output=True, text=True, timeout=300)
                out["library_context_cub"] = {
                    d["case"]: {"ms": d["ms"], "GB/s": d["GB/s"]}
                    for d in (json.loads(l) for l in r.stdout.splitlines() if l.startswith("{"))}
            except (subprocess.TimeoutExpired, ValueError) as e:
                out["library_context_cub"] = {"error": str(e)[:200]}
    # read-only HBM roofline probe: the simplest streaming read kernel, several shapes, 8 GiB;
    # a separate process (tools/read_probe.cu), skipped if it was not built
    probe = os.path.join(ROOT, "tools", "bin", "read_probe")
    if os.path.exists(probe):
        torch.cuda.synchronize()
        torch.cuda.empty_cache()
        try:
            r = subprocess.run([probe], capture_output=True, text=True, timeout=300)
            rows = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
            best = [d["read_probe_best_GBs"] for d in rows if "read_probe_best_GBs" in d]
            out["read_probe"] = {"best_GBs": best[0] if best else None,
                                 "variants": [d for d in rows if "probe" in d]}
            # the same probe over 1 GiB (the C2 / C3 size): the per-call cost of a 1 GiB stream, the fair
            # denominator for those rows
            r = subprocess.run([probe, "1024"], capture_output=True, text=True, timeout=300)
            rows = [json.loads(l) for l in r.stdout.splitlines() if l.startswith("{")]
            best = [d["read_probe_best_GBs"] for d in rows if "read_probe_best_GBs" in d]
            out["read_probe"]["best_GBs_1GiB"] = best[0] if best else None
            if best:
                for k, v in out.items():
                    if isinstance(v, dict) and "GB/s" in v and (k.startswith("C2_float32") or k.startswith("C3_")):
                        v["frac_of_read_probe_1GiB"] = v["GB/s"] / best[0]
        except (subprocess.TimeoutExpired, ValueError) as e:
            out["read_probe"] = {"error": str(e)[:200]}
    return out


def all_ranks_ok(local_bad: int, world: int, device) -> bool:
    """Every rank must take the same exchange path: True iff no rank reported a problem (MAX all-reduce of the
    per-rank flags; gloo on CPU in --dry-run, NCCL on the GPUs)."""
    import torch
    import torch.distributed as dist
    bad = torch.tensor([int(local_bad)], device=device)
    if world > 1:
        dist.all_reduce(bad, op=dist.ReduceOp.MAX)
    return int(bad.item()) == 0


def shard_partition_ok(ipm, world, rank):
    """This rank's contiguous shard of the C5 iteration space, and whether all ranks' shards tile [0, N) exactly."""
    import torch.distributed as dist
    lo, hi = ipm.shard_range(N_TOTAL, rank, world)
    shards = [(lo, hi)]
    if world > 1:
        shards = [None] * world
        dist.all_gather_object(shards, (lo, hi))
    ok = shards[0][0] == 0 and shards[-1][1] == N_TOTAL and all(
        a[1] == b[0] and a[0] <= a[1] for a, b in zip(shards, shards[1:]))
    return lo, hi, shards, ok


def run_dry(args, rank, world):
    """--dry-run: the N-rank wiring of the ours arm WITHOUT a GPU (gloo on CPU): shard plan, the NCCL-id bootstrap
    through the torch.distributed store, the fused-probe fallback decision. No kernel runs; the line says so."""
    import torch.distributed as dist

    from paper_1412_1127_b200 import ipm
    if world > 1:
        dist.init_process_group("gloo")
        store = dist.distributed_c10d._get_default_store()
    else:
        store = dist.HashStore()
    lo, hi, shards, part_ok = shard_partition_ok(ipm, world, rank)
    try:
        uid = ipm.Comm.bootstrap_id(rank, store, key="bench_dry_id")
        id_src = "ncclGetUniqueId"
    except ipm.IpmError:  # no usable network interface for NCCL's id on this host: the store path still runs
        if rank == 0:
            store.set("bench_dry_id", os.urandom(ipm.lib.ipm_comm_id_bytes()))
        uid = store.get("bench_dry_id")
        id_src = "random bytes (ncclGetUniqueId unavailable)"
    ids = [uid]
    if world > 1:
        ids = [None] * world
        dist.all_gather_object(ids, uid)
    # the fused-exchange probe: a rank whose probe failed (simulated by --dry-run-fail-rank) switches ALL ranks
    fused = all_ranks_ok(int(rank == args.dry_run_fail_rank), world, "cpu")
    paths = [fused]
    if world > 1:
        paths = [None] * world
        dist.all_gather_object(paths, fused)
    if rank == 0:
        line = {"metric": METRIC, "value": None, "unit": "GB/s", "n_gpus": world, "gpus_requested": args.gpus,
                "dry_run": True, "note": "wiring only (gloo on CPU): no GPU, no kernel, no timing",
                "shards": shards, "shards_partition": part_ok, "id_agree": all(i == ids[0] for i in ids),
                "id_source": id_src, "exchange": "fused peer-memory" if fused else "ncclAllGather+fold",
                "ranks_same_path": all(p == paths[0] for p in paths)}
        print(json.dumps(line), file=OUT, flush=True)
    if world > 1:
        dist.destroy_process_group()


def result_check(result, threads=None):
    """The oracle's answer for the WHOLE C5 input (2^34 elements): the plain compensated left fold, generated and
    folded on the host cores in 256 contiguous pieces merged in piece order (oracle.reduce_spec_split, SURVEY.md
    §8(d)); part of the CPU-baseline leg (the oracle's one use here besides cpu_baseline and the reference arm)."""
    import numpy as np

    import ipmgen
    import oracle
    t0 = time.perf_counter()
    want_t, want_ld, used = oracle.reduce_spec_split("+", ipmgen.Spec("float32", N_TOTAL, "random", seed=1),
                                                     pieces=256, threads=threads)
    dt = time.perf_counter() - t0
    rel = abs(float(np.longdouble(result) - want_ld)) / float(want_ld)
    return {"gpu": float(result), "oracle_ld": float(want_ld), "oracle_f32": float(want_t), "rel_err": rel,
            "tol": 1e-5, "ok": rel <= 1e-5, "bits_equal": bool(np.float32(result) == want_t),
            "oracle_seconds": dt, "oracle_threads": used,
            "how": "oracle.reduce_spec_split: 256 contiguous pieces of the generated C5 input, compensated long "
                   "double folds on the host cores, merged in piece order"}


def ctypes_err(ipm, comm):
    import ctypes
    e = ctypes.c_int(0)
    ipm.lib.ipm_comm_error(comm._h, ctypes.byref(e))
    return e.value


def run_ours(args, rank, world, local_rank):
    import numpy as np
    import torch
    import torch.distributed as dist

    import ipmgen
    from paper_1412_1127_b200 import ipm

    torch.cuda.set_device(local_rank)
    dev = torch.cuda.current_device()
    if world > 1:
        dist.init_process_group("nccl", device_id=torch.device("cuda", local_rank))
        store = dist.distributed_c10d._get_default_store()
    else:
        store = dist.HashStore()
    peak, peak_src = peaks()

    lo, hi, _, part_ok = shard_partition_ok(ipm, world, rank)
    assert part_ok, "the ranks' shards do not tile the iteration space"
    n_shard = hi - lo
    spec = ipmgen.Spec("float32", N_TOTAL, "random", seed=1)
    x = torch.empty(n_shard, dtype=torch.float32, device="cuda")
    ipmgen.fill_device(spec, x.data_ptr(), lo, n_shard, torch.cuda.current_stream().cuda_stream)
    comm = ipm.Comm(rank, world, dev, store=store)
    comm_fused = comm.fused
    if comm_fused and world > 1:
        # probe the fused peer-memory exchange once with a short timeout; fall back to NCCL everywhere if any rank
        # saw a peer time out (every rank must take the same path)
        ipm.set_option("dist_timeout_ms", 5000)
        probe = torch.ones(1024, dtype=torch.float32, device="cuda")
        got = comm.reduce_async("+", probe).cpu().numpy()[0]
        err = ctypes_err(ipm, comm)
        ok = all_ranks_ok(int(err or got != 1024.0 * world), world, "cuda")
        ipm.set_option("dist_timeout_ms", 30000)
        if not ok:
            ipm.set_option("dist_mode", "nccl")
            comm_fused = False
    ws = ipm.workspace()
    out = torch.empty(1, dtype=torch.float32, device="cuda")
    init = np.float32(0.0)

    def barrier():
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        torch.cuda.synchronize()

    # clock spin-up (setup, untimed): ~0.25 s of back-to-back steps so the timed steps run at steady clocks.
    # The count is a function of the shard size only, identical on every rank (every call is collective).
    spin = max(3, int(0.25 / (N_TOTAL / world * ELEM / 7.0e12)))
    spin = min(spin, 2000)
    for _ in range(spin):
        comm.reduce_async("+", x, init=init, out=out, ws=ws)
    torch.cuda.synchronize()
    for _ in range(args.warmup):
        comm.reduce_async("+", x, init=init, out=out, ws=ws)
    barrier()

    stream = torch.cuda.current_stream()
    step_ev = [(torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)) for _ in range(args.steps)]
    start, stop = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    with Clocks(dev) as clk, ipm.KernelTimer(4 * args.steps + 8) as kt:
        start.record(stream)
        for i in range(args.steps):
            step_ev[i][0].record(stream)
            comm.reduce_async("+", x, init=init, out=out, ws=ws)
            step_ev[i][1].record(stream)
        stop.record(stream)
        stop.synchronize()
    barrier()
    ms_local = start.elapsed_time(stop)
    t = torch.tensor([ms_local], dtype=torch.float64, device="cuda")
    if world > 1:
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
    ms_total = float(t.item())
    ms_step = ms_total / args.steps
    step_ms = [a.elapsed_time(b) for a, b in step_ev]
    kern_ms = [m for m, k in zip(kt.ms, kt.kinds) if k == 0]
    result = float(out.item())
    ranks_agree = True
    if world > 1:
        allr = [None] * world
        dist.all_gather_object(allr, out.cpu().numpy().tobytes())
        ranks_agree = all(r == allr[0] for r in allr)

    total_bytes = N_TOTAL * ELEM
    value = total_bytes / (ms_step / 1e3) / 1e9  # whole-job GB/s
    kern_avg = sum(kern_ms) / len(kern_ms)
    achieved = n_shard * ELEM / (kern_avg / 1e3) / 1e9

    # e2e through the public host-array call: pinned host shard -> device each step (ipm_reduce_host)
    e2e = None
    if not args.no_e2e:
        try:
            e2e_steps = max(1, min(args.steps, 3))
            host = torch.empty(n_shard, dtype=torch.float32, pin_memory=True)
            host.copy_(x)
            del x
            torch.cuda.empty_cache()
            # the e2e roofline: plain pinned host -> device copy bandwidth of this box (1 GiB cudaMemcpyAsync)
            pn = min(n_shard, 1 << 28)
            dbuf = torch.empty(pn, dtype=torch.float32, device="cuda")
            dbuf.copy_(host[:pn], non_blocking=True)
            h0, h1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            h0.record(stream)
            for _ in range(3):
                dbuf.copy_(host[:pn], non_blocking=True)
            h1.record(stream)
            h1.synchronize()
            h2d_gbs = 3 * pn * ELEM / (h0.elapsed_time(h1) / 1e3) / 1e9
            del dbuf
            for _ in range(1):
                comm.reduce_host("+", host, init=init, ws=ws)  # warm (allocates the staging buffers)
            barrier()
            t0 = torch.cuda.Event(enable_timing=True)
            t1 = torch.cuda.Event(enable_timing=True)
            t0.record(stream)
            for _ in range(e2e_steps):  # every rank: its pinned host shard -> device, exchange, global result
                part = comm.reduce_host("+", host, init=init, ws=ws)
            t1.record(stream)
            t1.synchronize()
            barrier()
            e_ms = torch.tensor([t0.elapsed_time(t1) / e2e_steps], dtype=torch.float64, device="cuda")
            if world > 1:
                dist.all_reduce(e_ms, op=dist.ReduceOp.MAX)
            e2e = {"value": total_bytes / (float(e_ms.item()) / 1e3) / 1e9, "unit": "GB/s",
                   "h2d_bytes_per_step": total_bytes, "d2h_bytes_per_step": 4 * world, "steps": e2e_steps,
                   "ms_per_step": float(e_ms.item()), "path": "ipm_reduce_host_dist: pinned host shard per rank, 64 MiB "
                   "chunks double-buffered H2D overlapped with the reduce kernels, then the rank exchange",
                   "host_result_rank0": float(part),
                   "h2d_probe_GBs_per_gpu": h2d_gbs,
                   "frac_of_h2d": total_bytes / (float(e_ms.item()) / 1e3) / 1e9 / (h2d_gbs * world),
                   "h2d_probe": "1 GiB pinned host -> device cudaMemcpyAsync, 3 reps, same process, before the e2e "
                                "steps; frac_of_h2d = e2e value / (probe x n_gpus)"}
            del host
            ipm.lib.ipm_release_staging()
        except Exception as ex:  # pinned allocation can fail on small hosts: say so, keep the device number
            e2e = {"value": None, "unit": "GB/s", "h2d_bytes_per_step": total_bytes, "d2h_bytes_per_step": 4 * world,
                   "error": repr(ex)[:200]}
    else:
        del x
    torch.cuda.empty_cache()

    if rank == 0:
        cpu = None  # the oracle baseline runs at N = 1 only (a bounded host sample; the same at any N)
        cpu_omp = None
        if not args.no_cpu and world == 1:
            xs = torch.empty(min(n_shard, 1 << 30), dtype=torch.float32, device="cuda")
            ipmgen.fill_device(spec, xs.data_ptr(), lo, xs.numel(), torch.cuda.current_stream().cuda_stream)
            cpu = cpu_baseline_oracle(xs)
            try:
                cpu_omp = cpu_native_omp(xs)
            except Exception as ex:  # a baseline only: never fail the bench line over it
                cpu_omp = {"value": None, "unit": "GB/s", "kind": "openmp", "error": repr(ex)[:200]}
            del xs
        # the oracle's answer for the whole 2^34 input against the timed steps' result (same on every rank)
        rcheck = None
        if not args.no_check:
            try:
                rcheck = result_check(result)
            except Exception as ex:  # the check must not hide the measurement; report why it did not run
                rcheck = {"ok": None, "error": repr(ex)[:200]}
        st = suite(ipm, torch, ipmgen, peak) if (world == 1 and not args.no_suite) else None
        traffic = None
        tp = os.path.join(ROOT, "profiles", "r01_traffic.json")
        if os.path.exists(tp):
            try:
                tr = json.load(open(tp))
                if int(tr.get("n_per_launch", -1)) == n_shard:
                    traffic = tr["dram_bytes_per_launch"]
            except Exception:
                pass
        line = {
            "metric": METRIC, "value": value, "unit": "GB/s", "n_gpus": world, "steps": args.steps,
            "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "strong",
            "vs_baseline": None, "dtype": "f64", "input_dtype": "f32", "data": "synthetic",
            "config": {"workload": WORKLOAD, "n_total": N_TOTAL, "n_per_gpu": n_shard,
                       "parallelism": f"shard{world}+" + ("fused peer-memory exchange in the reduction kernel"
                                                          if comm_fused else "ncclAllGather(8B/rank)+fold kernel"),
                       "l2": "inputs larger than L2 (64/N GiB per GPU): no flush needed"},
            "value_scope": "aggregate over all n_gpus (bench contract); per-GPU figures under per_gpu",
            "per_gpu": {"value": value / world, "unit": "GB/s", "pct_of_hbm_peak": 100.0 * value / world / peak,
                        "pct_of_8TBs": 100.0 * value / world / 8000.0, "elements_per_s": N_TOTAL / world /
                        (ms_step / 1e3)},
            "per_gpu_GBs": value / world, "pct_of_hbm_peak": 100.0 * value / world / peak,
            "elements_per_s": N_TOTAL / (ms_step / 1e3),
            "roofline": {"bound": "hbm", "achieved": achieved, "peak": peak, "unit": "GB/s",
                         "frac": achieved / peak, "traffic": traffic, "peak_source": peak_src,
                         "kernel": "k_flat_guided<Red<+,f32>,256,2,pipelined> (one launch per step per GPU)",
                         "bytes_per_launch": n_shard * ELEM, "kernel_ms_avg": kern_avg,
                         "kernel_ms_min": min(kern_ms), "launches_timed": len(kern_ms),
                         "vs_8TBs_spec": achieved / 8000.0},
            "step_stats_ms": {"harmonic_mean": harmonic(step_ms), "median": statistics.median(step_ms),
                              "min": min(step_ms)},
            "cpu_baseline": cpu, "cpu_native": cpu_omp, "e2e": e2e,
            "gpu_launches": (1 if comm_fused else 2) * args.steps,
            "gpu_launches_note": ("per step: 1 k_flat_guided (reduction + NVLink peer-memory exchange in one kernel)"
                                  if comm_fused else "per step: 1 k_flat_guided + 1 k_finalize (plus NCCL's own "
                                  "AllGather kernel)"),
            "clocks": clk.summary(), "result_rank0": result, "spinup_steps": spin,
            "ranks_agree": ranks_agree, "result_check": rcheck,
        }
        if st is not None:
            line["suite"] = st
            rp = (st.get("read_probe") or {}).get("best_GBs")
            if rp:  # the third denominator: the best plain streaming read measured in this run
                line["roofline"]["read_probe_GBs"] = rp
                line["roofline"]["frac_of_read_probe"] = achieved / rp
        print(json.dumps(line), file=OUT, flush=True)
    comm.close()
    if world > 1:
        dist.destroy_process_group()


def spawn_ranks(n: int) -> int:
    """`python bench.py --gpus N` without torchrun: relaunch this command under torch.distributed.run with N
    processes on this node (127.0.0.1 rendezvous); rank 0's JSON line goes to our stdout."""
    import socket
    with socket.socket() as so:
        so.bind(("127.0.0.1", 0))
        port = so.getsockname()[1]
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr=127.0.0.1", f"--master-port={port}", os.path.abspath(__file__), *sys.argv[1:]]
    print("bench.py: launching " + " ".join(cmd), file=sys.stderr, flush=True)
    return subprocess.run(cmd, stdout=OUT.fileno(), stderr=sys.stderr.fileno()).returncode


def _claim_stdout():
    """Everything below may print (NCCL's version banner goes to the C-level stdout); keep the real stdout for
    the one JSON line and send all other output to stderr."""
    sys.stdout.flush()
    real = os.fdopen(os.dup(1), "w")
    os.dup2(2, 1)
    return real


OUT = sys.stdout


def main():
    global OUT
    OUT = _claim_stdout()
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=30)
    ap.add_argument("--warmup", type=int, default=3)
    ap.add_argument("--impl", default="ours", choices=["ours", "reference"])
    ap.add_argument("--no-suite", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-cpu", action="store_true")
    ap.add_argument("--no-check", action="store_true", help="skip the whole-input oracle check of the C5 result")
    ap.add_argument("--dry-run", action="store_true", help="N-rank wiring on CPU (gloo), no GPU work")
    ap.add_argument("--dry-run-fail-rank", type=int, default=-1, help="--dry-run: this rank's exchange probe fails")
    args = ap.parse_args()
    if args.gpus < 1:
        ap.error("--gpus must be >= 1")
    if "WORLD_SIZE" not in os.environ and args.gpus > 1:
        sys.exit(spawn_ranks(args.gpus))       # no launcher: start one process per GPU ourselves
    rank = int(os.environ.get("RANK", 0))
    world = int(os.environ.get("WORLD_SIZE", 1))
    local_rank = int(os.environ.get("LOCAL_RANK", 0))
    if world != args.gpus:
        print(f"bench.py: --gpus {args.gpus} but the launcher started WORLD_SIZE={world} ranks", file=sys.stderr)
        sys.exit(2)
    if args.dry_run:
        run_dry(args, rank, world)
        return
    if args.impl == "reference":
        run_reference(args, rank, world)
        return
    run_ours(args, rank, world, local_rank)


if __name__ == "__main__":
    main()
