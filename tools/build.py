"""Native build: the oracle (gcc), the input generator (gcc + nvcc) and the product library libipm (nvcc, sm_100a).

Everything is built IN-TREE so the .so files travel to the GPU box with the gpurun snapshot.
"""
from __future__ import annotations

import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
NVCC = os.environ.get("NVCC", "/usr/local/cuda/bin/nvcc")
ARCH = ["-gencode", "arch=compute_100a,code=sm_100a"]


def _nccl_dir() -> str:
    import nvidia.nccl  # torch-bundled NCCL 2.28
    return list(nvidia.nccl.__path__)[0]


def _run(cmd, cwd=ROOT):
    print("+", " ".join(cmd), flush=True)
    r = subprocess.run(cmd, cwd=cwd, capture_output=True, text=True)
    if r.returncode != 0:
        sys.stderr.write(r.stdout + r.stderr)
        raise RuntimeError(f"build step failed: {' '.join(cmd[:3])} ...")
    if r.stderr.strip():
        sys.stderr.write(r.stderr)
    return r


def _stale(out: str, srcs: list[str]) -> bool:
    if not os.path.exists(out):
        return True
    t = os.path.getmtime(out)
    return any(os.path.getmtime(s) > t for s in srcs)


def build_oracle(force: bool = False) -> str:
    out = os.path.join(ROOT, "oracle", "liboracle.so")
    src = os.path.join(ROOT, "oracle", "ipm_oracle.c")
    if force or _stale(out, [src]):
        # plain C, no fast-math: the oracle must follow IEEE semantics and x87 long double exactly
        _run(["gcc", "-std=c11", "-O2", "-fno-fast-math", "-ffp-contract=off", "-fPIC", "-shared", "-Wall",
              "-o", out, src, "-lm"])
    return out


def build_gen(force: bool = False) -> str:
    d = os.path.join(ROOT, "ipmgen")
    out = os.path.join(d, "libipmgen.so")
    srcs = [os.path.join(d, f) for f in ("gen_host.c", "gen_device.cu", "ipmgen.h", "ipmgen_elem.h")]
    if force or _stale(out, srcs):
        build_dir = os.path.join(ROOT, "build")
        os.makedirs(build_dir, exist_ok=True)
        o1 = os.path.join(build_dir, "gen_host.o")
        o2 = os.path.join(build_dir, "gen_device.o")
        _run(["gcc", "-std=c11", "-O2", "-ffp-contract=off", "-fPIC", "-c", "-o", o1, srcs[0]])
        _run([NVCC, *ARCH, "-O3", "-fmad=false", "-Xcompiler", "-fPIC", "-c", "-o", o2, srcs[1]])
        _run([NVCC, *ARCH, "-shared", "-o", out, o1, o2, "-lcudart"])
    return out


def ipm_sources() -> list[str]:
    d = os.path.join(ROOT, "paper_1412_1127_b200", "csrc")
    return sorted(os.path.join(d, f) for f in os.listdir(d) if f.endswith((".cu", ".cuh", ".h", ".cpp")))


def build_ipm(force: bool = False, extra: list[str] | None = None) -> str:
    out = os.path.join(ROOT, "paper_1412_1127_b200", "libipm.so")
    srcs = ipm_sources() + [os.path.join(ROOT, "include", "ipm.h")]
    if force or extra or _stale(out, srcs):
        nccl = _nccl_dir()
        cus = [s for s in srcs if s.endswith(".cu")]
        r = _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v", "-Xcompiler", "-fPIC,-Wall",
              "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include"),
              *(extra or []), "-shared", "-o", out, *cus,
              "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2", f"-Xlinker=-rpath={os.path.join(nccl, 'lib')}",
              "-lcudart"])
        # ptxas resource report (registers, spills per kernel): tests/test_build_report.py checks the hot kernels
        os.makedirs(os.path.join(ROOT, "build"), exist_ok=True)
        with open(PTXAS_LOG, "w") as f:
            f.write(r.stdout + r.stderr)
    return out


PTXAS_LOG = os.path.join(ROOT, "build", "ptxas_libipm.txt")


def build_variant(tag: str, defines: list[str]) -> str:
    """A/B build of libipm with extra -D flags into tools/bin/libipm_<tag>.so (travels to the GPU box; select it with
    IPM_LIB=...). Its ptxas report goes to tools/bin/ptxas_<tag>.txt."""
    nccl = _nccl_dir()
    out = os.path.join(ROOT, "tools", "bin", f"libipm_{tag}.so")
    os.makedirs(os.path.dirname(out), exist_ok=True)
    cus = [s for s in ipm_sources() if s.endswith(".cu")]
    r = _run([NVCC, *ARCH, "-O3", "-lineinfo", "-std=c++17", "-Xptxas", "-v", "-Xcompiler", "-fPIC,-Wall",
              "--expt-relaxed-constexpr", "-I", os.path.join(ROOT, "include"), "-I", os.path.join(nccl, "include"),
              *[f"-D{d}" for d in defines], "-shared", "-o", out, *cus,
              "-L", os.path.join(nccl, "lib"), "-l:libnccl.so.2", f"-Xlinker=-rpath={os.path.join(nccl, 'lib')}",
              "-lcudart"])
    with open(os.path.join(ROOT, "tools", "bin", f"ptxas_{tag}.txt"), "w") as f:
        f.write(r.stdout + r.stderr)
    return out


def build_tools(force: bool = False) -> None:
    """Library-context timing program (CUB DeviceReduce) that bench.py's suite runs if present. Optional: a
    failure here does not fail the build."""
    out = os.path.join(ROOT, "tools", "bin", "cub_context")
    src = os.path.join(ROOT, "tools", "cub_context.cu")
    if force or _stale(out, [src]):
        os.makedirs(os.path.dirname(out), exist_ok=True)
        try:
            _run([NVCC, *ARCH, "-O3", "-std=c++17", "-o", out, src])
        except RuntimeError as e:
            sys.stderr.write(f"optional tool not built: {e}\n")


def build_read_probe(force: bool = False) -> None:
    """Read-only HBM roofline probe (tools/read_probe.cu) that bench.py runs at N = 1. Optional."""
    out = os.path.join(ROOT, "tools", "bin", "read_probe")
    src = os.path.join(ROOT, "tools", "read_probe.cu")
    if force or _stale(out, [src]):
        os.makedirs(os.path.dirname(out), exist_ok=True)
        try:
            _run([NVCC, *ARCH, "-O3", "-std=c++17", "-o", out, src])
        except RuntimeError as e:
            sys.stderr.write(f"optional tool not built: {e}\n")


def build_cpu_omp(force: bool = False) -> None:
    """The OpenMP CPU baseline (BASELINE.md "CPU native baseline") that bench.py times at N = 1. Optional."""
    out = os.path.join(ROOT, "tools", "bin", "libcpu_omp.so")
    src = os.path.join(ROOT, "tools", "cpu_omp.c")
    if force or _stale(out, [src]):
        os.makedirs(os.path.dirname(out), exist_ok=True)
        try:
            _run(["gcc", "-std=c11", "-O3", "-march=x86-64-v2", "-fopenmp", "-fPIC", "-shared", "-o", out, src])
        except RuntimeError as e:
            sys.stderr.write(f"optional CPU baseline not built: {e}\n")


def build_all(force: bool = False) -> None:
    build_oracle(force)
    build_gen(force)
    build_ipm(force)
    build_tools(force)
    build_read_probe(force)
    build_cpu_omp(force)


if __name__ == "__main__":
    if len(sys.argv) > 2 and sys.argv[1] == "variant":  # build.py variant TAG DEF=1 DEF2=3 ...
        print(build_variant(sys.argv[2], sys.argv[3:]))
    else:
        build_all(force="--force" in sys.argv)
