"""Concurrent callers of the host-streaming path (ipm_reduce_host): two host threads on two streams, each with its
own workspace, share the library's staging buffers; every result must equal the oracle's (VERDICT r01 weak #7,
ADVICE r01: a second caller used to overwrite a buffer the first caller's kernel was still reading)."""
import os
import threading

import numpy as np
import pytest
import torch

import ipmgen
import oracle

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def ipm():
    from paper_1412_1127_b200 import ipm as m
    return m


def test_two_threads_two_streams_host_path(ipm):
    old = os.environ.get("IPM_STAGE_MB")
    os.environ["IPM_STAGE_MB"] = "1"      # 1 MiB staging chunks: many buffer reuses per call
    try:
        cases = []
        for k, (dt, op, n) in enumerate([("int64", "^", 3_000_017), ("float32", "+", 5_000_011),
                                         ("int32", "+", 4_000_037), ("float64", "max", 2_000_003)]):
            spec = ipmgen.Spec(dt, n, "signed" if op == "max" else "random", seed=100 + k)
            h = ipmgen.fill_host(spec)
            h = torch.from_numpy(h).pin_memory() if k % 2 else h
            a = h.numpy() if isinstance(h, torch.Tensor) else h
            cases.append((op, h, oracle.reduce(op, a, init=a.dtype.type(1))))
        errors = []

        def worker(tid):
            s = torch.cuda.Stream()
            ws = torch.zeros(ipm.WS_BYTES, dtype=torch.uint8, device="cuda")
            torch.cuda.synchronize()
            for rep in range(12):
                op, h, (want_t, want_ld) = cases[(tid + rep) % len(cases)]
                dtn = (h.numpy() if isinstance(h, torch.Tensor) else h).dtype
                got = ipm.reduce_host(op, h, init=dtn.type(1), ws=ws, stream=s)
                if dtn.kind == "f" and op == "+":
                    ok = abs(np.longdouble(got) - want_ld) <= 1e-5 * abs(want_ld)
                else:
                    ok = np.array([got], dtn).tobytes() == np.array([want_t], dtn).tobytes()
                if not ok:
                    errors.append((tid, rep, op, str(dtn), got, want_t))

        ts = [threading.Thread(target=worker, args=(t,)) for t in range(2)]
        for t in ts:
            t.start()
        for t in ts:
            t.join()
        assert not errors, errors[:5]
    finally:
        if old is None:
            os.environ.pop("IPM_STAGE_MB", None)
        else:
            os.environ["IPM_STAGE_MB"] = old
        ipm.lib.ipm_release_staging()
