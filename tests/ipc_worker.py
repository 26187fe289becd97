"""One rank of the cross-process fused-exchange test (tests/test_gpu_parity.py::test_dist_ipc_processes_one_gpu).

    python tests/ipc_worker.py RANK WORLD STORE_FILE

Bootstraps with ipm.Comm.ipc (CUDA IPC handles through a torch FileStore, no NCCL), reduces its shard of every
case in CASES through the product path (device shards and host shards) and prints one JSON line per result with
the result's bits. Never imports oracle/: the parent test computes the expected values."""
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

# (op, dtype, generator kind, n) — the parent builds the same ipmgen.Spec(dtype, n, kind, seed=SEED)
CASES = [("+", "float32", "random", 10_000_019), ("^", "int64", "random", 1_000_003),
         ("max", "float64", "signed", 777), ("*", "int32", "odd", 65_537), ("&&", "int32", "nonzero", 3)]
SEED = 11
INITS = (1, 2)


def main():
    rank, world, path = int(sys.argv[1]), int(sys.argv[2]), sys.argv[3]
    import numpy as np
    import torch
    import torch.distributed as dist

    import ipmgen
    from paper_1412_1127_b200 import ipm

    store = dist.FileStore(path, world)
    comm = ipm.Comm.ipc(rank, world, 0, store)
    assert comm.fused
    td = {"int32": torch.int32, "int64": torch.int64, "float32": torch.float32, "float64": torch.float64}
    for op, dt, kind, n in CASES:
        spec = ipmgen.Spec(dt, n, kind, seed=SEED)
        lo, hi = ipm.shard_range(n, rank, world)
        x = torch.empty(hi - lo, dtype=td[dt], device="cuda")
        if hi > lo:
            ipmgen.fill_tensor(spec, x, lo)
        torch.cuda.synchronize()
        for init in INITS:
            v = comm.reduce(op, x, init=np.dtype(dt).type(init))
            print(json.dumps({"rank": rank, "op": op, "dt": dt, "init": init, "path": "device",
                              "bits": np.array([v], dtype=dt).tobytes().hex()}), flush=True)
        h = ipmgen.fill_host(spec, lo, hi - lo)
        v = comm.reduce_host(op, h, init=np.dtype(dt).type(INITS[0]))
        print(json.dumps({"rank": rank, "op": op, "dt": dt, "init": INITS[0], "path": "host",
                          "bits": np.array([v], dtype=dt).tobytes().hex()}), flush=True)
    store.set(f"done/{rank}", b"1")
    for q in range(world):  # keep every rank's slot buffer mapped until all ranks finished
        store.get(f"done/{q}")
    comm.close()


if __name__ == "__main__":
    main()
