"""World-size-2 gloo tests (CPU) of the multi-GPU path's host logic: shard ranges from libipm, the NCCL-id
bootstrap through the torch.distributed store, and the shard → partial → rank-ordered fold decomposition
(checked with the oracle standing in for each rank's kernel, since this container has no GPU)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, q):
    import sys
    sys.path.insert(0, ROOT)
    os.environ.update(MASTER_ADDR="127.0.0.1", MASTER_PORT=str(port))
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import ipmgen
        import oracle
        from paper_1412_1127_b200 import ipm
        res = {}
        # 1) NCCL unique-id bootstrap through the store (what ipm.Comm does before ncclCommInitRank)
        store = dist.distributed_c10d._get_default_store()
        nb = ipm.lib.ipm_comm_id_bytes()
        if rank == 0:
            import ctypes
            buf = ctypes.create_string_buffer(nb)
            rc = ipm.lib.ipm_comm_unique_id(buf)
            store.set("id", bytes(buf.raw) if rc == 0 else b"\0" * nb)
        ids = [None] * world
        dist.all_gather_object(ids, store.get("id"))
        res["id_same"] = all(i == ids[0] for i in ids) and len(ids[0]) == nb
        # 2) shard, partial, exchange, rank-ordered fold == whole fold
        out = []
        for op, dt, n in [("+", "int32", 1_000_003), ("^", "int64", 777), ("max", "float32", 100_001),
                          ("+", "float64", 50_001), ("&&", "int32", 3), ("|", "int64", 1), ("*", "int32", 12)]:
            spec = ipmgen.Spec(dt, n, "odd" if op == "*" else "random", seed=5)
            lo, hi = ipm.shard_range(n, rank, world)
            part = oracle.reduce(op, ipmgen.fill_host(spec, lo, hi - lo))[0]  # identity-started partial
            parts = [None] * world
            dist.all_gather_object(parts, part)
            init = np.array([3], dtype=spec.np_dtype)[0]
            merged = oracle.reduce(op, np.array(parts, dtype=spec.np_dtype), init=init)  # rank order, init once
            whole = oracle.reduce(op, ipmgen.fill_host(spec), init=init)
            if dt.startswith("float") and op == "+":
                ok = abs(float(merged[1]) - float(whole[1])) <= 1e-12 * abs(float(whole[1]))
            else:
                ok = merged[0] == whole[0]
            out.append((op, dt, bool(ok)))
        res["folds"] = out
        q.put((rank, res))
    finally:
        dist.destroy_process_group()


@pytest.mark.timeout(300)
def test_world2_gloo():
    world, port = 2, _free_port()
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    ps = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in ps:
        p.start()
    results = dict(q.get(timeout=240) for _ in range(world))
    for p in ps:
        p.join(60)
        assert p.exitcode == 0
    for r in range(world):
        assert results[r]["id_same"]
        assert all(ok for _, _, ok in results[r]["folds"]), results[r]["folds"]
