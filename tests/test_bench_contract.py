"""bench.py's output contract on CPU: the reference arm (the oracle, no GPU) prints exactly one JSON line on
stdout with the keys the driver reads."""
import json
import os
import subprocess
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def test_reference_arm_json_line():
    r = subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), "--impl", "reference", "--steps", "1",
                        "--warmup", "1"], capture_output=True, text=True, timeout=300, cwd=ROOT)
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    for k in ("impl", "metric", "value", "unit", "n_gpus", "steps", "warmup", "ms_per_step", "higher_is_better",
              "scaling", "vs_baseline", "dtype", "data", "config", "cpu_baseline", "e2e"):
        assert k in d, k
    assert d["impl"] == "reference" and d["value"] > 0 and d["unit"] == "GB/s"
    assert d["e2e"]["h2d_bytes_per_step"] == 0 and d["e2e"]["d2h_bytes_per_step"] == 0
    assert d["cpu_baseline"]["kind"] == "oracle" and d["cpu_baseline"]["cores"] == 1
    assert "workload" in d["config"]


def _bench(*args, env=None):
    e = dict(os.environ)
    e.pop("WORLD_SIZE", None)
    e.update(env or {})
    return subprocess.run([sys.executable, os.path.join(ROOT, "bench.py"), *args], capture_output=True, text=True,
                          timeout=300, cwd=ROOT, env=e)


def test_gpus_flag_without_launcher_spawns_ranks():
    """`python bench.py --gpus 2` with no launcher runs 2 ranks (here the CPU dry run of the wiring: gloo, shard
    plan, NCCL-id bootstrap through the store, exchange-path agreement) and prints ONE line from rank 0."""
    r = _bench("--gpus", "2", "--dry-run")
    assert r.returncode == 0, r.stderr[-2000:]
    lines = [l for l in r.stdout.splitlines() if l.strip()]
    assert len(lines) == 1, r.stdout
    d = json.loads(lines[0])
    assert d["dry_run"] and d["n_gpus"] == 2 and d["gpus_requested"] == 2
    assert d["shards"] == [[0, 1 << 33], [1 << 33, 1 << 34]] and d["shards_partition"]
    assert d["id_agree"] and d["ranks_same_path"] and d["exchange"] == "fused peer-memory"


def test_failed_probe_on_one_rank_switches_every_rank():
    r = _bench("--gpus", "3", "--dry-run", "--dry-run-fail-rank", "2")
    assert r.returncode == 0, r.stderr[-2000:]
    d = json.loads([l for l in r.stdout.splitlines() if l.strip()][0])
    assert d["n_gpus"] == 3 and d["exchange"] == "ncclAllGather+fold" and d["ranks_same_path"]
    assert d["shards_partition"] and d["shards"][-1][1] == 1 << 34


def test_world_size_must_match_gpus():
    r = _bench("--gpus", "2", "--dry-run", env={"WORLD_SIZE": "3", "RANK": "0"})
    assert r.returncode == 2 and "WORLD_SIZE=3" in r.stderr
