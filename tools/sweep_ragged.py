"""Writes the ragged recipes' offsets (DESIGN.md input recipe) to /tmp and runs tools/bin/sweep_ragged on each."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import ipmgen

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
for kind, rows, mean in [("powerlaw", 1 << 24, 16.0), ("const", 1 << 16, 4096.0), ("const", 1 << 25, 4.0)]:
    off = ipmgen.offsets_from_degrees(ipmgen.degrees(rows, seed=1, kind=kind, mean=mean))
    path = f"/tmp/off_{kind}_{rows}.bin"
    off.astype("int64").tofile(path)
    print(kind, rows, mean, flush=True)
    subprocess.run([os.path.join(ROOT, "tools/bin/sweep_ragged"), path], check=False)
