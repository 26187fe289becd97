"""Registers / spills / shared memory per instantiation of the kernels whose name contains a pattern, from a ptxas
-v log. usage: ptxas_kernels.py LOG PATTERN"""
import re, subprocess, sys

cur, out = None, []
for l in open(sys.argv[1]).read().splitlines():
    m = re.search(r"Function properties for (\S+)", l)
    if m:
        cur = m.group(1) if sys.argv[2] in m.group(1) else None
        spill = None
        continue
    if cur and "stack frame" in l:
        spill = l.strip()
    if cur and "Used" in l and "registers" in l:
        dm = subprocess.run(["c++filt", cur], capture_output=True, text=True).stdout.strip().replace("ipm::", "")
        out.append(f"{dm[:70]:70s} {l.split('info    :')[-1].strip()} | {spill}")
        cur = None
print("\n".join(out))
