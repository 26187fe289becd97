"""Best-of-rounds table of gpurun_out/ab_ragged.txt (tools/gpu_ragged_ab.sh): one line per graph / op / dtype,
one column per library build and kernel. usage: ab_ragged_table.py [file]"""
import collections, re, sys

d = collections.defaultdict(lambda: collections.defaultdict(list))
for l in open(sys.argv[1] if len(sys.argv) > 1 else "gpurun_out/ab_ragged.txt"):
    m = re.match(r"(\S+)\s+(\S+)\s+(\S+)\s+rows=\s*(\d+)\s+mean=\s*(\d+)\s+(\S+)\s+(\S+).*?([\d.]+) GB/s", l)
    if m:
        lib, k, kind, rows, mean, op, dt, gbs = m.groups()
        d[(kind, rows, op, dt)][lib.replace("libipm", "").replace(".so", "") + "/" + k].append(float(gbs))
for key, v in d.items():
    print(f"{key[0]:8s} {key[1]:>9s} {key[2]:2s} {key[3]:8s} " + "  ".join(f"{n}={max(g):.0f}" for n, g in v.items()))
