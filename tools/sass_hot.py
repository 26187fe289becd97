"""Summarise an ncu SASS source export (gzip CSV): executed-instruction totals per straight-line run, hottest
first.  usage: python tools/sass_hot.py gpurun_out/ncu_X_sass.csv.gz [N]"""
import csv, gzip, sys

rows = list(csv.reader(gzip.open(sys.argv[1], "rt")))
h = rows[1]
ie, src, st = h.index("Instructions Executed"), h.index("Source"), h.index("Warp Stall Sampling (All Samples)")
ins = [(int(r[ie] or 0), int(r[st] or 0), r[src].strip()) for r in rows[2:]]
tot = sum(e for e, _, _ in ins)
runs, cur = [], None
for i, (e, s, t) in enumerate(ins):
    if cur and cur[2] == e:
        cur[1] = i
        cur[3] += s
    else:
        if cur:
            runs.append(cur)
        cur = [i, i, e, s]
runs.append(cur)
print(f"total warp-instructions executed {tot/1e6:.1f} M over {len(ins)} SASS lines")
for a, b, e, s in sorted(runs, key=lambda r: -(r[1] - r[0] + 1) * r[2])[: int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    n = b - a + 1
    print(f"{a:5d}-{b:5d} n={n:4d} exec={e:9d} total={n*e/1e6:7.1f}M stall_samples={s:6d}  first: {ins[a][2][:60]}")
