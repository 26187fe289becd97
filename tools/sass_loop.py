"""Instruction count of the innermost backward-branch loop(s) of a kernel's SASS (cuobjdump -sass output).
usage: cuobjdump -sass X.o | python tools/sass_loop.py FUNCTION_SUBSTRING"""
import re, sys

want = sys.argv[1]
cur, funcs = None, {}
for line in sys.stdin:
    m = re.search(r"Function : (\S+)", line)
    if m:
        cur = m.group(1)
        funcs[cur] = []
        continue
    m = re.match(r"\s+/\*([0-9a-f]{4,})\*/\s+(.*?);", line)
    if m and cur:
        funcs[cur].append((int(m.group(1), 16), m.group(2).strip()))
for name, ins in funcs.items():
    if want not in name:
        continue
    addr = [a for a, _ in ins]
    for a, t in ins:
        m = re.search(r"BRA (?:`\(\.L_x_\d+\)|0x([0-9a-f]+))", t)
        if m and m.group(1):
            tgt = int(m.group(1), 16)
            if tgt < a:
                body = [x for x in ins if tgt <= x[0] <= a]
                ops = {}
                for _, tt in body:
                    op = tt.split()[0] if not tt.startswith("@") else tt.split()[1]
                    ops[op] = ops.get(op, 0) + 1
                print(f"{name[:60]}: loop {tgt:#x}-{a:#x} {len(body)} instructions; "
                      + ", ".join(f"{k} {v}" for k, v in sorted(ops.items(), key=lambda kv: -kv[1])[:8]))
