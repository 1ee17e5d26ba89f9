"""Summarise an ncu report's SASS source page: executed instructions by
opcode class and by execution count (hot-loop body), plus stall samples."""
import collections
import csv
import re
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
kern, cur = [], None
for r in rows:
    if r and r[0] == "Kernel Name":
        cur = []
        kern.append(cur)
        continue
    if cur is not None:
        cur.append(r)
k = kern[-1]
hdr = k[0]
ix = {h: i for i, h in enumerate(hdr)}
c, smp, bycount = collections.Counter(), collections.Counter(), collections.defaultdict(collections.Counter)
tot = 0
lines = []
for r in k[1:]:
    if len(r) < len(hdr):
        continue
    src = r[ix["Source"]].strip()
    op = re.sub(r"^@!?U?P[0-9T]+\s+", "", src).split()[0].split(".")[0] if src else "?"
    n = int(r[ix["Instructions Executed"]] or 0)
    s = int(r[ix["Warp Stall Sampling (All Samples)"]] or 0)
    c[op] += n
    smp[op] += s
    tot += n
    bycount[n][op] += 1
    lines.append((n, s, src))
fp = sum(c[x] for x in ["DMUL", "DADD", "DFMA", "DSETP", "DMNMX"])
print(f"total warp instructions {tot}, fp64 fraction {fp / max(tot, 1):.3f}")
for op, n in c.most_common(25):
    print(f"  {op:8s} {n:11d} {100 * n / tot:5.1f}%  stall samples {smp[op]}")
print("instructions by execution count (count: #static instr, top opcodes):")
for n in sorted(bycount, key=lambda x: -x * sum(bycount[x].values()))[:8]:
    ops = bycount[n]
    print(f"  {n:9d}: {sum(ops.values()):5d}  {dict(ops.most_common(10))}")
if len(sys.argv) > 2:
    with open(sys.argv[2], "w") as f:
        for n, s, src in lines:
            f.write(f"{n:9d} {s:5d}  {src}\n")
