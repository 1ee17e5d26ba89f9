"""Static SASS summary: basic blocks of a cuobjdump -sass dump with many FP64
instructions (the hot loops), with their opcode mix.

    cuobjdump -sass -fun NAME lib.so > x.sass; python tools/sass_blocks.py x.sass [min_fp64]
"""
import collections
import re
import sys

pat = re.compile(r"^\s+/\*([0-9a-f]+)\*/\s+(?:@!?U?P[0-9T]+\s+)?([A-Z0-9_]+)[.\s;]")
blocks, cur = [], []
for line in open(sys.argv[1]):
    if re.match(r"^\s*\.L_x_\d+:", line):
        if cur:
            blocks.append(cur)
        cur = []
        continue
    m = pat.match(line)
    if not m:
        continue
    cur.append(m.group(2))
    if m.group(2) in ("BRA", "EXIT", "RET", "CALL", "BRX", "JMP"):
        blocks.append(cur)
        cur = []
if cur:
    blocks.append(cur)
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 60
for b in blocks:
    c = collections.Counter(b)
    f64 = c["DMUL"] + c["DADD"] + c["DFMA"]
    if f64 >= thr:
        print(len(b), "instrs, fp64", f64, dict(c.most_common(14)))
