"""Static schedule summary of the hot basic blocks of a cuobjdump -sass dump:
per block, the instruction count, FP64 count, the sum of the encoded stall
counts (a lone warp's minimum traversal time, variable-latency waits
excluded) and the stall histogram by opcode.

    cuobjdump -sass -fun NAME lib.so > x.sass; python tools/sass_stalls.py x.sass [min_fp64]
"""
import collections
import re
import sys

ins = re.compile(r"^\s+/\*([0-9a-f]{4,})\*/\s+(?:@!?U?P[0-9T]+\s+)?([A-Z0-9_]+)([.\w]*)\s.*?/\* 0x([0-9a-f]{16}) \*/")
ctl = re.compile(r"^\s+/\* 0x([0-9a-f]{16}) \*/")
blocks, cur, pending = [], [], None
for line in open(sys.argv[1]):
    if re.match(r"^\s*\.L_x_\d+:", line):
        if cur:
            blocks.append(cur)
        cur = []
        continue
    m = ins.match(line)
    if m:
        pending = (m.group(2), m.group(3))
        continue
    m = ctl.match(line)
    if m and pending:
        hi = int(m.group(1), 16)
        stall = (hi >> 41) & 0xF
        yld = (hi >> 45) & 1
        wmask = (hi >> 52) & 0x3F
        cur.append((pending[0], stall, yld, wmask))
        if pending[0] in ("BRA", "EXIT", "RET", "CALL", "BRX", "JMP"):
            blocks.append(cur)
            cur = []
        pending = None
if cur:
    blocks.append(cur)
thr = int(sys.argv[2]) if len(sys.argv) > 2 else 60
for b in blocks:
    f64 = sum(1 for o, *_ in b if o in ("DMUL", "DADD", "DFMA"))
    if f64 < thr:
        continue
    tot = sum(s for _, s, _, _ in b)
    by = collections.Counter()
    n = collections.Counter()
    for o, s, _, _ in b:
        by[o] += s
        n[o] += 1
    waits = sum(1 for _, _, _, w in b if w)
    hist = collections.Counter(s for o, s, _, _ in b if o in ("DMUL", "DADD", "DFMA"))
    print(f"{len(b)} instrs, fp64 {f64}, sum(stall) {tot}, fp64 pipe cycles {2 * f64}, "
          f"instrs waiting on a scoreboard {waits}")
    print("   stall cycles by opcode:", dict(by.most_common(10)))
    print("   fp64 stall histogram:", dict(sorted(hist.items())))
