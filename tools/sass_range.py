"""Opcode histogram of a SASS address range: python tools/sass_range.py file.sass 0x2970 0x3a70 [--list]"""
import re, sys, collections
path, lo, hi = sys.argv[1], int(sys.argv[2], 16), int(sys.argv[3], 16)
ops = collections.Counter(); lines = []
for line in open(path):
    m = re.match(r'\s*/\*([0-9a-f]{4,})\*/\s+(.*?);', line)
    if not m: continue
    a = int(m.group(1), 16)
    if lo <= a < hi:
        ins = m.group(2).strip(); lines.append((a, ins))
        tok = ins.split()
        op = tok[1] if tok[0].startswith('@') else tok[0]
        ops[op.split('.')[0]] += 1
for op, n in ops.most_common(): print(f"{n:5d} {op}")
print("total", sum(ops.values()))
if '--list' in sys.argv:
    for a, ins in lines: print(hex(a), ins)
