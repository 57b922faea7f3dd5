"""Per-instruction stall attribution from `ncu --page source --csv --print-source sass`.
usage: python tools/ncu_stalls.py src.csv [reason ...]  -> top instructions by not-issued samples"""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; data = rows[2:]
idx = {c: i for i, c in enumerate(h)}
reasons = [c for c in h if c.startswith('stall_') and c.endswith('(Not Issued)')]
tot = collections.Counter()
per = []
for r in data:
    s = {c: float(r[idx[c]] or 0) for c in reasons}
    for c, v in s.items(): tot[c] += v
    per.append((sum(s.values()), r[idx['Address']][-5:], r[idx['Source']].strip()[:60], s))
T = sum(tot.values())
print("total not-issued samples", T)
for c, v in tot.most_common(12): print(f"  {c:40s} {v:8.0f} {100*v/T:5.1f}%")
print("top instructions:")
for tsum, a, src, s in sorted(per, key=lambda t: -t[0])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    top = ", ".join(f"{k.split('_',1)[1].replace(' (Not Issued)','')}={v:.0f}" for k, v in sorted(s.items(), key=lambda kv: -kv[1])[:3] if v)
    print(f"{tsum:7.0f} {a} {src:60s} {top}")
