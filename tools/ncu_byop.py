"""Stall samples aggregated by SASS opcode from an ncu source-page CSV: python tools/ncu_byop.py src.csv"""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]; data = rows[2:]
idx = {c: i for i, c in enumerate(h)}
reasons = [c for c in h if c.startswith('stall_') and c.endswith('(Not Issued)')]
byop = collections.defaultdict(collections.Counter)
for r in data:
    tok = r[idx['Source']].strip().split()
    if not tok:
        continue
    op = (tok[1] if tok[0].startswith('@') else tok[0]).split('.')[0]
    byop[op]['exec'] += float(r[idx['Instructions Executed']] or 0)
    byop[op]['all'] += float(r[idx['Warp Stall Sampling (All Samples)']] or 0)
    for c in reasons:
        v = float(r[idx[c]] or 0)
        if v:
            byop[op][c.replace('stall_', '').replace(' (Not Issued)', '')] += v
T = sum(v['all'] for v in byop.values()) or 1
for op, v in sorted(byop.items(), key=lambda kv: -kv[1]['all'])[:int(sys.argv[2]) if len(sys.argv) > 2 else 16]:
    top = sorted([(k, x) for k, x in v.items() if k not in ('exec', 'all')], key=lambda t: -t[1])[:4]
    print(f"{op:8s} exec={v['exec']:14.0f} samples={v['all']:8.0f} ({100 * v['all'] / T:4.1f}%)  {top}")
