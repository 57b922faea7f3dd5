"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list: per-kernel count, time, share."""
import collections, csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if r]
hdr_i = [i for i, r in enumerate(rows) if r[0] == "ID"][0]
hdr = rows[hdr_i]
ki, vi, ui = hdr.index("Kernel Name"), hdr.index("Metric Value"), hdr.index("Metric Unit")
scale = {"ns": 1e-6, "nsecond": 1e-6, "us": 1e-3, "usecond": 1e-3, "ms": 1.0, "msecond": 1.0, "s": 1e3, "second": 1e3}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hdr_i + 1:]:
    name = r[ki].split("(")[0]
    tot[name] += float(r[vi].replace(",", "")) * scale[r[ui]]
    cnt[name] += 1
T = sum(tot.values())
print(f"{'launches':>8} {'total ms':>12} {'share':>7}  kernel")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{cnt[k]:8d} {tot[k]:12.3f} {100 * tot[k] / T:6.2f}%  {k}")
print(f"{sum(cnt.values()):8d} {T:12.3f} 100.00%  (all)")
