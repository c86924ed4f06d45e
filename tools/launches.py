"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list."""
import collections, csv, statistics, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; ki = h.index('Kernel Name'); vi = h.index('Metric Value')
agg = collections.defaultdict(list)
for r in rows[hi + 1:]:
    if len(r) > vi:
        agg[r[ki].split('(')[0]].append(float(r[vi].replace(',', '')) / 1e3)
tot = sum(sum(v) for v in agg.values())
print("launches  total_us  share  median_us  kernel")
for k, v in sorted(agg.items(), key=lambda x: -sum(x[1])):
    print(f"{len(v):8d} {sum(v):9.1f} {100*sum(v)/tot:5.1f}% {statistics.median(v):9.1f}  {k[:80]}")
