"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list (per-kernel mean/share)."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]; data = rows[hi + 1:]
ki = h.index('Kernel Name'); mi = h.index('Metric Name'); vi = h.index('Metric Value'); ui = h.index('Metric Unit')
scale = {'nsecond': 1e-3, 'usecond': 1.0, 'msecond': 1e3, 'second': 1e6, 'ns': 1e-3, 'us': 1.0, 'ms': 1e3, 's': 1e6}
agg = collections.defaultdict(list)
for r in data:
    if r[mi] == 'gpu__time_duration.sum':
        agg[r[ki].split('(')[0][:48]].append(float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0))
tot = sum(sum(v) for v in agg.values())
print(f"{'kernel':48s} {'launches':>8s} {'mean_us':>9s} {'total_us':>10s} {'share':>6s}")
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{k:48s} {len(v):8d} {sum(v)/len(v):9.2f} {sum(v):10.1f} {sum(v)/tot:6.3f}")
