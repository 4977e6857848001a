"""Kernel shares of an ncu launch list (--metrics gpu__time_duration.sum CSV)."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hi = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hi]
ki, mi, vi, ui = h.index('Kernel Name'), h.index('Metric Name'), h.index('Metric Value'), h.index('Metric Unit')
scale = {'ns': 1e-6, 'nsecond': 1e-6, 'us': 1e-3, 'usecond': 1e-3, 'ms': 1.0, 'msecond': 1.0}
tot, cnt = collections.defaultdict(float), collections.Counter()
for r in rows[hi + 1:]:
    if r[mi] != 'gpu__time_duration.sum':
        continue
    name = r[ki].replace('<unnamed>::', '').split('(')[0][:40]
    tot[name] += float(r[vi].replace(',', '')) * scale.get(r[ui], 1.0)
    cnt[name] += 1
s = sum(tot.values())
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k:44s} {cnt[k]:6d} {v:10.2f} {100 * v / s:5.1f}%")
print(f"total {s:.1f} ms")
