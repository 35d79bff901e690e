"""Summarise an ncu launch-list CSV (gpu__time_duration.sum) by kernel."""
import csv, collections, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
h = rows[hdr_i]
ki, vi, ui = h.index('Kernel Name'), h.index('Metric Value'), h.index('Metric Unit')
tot, cnt = collections.OrderedDict(), collections.Counter()
scale = {'nsecond': 1e-3, 'usecond': 1.0, 'msecond': 1e3, 'ns': 1e-3, 'us': 1.0, 'ms': 1e3}
n = 0
for r in rows[hdr_i + 1:]:
    if len(r) <= vi:
        continue
    us = float(r[vi].replace(',', '')) * scale.get(r[ui], 1e-3)
    name = r[ki].split('(')[0][:70]
    tot[name] = tot.get(name, 0.0) + us
    cnt[name] += 1
    n += 1
print(f"{n} launches, {sum(tot.values()) / 1e3:.2f} ms total")
for k, v in sorted(tot.items(), key=lambda x: -x[1])[:int(sys.argv[2]) if len(sys.argv) > 2 else 25]:
    print(f"{v / 1e3:9.3f} ms  {cnt[k]:5d}  {k}")
