"""Aggregate an ncu --csv launch list (gpu__time_duration.sum) by kernel name."""
import csv, sys, collections
rows = list(csv.reader(open(sys.argv[1])))
hdr_i = next(i for i, r in enumerate(rows) if 'Kernel Name' in r)
hdr = rows[hdr_i]
ki, mi, vi = hdr.index('Kernel Name'), hdr.index('Metric Name'), hdr.index('Metric Value')
agg = collections.defaultdict(lambda: [0, 0.0])
for r in rows[hdr_i + 1:]:
    if len(r) <= vi or r[mi] != 'gpu__time_duration.sum':
        continue
    name = r[ki].replace('void ', '').replace('(anonymous namespace)::', '').replace('<unnamed>::', '')
    name = name.replace('hc::', '').split('(')[0]
    v = float(r[vi].replace(',', ''))
    agg[name][0] += 1
    agg[name][1] += v
unit = rows[hdr_i + 1][hdr.index('Metric Unit')] if 'Metric Unit' in hdr else ''
tot = sum(v for _, v in agg.values())
print(f'total {tot:.1f} {unit} over {sum(n for n, _ in agg.values())} launches')
for name, (n, v) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
    print(f'{v / tot * 100:6.2f}%  {v:12.1f} {unit}  {n:6d} x  avg {v / n:9.2f}  {name}')
