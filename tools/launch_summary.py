"""Summarise an ncu --csv launch list (gpu__time_duration.sum) by kernel."""
import collections, csv, sys
rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if 'Kernel Name' in r:
        hdr = r; continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.defaultdict(lambda: [0, 0.0])
scale = {'nsecond': 1.0, 'usecond': 1e3, 'msecond': 1e6, 'second': 1e9}
for d in data:
    if d.get('Metric Name') != 'gpu__time_duration.sum':
        continue
    name = d['Kernel Name'].split('(')[0][:70]
    v = float(d['Metric Value'].replace(',', '')) * scale.get(d['Metric Unit'], 1.0)
    agg[name][0] += 1
    agg[name][1] += v
tot = sum(v[1] for v in agg.values())
n = sum(v[0] for v in agg.values())
print(f"{n} launches, {tot/1e6:.3f} ms total GPU time (serialised, cold-cache)")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][1])[:25]:
    print(f"{v[1]/1e6:9.3f} ms {100*v[1]/tot:5.1f}% {v[0]:6d} launches {v[1]/v[0]/1e3:8.1f} us/launch  {k}")
