"""Aggregate an ncu --metrics gpu__time_duration.sum CSV launch list into a markdown table."""
import collections
import csv
import sys

agg = collections.defaultdict(lambda: [0, 0.0])
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if 'Kernel Name' in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get('Metric Name') == 'gpu__time_duration.sum':
            k = d['Kernel Name'].split('(')[0].replace('void ', '')[:70]
            agg[k][0] += 1
            agg[k][1] += float(d['Metric Value'].replace(',', '')) * (1e3 if d['Metric Unit'] == 'us' else 1)
tot = sum(v[1] for v in agg.values())
print("| kernel | launches | total us | mean us | share |\n|---|---|---|---|---|")
for k, v in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"| `{k}` | {v[0]} | {v[1]/1e3:.1f} | {v[1]/v[0]/1e3:.2f} | {100*v[1]/tot:.1f}% |")
print(f"| **total** | {sum(v[0] for v in agg.values())} | {tot/1e3:.1f} | | 100% |")
