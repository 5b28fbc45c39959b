"""Per-source-line totals from `ncu -i R --page source --csv --print-source cuda,sass`:
python tools/srclines.py <cs.csv> [top]  -> lines sorted by warp-instructions executed,
with stall samples."""
import csv
import sys

top = int(sys.argv[2]) if len(sys.argv) > 2 else 40
fname = None
agg = {}
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if len(r) >= 2 and r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 9 or not r[0].isdigit():
        continue
    if r[2] != "-":  # sass row under a line
        continue
    key = (fname, int(r[0]))
    ie = int(r[7] or 0)
    smp = int(r[4] or 0)
    a = agg.setdefault(key, [0, 0, r[1][:90]])
    a[0] += ie
    a[1] += smp
tot_i = sum(v[0] for v in agg.values()) or 1
tot_s = sum(v[1] for v in agg.values()) or 1
print(f"total warp-inst {tot_i}, samples {tot_s}")
for k, v in sorted(agg.items(), key=lambda kv: -kv[1][0])[:top]:
    print(f"{k[0]:18s}:{k[1]:5d} inst {100*v[0]/tot_i:5.1f}% stall {100*v[1]/tot_s:5.1f}%  {v[2]}")
