"""Per-instruction stall attribution from an ncu source-page CSV:
python tools/stalls.py <src.csv> [reason] [top]"""
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
h = rows[1]
reason = sys.argv[2] if len(sys.argv) > 2 else "stall_short_sb"
top = int(sys.argv[3]) if len(sys.argv) > 3 else 15
si, ie, ri = h.index("Source"), h.index("Instructions Executed"), h.index(reason)
data = [r for r in rows[2:] if len(r) == len(h) and r[ie].isdigit()]
tot = sum(int(r[ri] or 0) for r in data)
print(reason, "total", tot)
idx = sorted(range(len(data)), key=lambda i: -int(data[i][ri] or 0))[:top]
for i in sorted(idx):
    print(i, data[i][ie], data[i][ri], data[i][si][:80])
    for j in range(max(0, i - 3), i):
        print("      ", j, data[j][si][:70])
