"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv) per kernel."""
import csv
import sys
from collections import defaultdict

rows = [r for r in csv.reader(open(sys.argv[1])) if r]
start = next(i for i, r in enumerate(rows) if r[0] == "ID")
h = rows[start]
iname, ival, iunit = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
scale = {"ns": 1e-9, "nsecond": 1e-9, "us": 1e-6, "usecond": 1e-6, "ms": 1e-3, "msecond": 1e-3, "s": 1.0}
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[start + 1:]:
    k = r[iname].split("(")[0]
    tot[k] += float(r[ival].replace(",", "")) * scale[r[iunit]]
    cnt[k] += 1
T = sum(tot.values())
print(f"{'kernel':32s} {'launches':>8s} {'total ms':>10s} {'mean ms':>9s} {'share':>6s}")
for k in sorted(tot, key=lambda k: -tot[k]):
    print(f"{k:32s} {cnt[k]:8d} {tot[k]*1e3:10.3f} {tot[k]*1e3/cnt[k]:9.3f} {100*tot[k]/T:5.1f}%")
print(f"{'TOTAL':32s} {sum(cnt.values()):8d} {T*1e3:10.3f}")
