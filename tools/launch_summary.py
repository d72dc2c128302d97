"""Summarise an ncu launch list (--metrics gpu__time_duration.sum --csv).

usage: python tools/launch_summary.py launches.csv [first_id last_id]

Per-kernel launch counts, total serialised time and share. With an ID range
only the launches of that window are counted (e.g. the one timed bench step).
"""
import csv
import sys
from collections import defaultdict

path = sys.argv[1]
lo = int(sys.argv[2]) if len(sys.argv) > 2 else None
hi = int(sys.argv[3]) if len(sys.argv) > 3 else None
rows = [r for r in csv.reader(l for l in open(path) if l.startswith('"'))]
hdr = rows[0]
iid, iname, ival = hdr.index("ID"), hdr.index("Kernel Name"), hdr.index("Metric Value")
imet = hdr.index("Metric Name") if "Metric Name" in hdr else None
tot, cnt = defaultdict(float), defaultdict(int)
for r in rows[1:]:
    if imet is not None and r[imet] != "gpu__time_duration.sum":
        continue
    i = int(r[iid])
    if lo is not None and not (lo <= i <= hi):
        continue
    name = r[iname].split("(")[0]
    tot[name] += float(r[ival].replace(",", "")) / 1e6  # ns -> ms
    cnt[name] += 1
all_ms = sum(tot.values())
print(f"{'kernel':60s} {'n':>6s} {'total ms':>10s} {'share':>7s}")
for k, v in sorted(tot.items(), key=lambda kv: -kv[1]):
    print(f"{k[:60]:60s} {cnt[k]:6d} {v:10.3f} {100 * v / all_ms:6.1f}%")
print(f"{'all':60s} {sum(cnt.values()):6d} {all_ms:10.3f}")
