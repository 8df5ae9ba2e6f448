"""Print the last N launches of an ncu launch-list CSV (duration ns, grid size)."""
import csv, sys
from collections import OrderedDict
rows = list(csv.reader(open(sys.argv[1])))
n = int(sys.argv[2]) if len(sys.argv) > 2 else 40
hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r); h = rows[hi]
ki, vi, mi, idi = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Name"), h.index("ID")
L = OrderedDict()
for r in rows[hi + 1:]:
    if len(r) <= vi:
        continue
    L.setdefault(r[idi], {})['k'] = r[ki].split('(')[0].replace('<unnamed>::', '')
    L[r[idi]][r[mi]] = r[vi]
items = list(L.values())[-n:]
tot = 0
for it in items:
    d = float(it.get('gpu__time_duration.sum', '0').replace(',', ''))
    tot += d
    print(f"{it['k'][:34]:34s} {d/1000:8.2f} us  grid {it.get('launch__grid_size', '')}")
print(f"total {tot/1000:.1f} us over {len(items)} launches")
