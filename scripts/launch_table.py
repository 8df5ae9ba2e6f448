"""Summarise an ncu --csv launch list (gpu__time_duration.sum): per-launch table
and per-kernel totals.  usage: launch_table.py launches.csv [--skip-prefix at::]"""
import csv, sys
from collections import OrderedDict, defaultdict
rows = list(csv.reader(open(sys.argv[1])))
hdr = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
h = rows[hdr]
ki, mi, vi, ii, gi = (h.index(x) for x in ("Kernel Name", "Metric Name", "Metric Value", "ID", "Grid Size"))
L = OrderedDict()
for r in rows[hdr + 1:]:
    L.setdefault(r[ii], {"k": r[ki], "g": r[gi]})[r[mi]] = r[vi]
tot = 0.0
agg = defaultdict(lambda: [0, 0.0])
verbose = "-v" in sys.argv
for k, v in L.items():
    if v["k"].startswith("void at::") or v["k"].startswith("at::") or "cutlass" in v["k"]:
        continue
    t = float(v["gpu__time_duration.sum"].replace(",", "")) / 1000.0
    tot += t
    name = v["k"].split("(")[0].replace("void ", "").replace("<unnamed>::", "")
    agg[name][0] += 1
    agg[name][1] += t
    if verbose:
        print(f"{k:>5} {name[:45]:45} {v['g']:>16} {t:9.1f}")
for name, (n, t) in sorted(agg.items(), key=lambda x: -x[1][1]):
    print(f"{n:5d} x {name[:60]:60} {t:10.1f} us  {100*t/tot:5.1f}%")
print(f"total {tot:.1f} us")
