"""Summarise ncu outputs: a launch-list CSV (gpu__time_duration per kernel) and/or a
--set full report (DRAM bytes, throughput %, registers) -> JSON/markdown under profiles/."""
import collections
import csv
import json
import re
import subprocess
import sys


def _name(s):
    s = s.replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
    m = re.match(r"(?:void\s+)?([A-Za-z_][\w:]*)", s)
    return m.group(1) if m else s


def launches(path):
    rows = list(csv.reader(open(path)))
    hi = next(i for i, r in enumerate(rows) if "Kernel Name" in r)
    h = rows[hi]
    ki, vi, ui = h.index("Kernel Name"), h.index("Metric Value"), h.index("Metric Unit")
    mi = h.index("Metric Name") if "Metric Name" in h else None
    agg = collections.OrderedDict()
    for r in rows[hi + 1:]:
        if len(r) <= vi or (mi is not None and r[mi] != "gpu__time_duration.sum"):
            continue
        v = float(r[vi].replace(",", ""))
        scale = {"nsecond": 1e-3, "ns": 1e-3, "usecond": 1.0, "us": 1.0, "msecond": 1e3,
                 "ms": 1e3, "second": 1e6, "s": 1e6}.get(r[ui], 1.0)
        c, t = agg.get(_name(r[ki]), (0, 0.0))
        agg[_name(r[ki])] = (c + 1, t + v * scale)
    tot = sum(t for _, t in agg.values())
    out = [dict(kernel=n, launches=c, total_us=round(t, 2), share=round(t / tot, 4))
           for n, (c, t) in sorted(agg.items(), key=lambda kv: -kv[1][1])]
    return dict(total_us=round(tot, 2), kernels=out)


WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed", "launch__registers_per_thread",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__grid_size",
        "launch__block_size", "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "smsp__inst_executed_pipe_fp64.sum"]


def full(path):
    txt = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(txt.splitlines()))
    h, units = rows[0], rows[1]
    res = []
    for v in rows[2:]:
        d = {"kernel": _name(v[h.index("Kernel Name")])}
        for i, n in enumerate(h):
            if n in WANT or "dmma" in n.lower() or ("tensor" in n.lower() and "pct" in n.lower()
                                                     and "fp64" in n.lower()):
                d[n] = f"{v[i]} {units[i]}".strip()
        res.append(d)
    return res


if __name__ == "__main__":
    kind, path, outp = sys.argv[1], sys.argv[2], sys.argv[3]
    data = launches(path) if kind == "launches" else full(path)
    json.dump(data, open(outp, "w"), indent=1)
    if kind == "launches":
        print(f"total {data['total_us'] / 1e3:.2f} ms")
        for k in data["kernels"][:20]:
            print(f"  {k['kernel']:34s} {k['launches']:5d} {k['total_us'] / 1e3:9.3f} ms {100 * k['share']:5.1f}%")
    else:
        print(json.dumps(data, indent=1))
