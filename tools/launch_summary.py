"""Mean per-launch time by kernel from an ncu --metrics gpu__time_duration.sum --csv log."""
import collections
import csv
import sys

agg = collections.defaultdict(list)
hdr = None
for r in csv.reader(open(sys.argv[1])):
    if "Kernel Name" in r:
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d.get("Metric Name") == "gpu__time_duration.sum":
            unit = d.get("Metric Unit", "nsecond")
            v = float(d["Metric Value"].replace(",", ""))
            v *= {"nsecond": 1e-3, "usecond": 1.0, "msecond": 1e3}.get(unit, 1e-3)
            agg[d["Kernel Name"][:90]].append(v)
tot = sum(sum(v) for v in agg.values())
for k, v in sorted(agg.items(), key=lambda kv: -sum(kv[1])):
    print(f"{sum(v) / tot * 100:5.1f}%  n={len(v):4d}  mean={sum(v) / len(v):12.1f} us  {k}")
