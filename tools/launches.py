"""Summarise an ncu --metrics gpu__time_duration.sum CSV launch list per kernel."""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    k = d["Kernel Name"].split("(")[0][-40:]
    agg.setdefault(k, []).append(float(d["Metric Value"]))
total = sum(sum(v) for k, v in agg.items() if "at::" not in k)
for k, v in agg.items():
    share = "" if "at::" in k else f" share={sum(v) / total:6.1%}"
    print(f"{k:42s} n={len(v):3d} mean={sum(v) / len(v) / 1e3:9.1f}us{share}")
