"""Parse an ncu launch list (gpu__time_duration.sum CSV) into per-step
kernel-time tables: a step starts at each launch of --first (default k_zero
following k_set_opt / the first k_zero of a step)."""
import csv
import sys
from collections import OrderedDict


def main(path, first="k_sample"):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr, start = r, i + 1
            break
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    steps, cur = [], None
    for r in rows[start:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("void ", "").replace("tagc_b200::", "").replace("<unnamed>::", "")
        t = float(r[vi].replace(",", "")) / 1000.0
        if name.startswith(first):
            cur = OrderedDict()
            steps.append(cur)
        if cur is not None:
            cur[name] = cur.get(name, 0.0) + t
    names = []
    for s in steps:
        for n in s:
            if n not in names:
                names.append(n)
    print("kernel".ljust(28) + "".join(f"{i:>8d}" for i in range(len(steps))))
    for n in names:
        print(n[:27].ljust(28) + "".join(f"{s.get(n, 0.0):8.1f}" for s in steps))
    print("total".ljust(28) + "".join(f"{sum(s.values()):8.1f}" for s in steps))


if __name__ == "__main__":
    main(*sys.argv[1:])
