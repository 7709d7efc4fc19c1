"""Per-kernel summary of an ncu launch list (gpu__time_duration.sum CSV):
launch count, mean duration and share of the library's device time
(torch's input-generation kernels are listed without a share)."""
import csv
import sys
from collections import OrderedDict


def main(path):
    rows = list(csv.reader(open(path)))
    for i, r in enumerate(rows):
        if r and r[0] == "ID":
            hdr, start = r, i + 1
            break
    ki, vi = hdr.index("Kernel Name"), hdr.index("Metric Value")
    agg = OrderedDict()
    for r in rows[start:]:
        if len(r) <= vi:
            continue
        name = r[ki].split("(")[0].replace("(anonymous namespace)::", "").replace("<unnamed>::", "")
        t = float(r[vi].replace(",", "")) / 1000.0
        n, s = agg.get(name, (0, 0.0))
        agg[name] = (n + 1, s + t)
    ours = sum(s for k, (n, s) in agg.items() if "tagc_b200" in k)
    for k, (n, s) in agg.items():
        share = f" share={100.0 * s / ours:5.1f}%" if "tagc_b200" in k else ""
        print(f"{k[-42:]:>42s}   n={n:3d} mean={s / n:9.1f}us{share}")
    print(f"library device time {ours:.1f} us over the list")


if __name__ == "__main__":
    main(sys.argv[1])
