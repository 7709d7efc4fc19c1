"""Top source lines / SASS instructions by stall samples from an .ncu-rep source page.
usage: ncu_hot.py REP [cuda|sass] [N] [KERNEL_REGEX]"""
import csv
import subprocess
import sys

rep, view = sys.argv[1], (sys.argv[2] if len(sys.argv) > 2 else "cuda")
n = int(sys.argv[3]) if len(sys.argv) > 3 else 25
kfilter = ["-k", "regex:" + sys.argv[4]] if len(sys.argv) > 4 else []
out = subprocess.run(["ncu", "-i", rep] + kfilter + ["--page", "source", "--csv", "--print-source",
                      "cuda,sass" if view == "cuda" else view],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr, data, fname = None, [], ""
for r in rows:
    if len(r) >= 2 and r[0] in ("File Path", "File Name"):
        fname = r[1].split("/")[-1]
        continue
    if r and r[0] in ("Line No", "Address"):
        hdr = [h if h != "Source" or i == r.index("Source") else "SASS" for i, h in enumerate(r)]
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        d["_file"] = fname
        if view == "cuda" and not d.get("Line No"):
            continue  # per-instruction rows under a source line
        data.append(d)
key = "Warp Stall Sampling (All Samples)"
tot = sum(float(d.get(key) or 0) for d in data)
data.sort(key=lambda d: -float(d.get(key) or 0))
stall_cols = [h for h in (hdr or []) if h.startswith("stall_")]
for d in data[:n]:
    s = float(d.get(key) or 0)
    top = sorted(((c[6:], float(d.get(c) or 0)) for c in stall_cols), key=lambda kv: -kv[1])[:3]
    loc = d.get("Line No") or d.get("Address")
    src = d.get("Source", "")[:90]
    print(f"{s / tot:6.1%} {d['_file']}:{loc:>6} exec={d.get('Instructions Executed', '')} "
          f"[{', '.join(f'{k}={int(v)}' for k, v in top if v)}] {src}")
