"""Print the key counters and top stall reasons of every kernel in an .ncu-rep."""
import csv
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed"]
out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
hdr = rows[0]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    print("==", d.get("Kernel Name", "")[:90])
    for k in KEYS:
        print(f"  {k:60s} {d.get(k)}")
    st = [(k.replace("smsp__pcsamp_warps_issue_stalled_", ""), float(v or 0)) for k, v in d.items()
          if "pcsamp_warps_issue_stalled" in k and not k.endswith("not_issued")]
    st.sort(key=lambda kv: -kv[1])
    print("  stalls:", ", ".join(f"{k}={int(v)}" for k, v in st[:8]))
