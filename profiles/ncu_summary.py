"""Summarise an ncu report: time, DRAM bytes, occupancy, issue activity, top stalls."""
import csv
import subprocess
import sys

rep = sys.argv[1]
out = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
want = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "smsp__inst_executed.sum",
        "l1tex__t_sector_hit_rate.pct", "lts__t_sector_hit_rate.pct",
        "dram__throughput.avg.pct_of_peak_sustained_elapsed", "launch__grid_size"]
for r in rows[2:]:
    d = {w: r[h.index(w)] for w in want if w in h}
    print(" | ".join(f"{k.split('__')[-1] if '__' in k else k}={v[:14]}" for k, v in d.items()))
    st = [(k, float(r[h.index(k)] or 0)) for k in h
          if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("_per_issue_active.ratio")]
    st.sort(key=lambda x: -x[1])
    print("   stalls/issue:", ", ".join(f"{a[len('smsp__average_warps_issue_stalled_'):-len('_per_issue_active.ratio')]}={b:.2f}"
                                        for a, b in st[:6]))
