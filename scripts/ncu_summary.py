"""Summarise an ncu report: SOL, occupancy, stall reasons, DRAM bytes."""
import csv
import io
import subprocess
import sys

rep = sys.argv[1]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
for vals in rows[2:]:
    d = dict(zip(hdr, vals))
    u = dict(zip(hdr, units))
    print("kernel:", d.get("Kernel Name", "")[:80])
    keys = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
            "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__throughput.avg.pct_of_peak_sustained_elapsed",
            "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
            "smsp__issue_active.avg.pct_of_peak_sustained_active",
            "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
            "l1tex__t_sector_hit_rate.pct", "sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active"]
    for k in keys:
        if k in d:
            print(f"  {k} = {d[k]} {u.get(k, '')}")
    st = {k: v for k, v in d.items() if "average_warps_issue_stalled" in k and "per_issue_active" in k}
    top = sorted(st.items(), key=lambda kv: -float(kv[1].replace(",", "") or 0))[:8]
    for k, v in top:
        print(f"  stall {k.split('stalled_')[1].split('_per')[0]} = {v}")
