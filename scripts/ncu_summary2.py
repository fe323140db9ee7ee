"""Key metrics of every kernel in an ncu report (ncu -i ... --page raw --csv)."""
import csv
import subprocess
import sys

WANT = ['Kernel Name', 'gpu__time_duration.sum', 'dram__bytes_read.sum', 'dram__bytes_write.sum',
        'gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__throughput.avg.pct_of_peak_sustained_elapsed',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'launch__registers_per_thread',
        'launch__occupancy_limit_shared_mem', 'launch__occupancy_limit_registers',
        'smsp__issue_active.avg.pct_of_peak_sustained_active', 'launch__grid_size',
        'sm__warps_active.avg.per_cycle_active', 'l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum',
        'smsp__average_warp_latency_issue_stalled_barrier', 'lts__t_sector_hit_rate.pct']


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    hdr, units = rows[0], rows[1]
    stall = [i for i, h in enumerate(hdr)
             if h.startswith("smsp__average_warp_latency_issue_stalled_") and h.endswith("_ratio") is False
             and "pct" not in h]
    for r in rows[2:]:
        print("---")
        for w in WANT:
            if w in hdr:
                i = hdr.index(w)
                print(f"  {w}: {r[i]} {units[i]}")
        st = sorted(((float(r[i].replace(',', '')) if r[i] else 0.0, hdr[i]) for i in stall
                     if r[i] not in ("", "n/a")), reverse=True)[:8]
        for v, h in st:
            print(f"  stall {h.replace('smsp__average_warp_latency_issue_stalled_', '')}: {v:.2f}")


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("#", p)
        main(p)
