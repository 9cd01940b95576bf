"""Print the key metrics of an ncu report (run here, no GPU needed):
    python tools/ncu_summary.py gpurun_out/prof.ncu-rep"""
import csv
import subprocess
import sys

WANT = [
    "Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
    "dram__throughput.avg.pct_of_peak_sustained_elapsed", "lts__t_sector_hit_rate.pct",
    "sm__warps_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.per_cycle_active",
    "launch__registers_per_thread", "launch__occupancy_limit_registers",
    "launch__occupancy_limit_shared_mem", "launch__grid_size", "launch__block_size",
    "sm__throughput.avg.pct_of_peak_sustained_elapsed",
    "lts__throughput.avg.pct_of_peak_sustained_elapsed",
    "l1tex__throughput.avg.pct_of_peak_sustained_active",
    "smsp__inst_executed.sum", "smsp__cycles_active.avg",
]
STALL = "smsp__average_warps_issue_stalled_"


def main(path):
    out = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(out.splitlines()))
    head, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(head, r))
        u = dict(zip(head, units))
        for w in WANT:
            if w in d:
                print(f"{w:60s} {d[w]} {u.get(w, '')}")
        stalls = [(k, float(v)) for k, v in d.items()
                  if k.startswith(STALL) and k.endswith("_per_issue_active.ratio") and v]
        stalls.sort(key=lambda kv: -kv[1])
        for k, v in stalls[:8]:
            print(f"  stall {k[len(STALL):-len('_per_issue_active.ratio')]:30s} {v:.2f}")
        print()


if __name__ == "__main__":
    for p in sys.argv[1:]:
        print("==", p)
        main(p)
