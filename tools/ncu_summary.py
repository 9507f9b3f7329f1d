"""Summarise an ncu --set full report (read here, no GPU): key counters of every kernel."""
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__occupancy_limit_shared_mem", "launch__occupancy_limit_registers",
        "sm__inst_executed.avg.per_cycle_active", "inst_executed", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "dram__throughput.avg.pct_of_peak_sustained_elapsed",
        "launch__grid_size", "launch__block_size", "sm__cycles_elapsed.avg"]
STALL = "smsp__average_warps_issue_stalled_"


def main(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        print("kernel:", d.get("Kernel Name"))
        for k in KEYS:
            if k in d:
                print(f"  {k} = {d[k]} {u.get(k, '')}")
        st = sorted(((float(d[k]), k[len(STALL):]) for k in hdr if k.startswith(STALL) and k.endswith("per_issue_active.ratio")
                     and d[k] not in ("", "n/a")), reverse=True)[:8]
        print("  stalls/issue:", ", ".join(f"{n.replace('_per_issue_active.ratio','')}={v:.2f}" for v, n in st))


if __name__ == "__main__":
    main(sys.argv[1])
