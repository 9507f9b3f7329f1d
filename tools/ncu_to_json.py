"""Condense an ncu --set full report into a small JSON summary for profiles/ (run here, no GPU).

    python tools/ncu_to_json.py gpurun_out/X/prof.ncu-rep profiles/NAME.json [--algorithmic-bytes B]
"""
import argparse
import csv
import io
import json
import subprocess

KEYS = {"gpu__time_duration.sum": "duration", "dram__bytes_read.sum": "dram_read", "dram__bytes_write.sum": "dram_write",
        "sm__warps_active.avg.pct_of_peak_sustained_active": "warps_active_pct",
        "sm__inst_executed.avg.per_cycle_active": "sm_ipc", "inst_executed": "inst_executed",
        "launch__registers_per_thread": "registers", "launch__grid_size": "grid", "launch__block_size": "block",
        "launch__shared_mem_per_block_dynamic": "smem_dynamic", "launch__occupancy_limit_shared_mem": "occ_limit_smem",
        "lts__t_sector_hit_rate.pct": "l2_hit_pct", "dram__throughput.avg.pct_of_peak_sustained_elapsed": "dram_pct_of_peak",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum": "smem_bank_conflicts", "sm__cycles_elapsed.avg": "sm_cycles"}
SCALE = {"Gbyte": 1e9, "Mbyte": 1e6, "Kbyte": 1e3, "byte": 1, "ms": 1e-3, "us": 1e-6, "usecond": 1e-6, "msecond": 1e-3,
         "ns": 1e-9, "nsecond": 1e-9, "s": 1.0}


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("rep")
    ap.add_argument("out")
    ap.add_argument("--algorithmic-bytes", type=float, default=None)
    ap.add_argument("--note", default="")
    a = ap.parse_args()
    raw = subprocess.run(["ncu", "-i", a.rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d, u = dict(zip(hdr, r)), dict(zip(hdr, units))
        e = {"kernel": d.get("Kernel Name")}
        for k, nm in KEYS.items():
            if k in d and d[k] not in ("", "n/a"):
                v = float(d[k].replace(",", ""))
                unit = u.get(k, "")
                if unit in SCALE:
                    v *= SCALE[unit]
                    nm = nm + ("_bytes" if "byte" in unit else "_s")
                e[nm] = v
        if "dram_read_bytes" in e and "dram_write_bytes" in e:
            e["traffic_bytes"] = e["dram_read_bytes"] + e["dram_write_bytes"]
            if "duration_s" in e:
                e["dram_GBps"] = e["traffic_bytes"] / e["duration_s"] / 1e9
        stalls = {k.split("stalled_")[1].replace("_per_issue_active.ratio", ""): float(d[k]) for k in hdr
                  if k.startswith("smsp__average_warps_issue_stalled_") and k.endswith("per_issue_active.ratio")
                  and d[k] not in ("", "n/a")}
        e["top_stalls_per_issue"] = dict(sorted(stalls.items(), key=lambda kv: -kv[1])[:6])
        if a.algorithmic_bytes:
            e["algorithmic_bytes"] = a.algorithmic_bytes
            e["traffic_over_algorithmic"] = e.get("traffic_bytes", 0) / a.algorithmic_bytes
        out.append(e)
    res = {"source": a.rep, "note": a.note, "kernels": out}
    if len(out) == 1 and "traffic_bytes" in out[0]:
        res["bytes_per_launch"] = out[0]["traffic_bytes"]
    with open(a.out, "w") as f:
        json.dump(res, f, indent=1)
    print(json.dumps(res, indent=1)[:2000])


if __name__ == "__main__":
    main()
