"""Extract the key metrics of every kernel result in an ncu report into JSON (profiles/ summaries).
    python ncu_extract.py report.ncu-rep [label] > out.json"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "smsp__inst_executed.sum",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active", "lts__t_sector_hit_rate.pct",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem", "sm__throughput.avg.pct_of_peak_sustained_elapsed"]
STALL = "smsp__average_warps_issue_stalled_"


def main():
    rep = sys.argv[1]
    raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    hdr, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = dict(zip(hdr, r))
        u = dict(zip(hdr, units))
        rec = {"kernel": d.get("Kernel Name", "")[:60], "id": d.get("ID")}
        for k in KEYS:
            if k in d:
                rec[k] = f"{d[k]} {u.get(k, '')}".strip()
        stalls = {k[len(STALL):].replace("_per_issue_active.ratio", ""): d[k] for k in hdr
                  if k.startswith(STALL) and k.endswith("_per_issue_active.ratio") and d.get(k)}
        rec["stalls_per_issue"] = stalls
        out.append(rec)
    print(json.dumps({"report": rep, "label": sys.argv[2] if len(sys.argv) > 2 else "", "results": out}, indent=1))


if __name__ == "__main__":
    main()
