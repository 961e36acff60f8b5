"""Summarise an ncu report into profiles/: key metrics per kernel (json + text).

    python profiles/summarize_ncu.py gpurun_out/prof_r1.ncu-rep profiles/r1_ncu_full
"""
import csv
import io
import json
import subprocess
import sys

KEYS = ["Kernel Name", "gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "launch__shared_mem_per_block_dynamic", "smsp__issue_active.avg.pct_of_peak_sustained_active",
        "smsp__warps_eligible.avg.per_cycle_active", "smsp__inst_executed.sum", "lts__t_sector_hit_rate.pct",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum",
        "smsp__average_warps_issue_stalled_long_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_short_scoreboard_per_issue_active.ratio",
        "smsp__average_warps_issue_stalled_wait_per_issue_active.ratio"]
SCALE = {"Kbyte": 1e3, "Mbyte": 1e6, "Gbyte": 1e9, "byte": 1.0, "usecond": 1e-3, "msecond": 1.0, "ms": 1.0,
         "us": 1e-3, "nsecond": 1e-6}

rep, out = sys.argv[1], sys.argv[2]
raw = subprocess.run(["ncu", "-i", rep, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
hdr, units = rows[0], rows[1]
kernels = []
for r in rows[2:]:
    d = {}
    for k in KEYS:
        if k in hdr:
            i = hdr.index(k)
            d[k] = r[i] + (f" {units[i]}" if units[i] else "")
    rd, wr = hdr.index("dram__bytes_read.sum"), hdr.index("dram__bytes_write.sum")
    d["dram_bytes_per_launch"] = (float(r[rd].replace(",", "")) * SCALE.get(units[rd], 1.0)
                                  + float(r[wr].replace(",", "")) * SCALE.get(units[wr], 1.0))
    tm = hdr.index("gpu__time_duration.sum")
    d["time_ms"] = float(r[tm].replace(",", "")) * SCALE.get(units[tm], 1.0)
    kernels.append(d)
json.dump(kernels, open(out + ".json", "w"), indent=1)
with open(out + ".txt", "w") as fh:
    for d in kernels:
        for k, v in d.items():
            fh.write(f"{k} = {v}\n")
        fh.write("\n")
print(open(out + ".txt").read())
