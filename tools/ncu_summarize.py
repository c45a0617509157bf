"""Summarise ncu reports into profiles/ (run in the build container).

    python tools/ncu_summarize.py <tag> gpurun_out/prof_*_<tag>.ncu-rep ...
"""
import csv
import json
import subprocess
import sys
from io import StringIO

WANT = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__occupancy_limit_registers", "launch__occupancy_limit_shared_mem",
        "launch__grid_size", "launch__block_size", "launch__shared_mem_per_block_dynamic",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_fp64.avg.pct_of_peak_sustained_active",
        "l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "smsp__inst_executed.sum",
        "sm__cycles_active.avg", "gpc__cycles_elapsed.max", "lts__t_bytes.sum",
        "sm__cycles_elapsed.avg.per_second",
        "TPC.TriageCompute.sm__pipe_tensor_cycles_active_realtime.avg.pct_of_peak_sustained_elapsed",
        "l1tex__throughput.avg.pct_of_peak_sustained_elapsed",
        "lts__throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_xu.avg.pct_of_peak_sustained_active"]


def summarize(path):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True,
                         text=True).stdout
    rows = list(csv.reader(StringIO(raw)))
    h, units = rows[0], rows[1]
    out = []
    for r in rows[2:]:
        d = {"kernel": r[h.index("Kernel Name")].split("(")[0]}
        for w in WANT:
            if w in h:
                d[w] = f"{r[h.index(w)]} {units[h.index(w)]}".strip()
        out.append(d)
    return out


if __name__ == "__main__":
    tag = sys.argv[1]
    res = {p: summarize(p) for p in sys.argv[2:]}
    json.dump(res, open(f"profiles/{tag}_ncu_kernels.json", "w"), indent=1)
    for p, ks in res.items():
        for d in ks:
            print(d["kernel"], "|", d.get("gpu__time_duration.sum"), "| dram",
                  d.get("dram__bytes_read.sum"), "+", d.get("dram__bytes_write.sum"), "|",
                  d.get("gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed"), "| fp64",
                  d.get("sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active"),
                  "| regs", d.get("launch__registers_per_thread"))
