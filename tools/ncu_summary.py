"""Summarise an ncu --set full report: the metrics DESIGN.md and bench.py cite, per kernel
(mean over captured launches). Usage: python tools/ncu_summary.py report.ncu-rep > summary.txt"""
import csv
import subprocess
import sys
from collections import defaultdict

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__pipe_tensor_cycles_active.avg.pct_of_peak_sustained_active",
        "sm__warps_active.avg.pct_of_peak_sustained_active", "launch__registers_per_thread",
        "launch__grid_size", "launch__block_size", "smsp__inst_executed.sum",
        "l1tex__data_pipe_lsu_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "l1tex__data_pipe_tc_wavefronts_mem_shared.sum.pct_of_peak_sustained_elapsed",
        "lts__t_bytes.sum", "sm__cycles_elapsed.avg.per_second"]

out = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(out.splitlines()))
h = rows[0]
ki = h.index("Kernel Name")
units = rows[1]
agg = defaultdict(lambda: defaultdict(list))
for r in rows[2:]:
    name = r[ki].split("(")[0]
    for k in KEYS:
        if k in h:
            try:
                agg[name][k].append(float(r[h.index(k)].replace(",", "")))
            except ValueError:
                pass
for name, m in agg.items():
    print(f"== {name} (mean over {max(len(v) for v in m.values())} launches; ncu --set full, --clock-control none)")
    for k in KEYS:
        if k in m and m[k]:
            print(f"  {k:90s} {sum(m[k]) / len(m[k]):16.4f} {units[h.index(k)]}")
