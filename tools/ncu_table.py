"""Key metrics of every launch in an ncu report: python tools/ncu_table.py <rep>"""
import csv
import io
import subprocess
import sys

raw = subprocess.run(["ncu", "-i", sys.argv[1], "--page", "raw", "--csv"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(raw)))
h = rows[0]
keys = [("Kernel Name", "kernel"), ("gpu__time_duration.sum", "us"), ("dram__bytes_read.sum", "rdMB"),
        ("dram__bytes_write.sum", "wrMB"), ("smsp__inst_executed.sum", "winst"),
        ("smsp__issue_active.avg.pct_of_peak_sustained_active", "issue%"),
        ("sm__warps_active.avg.pct_of_peak_sustained_active", "occ%"),
        ("gpu__compute_memory_throughput.avg.pct_of_peak_sustained_elapsed", "mem%"),
        ("l1tex__data_bank_conflicts_pipe_lsu_mem_shared.sum", "bankconf"),
        ("l1tex__data_pipe_lsu_wavefronts_mem_shared.sum", "smem_wf"),
        ("launch__registers_per_thread", "regs"), ("launch__grid_size", "grid")]
print(" | ".join(k[1] for k in keys))
for r in rows[2:]:
    d = dict(zip(h, r))
    out = []
    for k, _ in keys:
        v = d.get(k, "?")
        out.append(v[:38] if k == "Kernel Name" else v)
    print(" | ".join(out))
