"""Per-kernel roofline table (north_star: each kernel's achieved HBM GB/s and FP32 issue against the
B200 peaks, atomic traffic for the backward) from a `tools/summarize_ncu.py full` summary:
    python tools/kernel_roofline.py profiles/<tag>_full.md [out.md]"""
import json
import os
import re
import sys

src = sys.argv[1]
root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
hbm = json.load(open(os.path.join(root, "MEASURED_PEAKS.json"))).get("hbm_gbs", 6540.8)
txt = open(src).read()
lines = [f"Per-kernel ncu figures (`{os.path.basename(src)}`: one `--set full` launch each, cold-ish "
         f"cache, serialised); HBM peak {hbm:.0f} GB/s (MEASURED_PEAKS.json).  FMA pipe % = "
         "`sm__inst_executed_pipe_fma` of peak (the FP32 issue roofline); RED sectors = "
         "`lts__t_sectors_srcunit_tex_op_red` (global reductions reaching L2: the backward's "
         "fixed-point gradient atomics, the preprocess's per-tile bucket counts).", "",
         "| kernel | µs | DRAM MB | GB/s | % of HBM peak | FMA pipe % | issue active % | warps active % | RED sectors | regs/thread |",
         "|---|---|---|---|---|---|---|---|---|---|"]
for sec in re.split(r"^## ", txt, flags=re.M)[1:]:
    name = sec.split("`")[1].split("(")[0].replace("void ", "")
    d = {m.group(1): float(m.group(2).replace(",", ""))
         for m in re.finditer(r"\| (\S+) \| ([0-9.,]+) ?[A-Za-z/%]* \|", sec)}
    t = d.get("gpu__time_duration.sum", 0.0)
    mb = d.get("dram__bytes_read.sum", 0.0) + d.get("dram__bytes_write.sum", 0.0)
    gbs = mb * 1e6 / (t * 1e-6) / 1e9 if t else 0.0
    lines.append(f"| `{name}` | {t:.1f} | {mb:.0f} | {gbs:.0f} | {100 * gbs / hbm:.0f} | "
                 f"{d.get('sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active', 0):.0f} | "
                 f"{d.get('smsp__issue_active.avg.pct_of_peak_sustained_active', 0):.0f} | "
                 f"{d.get('sm__warps_active.avg.pct_of_peak_sustained_active', 0):.0f} | "
                 f"{int(d.get('lts__t_sectors_srcunit_tex_op_red.sum', 0)):,} | "
                 f"{int(d.get('launch__registers_per_thread', 0))} |")
out = "\n".join(lines) + "\n"
if len(sys.argv) > 2:
    open(sys.argv[2], "w").write(out)
print(out)
