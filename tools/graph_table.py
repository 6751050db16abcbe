"""Per-kernel table of a warm graph-replay ncu metric list: python tools/graph_table.py <csv> [iters] [out.md]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 8
hdr, data = None, []
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        data.append(dict(zip(hdr, r)))
agg = collections.OrderedDict()
for d in data:
    nm = d["Kernel Name"].split("(")[0].replace("void ", "")
    a = agg.setdefault(nm, collections.defaultdict(float))
    a[d["Metric Name"]] += float(d["Metric Value"].replace(",", ""))
    if d["Metric Name"] == "gpu__time_duration.sum":
        a["n"] += 1
tot = sum(a["gpu__time_duration.sum"] for a in agg.values())
lines = [f"Warm-cache graph replay (`ncu --cache-control none --clock-control none`), {iters} iterations; "
         f"per-iteration kernel time {tot / iters / 1e3:.1f} us (serialised by the profiler).", "",
         "| kernel | launches/iter | us / launch | DRAM rd MB | DRAM wr MB | GB/s | warp instr (M) | issue active % | warps active % | share |",
         "|---|---|---|---|---|---|---|---|---|---|"]
for k, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    n = a["n"]
    us = a["gpu__time_duration.sum"] / n / 1e3
    rd, wr = a["dram__bytes_read.sum"] / n / 1e6, a["dram__bytes_write.sum"] / n / 1e6
    ins = a.get("smsp__inst_executed.sum", 0.0) / n / 1e6
    iss = a.get("smsp__issue_active.avg.pct_of_peak_sustained_active", 0.0) / n
    wa = a.get("sm__warps_active.avg.pct_of_peak_sustained_active", 0.0) / n
    lines.append(f"| `{k}` | {n / iters:g} | {us:.1f} | {rd:.1f} | {wr:.1f} | {(rd + wr) / us * 1e3:.0f} | {ins:.1f} | "
                 f"{iss:.0f} | {wa:.0f} | {a['gpu__time_duration.sum'] / tot:.3f} |")
out = "\n".join(lines)
print(out)
if len(sys.argv) > 3:
    open(sys.argv[3], "w").write(out + "\n")
