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
         "| kernel | launches/iter | us / launch | DRAM rd MB | DRAM wr MB | GB/s | share |", "|---|---|---|---|---|---|---|"]
for k, a in sorted(agg.items(), key=lambda x: -x[1]["gpu__time_duration.sum"]):
    n = a["n"]
    us = a["gpu__time_duration.sum"] / n / 1e3
    rd, wr = a["dram__bytes_read.sum"] / n / 1e6, a["dram__bytes_write.sum"] / n / 1e6
    lines.append(f"| `{k}` | {n / iters:g} | {us:.1f} | {rd:.1f} | {wr:.1f} | {(rd + wr) / us * 1e3:.0f} | "
                 f"{a['gpu__time_duration.sum'] / tot:.3f} |")
out = "\n".join(lines)
print(out)
if len(sys.argv) > 3:
    open(sys.argv[3], "w").write(out + "\n")
