"""profiles/traffic.json: ncu DRAM bytes (read + write) per iteration of each bench phase, from a
warm graph-replay metric list (tools/gpu_quick2.sh):  python tools/traffic.py <graph.csv> [iters]"""
import collections
import csv
import json
import os
import sys

PHASE = {"preprocess": ("preprocess_kernel", "big_bands", "big_exact", "big_cull"),
         "bin": ("huge_sort", "huge_transpose", "tile_scan", "bucket_fill", "tile_sort_merge"),
         "render_fwd": ("render_fwd", "lazy_fill", "tile_finish"),
         "loss": ("loss_tables", "ssim_fwd", "ssim_bwd", "depth_loss", "loss_finalize"),
         "render_bwd": ("zero_g2d", "render_bwd"),
         "chain_adam": ("chain_kernel", "adam_list")}
rows = list(csv.reader(open(sys.argv[1])))
iters = int(sys.argv[2]) if len(sys.argv) > 2 else 8
hdr, acc = None, collections.Counter()
for r in rows:
    if r and r[0] == "ID":
        hdr = r
        continue
    if hdr and len(r) == len(hdr):
        d = dict(zip(hdr, r))
        if d["Metric Name"] not in ("dram__bytes_read.sum", "dram__bytes_write.sum"):
            continue
        for ph, ks in PHASE.items():
            if any(k in d["Kernel Name"] for k in ks):
                acc[ph] += float(d["Metric Value"].replace(",", ""))
out = {ph: int(v / iters) for ph, v in acc.items()}
out["_source"] = os.path.basename(sys.argv[1]) + f": ncu --cache-control none warm graph replay, {iters} iterations"
path = os.path.join(os.path.dirname(os.path.dirname(os.path.abspath(__file__))), "profiles", "traffic.json")
json.dump(out, open(path, "w"), indent=1)
print(out)
