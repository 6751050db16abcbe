"""Summarise ncu outputs from gpurun_out/ into profiles/ (tracked).

    python tools/summarize_ncu.py launches <launches.csv> <out.md> [iterations]
    python tools/summarize_ncu.py full <prof.ncu-rep> <out.md>
"""
import collections
import csv
import io
import subprocess
import sys

KEYS = ["gpu__time_duration.sum", "dram__bytes_read.sum", "dram__bytes_write.sum",
        "gpu__dram_throughput.avg.pct_of_peak_sustained_elapsed", "sm__throughput.avg.pct_of_peak_sustained_elapsed",
        "smsp__inst_executed.sum", "sm__inst_executed_pipe_fma.avg.pct_of_peak_sustained_active",
        "sm__inst_executed_pipe_alu.avg.pct_of_peak_sustained_active",
        "sm__pipe_fp64_cycles_active.avg.pct_of_peak_sustained_active",
        "smsp__issue_active.avg.pct_of_peak_sustained_active", "sm__warps_active.avg.pct_of_peak_sustained_active",
        "launch__registers_per_thread", "launch__grid_size", "launch__block_size",
        "lts__t_sectors_srcunit_tex_op_red.sum", "lts__t_sectors_srcunit_tex_op_atom.sum",
        "l1tex__t_bytes.sum", "lts__t_bytes.sum", "smsp__average_warp_latency_issue_stalled_short_scoreboard",
        ]


def launches(path, out, iters):
    rows = list(csv.reader(open(path)))
    hdr, data = None, []
    for r in rows:
        if r and r[0] == "ID":
            hdr = r
            continue
        if hdr and len(r) == len(hdr):
            data.append(dict(zip(hdr, r)))
    agg = collections.OrderedDict()
    data = [d for d in data if "gs::" in d["Kernel Name"]]  # ours only (scene set-up is torch)
    for d in data:
        nm = d["Kernel Name"].split("(")[0].replace("void ", "")
        a = agg.setdefault(nm, [0, 0.0])
        a[0] += 1
        a[1] += float(d["Metric Value"].replace(",", ""))
    tot = sum(a[1] for a in agg.values())
    with open(out, "w") as fh:
        fh.write(f"# ncu launch list: {path}\n\n`ncu --metrics gpu__time_duration.sum --clock-control none` over "
                 f"{iters} eager iterations (cold-cache, serialised: compare shares, not absolutes).\n\n")
        fh.write(f"Total {tot/1e3:.1f} us, {len(data)} launches of ours (the set-up binning passes of the "
                 f"engine's views are included).\n\n")
        fh.write("| kernel | launches | us total | us / launch | share |\n|---|---|---|---|---|\n")
        for k, (c, v) in sorted(agg.items(), key=lambda x: -x[1][1]):
            fh.write(f"| `{k}` | {c} | {v/1e3:.1f} | {v/1e3/c:.1f} | {100*v/tot:.1f}% |\n")
    print(open(out).read())


def full(path, out):
    raw = subprocess.run(["ncu", "-i", path, "--page", "raw", "--csv"], capture_output=True, text=True).stdout
    rows = list(csv.reader(io.StringIO(raw)))
    h, units = rows[0], rows[1]
    with open(out, "w") as fh:
        fh.write(f"# ncu --set full: {path}\n\n")
        for r in rows[2:]:
            d = dict(zip(h, r))
            fh.write(f"## `{d.get('Kernel Name', '?')[:120]}`\n\n| metric | value |\n|---|---|\n")
            for k in KEYS:
                if k in h:
                    fh.write(f"| {k} | {d[k]} {units[h.index(k)]} |\n")
            fh.write("\n")
    print(open(out).read())


if __name__ == "__main__":
    if sys.argv[1] == "launches":
        launches(sys.argv[2], sys.argv[3], int(sys.argv[4]) if len(sys.argv) > 4 else 1)
    else:
        full(sys.argv[2], sys.argv[3])
