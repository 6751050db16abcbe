"""Per-instruction execution counts of one kernel (address order, runs of equal counts):
python tools/sass_runs.py <rep> <kernel-regex> [min-count]"""
import csv, io, subprocess, sys
rep, k = sys.argv[1], sys.argv[2]
mn = int(sys.argv[3]) if len(sys.argv) > 3 else 0
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{k}", "--launch-count", "1"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
seen, d2 = set(), []
for r in rows[2:]:
    if len(r) == len(h) and r[0].startswith("0x") and r[0] not in seen:
        seen.add(r[0]); d2.append(dict(zip(h, r)))
prev = None; start = None; n = 0; stall = 0; first = ""
def flush():
    if prev is not None and prev >= mn:
        print(f"{start[-5:]} x{n:4d} exec {prev:9d} stall {stall:5d}  {first[:60]}")
for d in d2:
    e = int(d["Instructions Executed"] or 0)
    s = int(d["Warp Stall Sampling (All Samples)"] or 0)
    if e != prev:
        flush(); prev = e; start = d["Address"]; n = 0; stall = 0; first = d["Source"]
    n += 1; stall += s
flush()
