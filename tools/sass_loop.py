"""Print the SASS of a kernel's instructions executed at least <min> times (the hot loops), from
an ncu report: python tools/sass_loop.py <rep> <kernel-regex> <min-exec>"""
import csv
import io
import subprocess
import sys

rep, k, lo = sys.argv[1], sys.argv[2], int(sys.argv[3])
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{k}", "--print-source", "sass"],
                     capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
for i, r in enumerate(rows):
    if "Address" in r and "Source" in r:
        h, start = r, i + 1
        break
ix = {n: j for j, n in enumerate(h)}
n = 0
for r in rows[start:]:
    if len(r) != len(h) or not r[ix["Address"]].startswith("0x"):
        continue
    ex = int(r[ix["Instructions Executed"]] or 0)
    if ex >= lo:
        n += 1
        print(r[ix["Address"]][-5:], ex, r[ix["Warp Stall Sampling (All Samples)"]], r[ix["Source"]])
print(n, "instructions")
