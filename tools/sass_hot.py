"""Hot SASS of one kernel from an ncu report: python tools/sass_hot.py <rep> <kernel-regex> [launch-skip]"""
import collections
import csv
import io
import subprocess
import sys

rep, k = sys.argv[1], sys.argv[2]
skip = sys.argv[3] if len(sys.argv) > 3 else "0"
out = subprocess.run(["ncu", "-i", rep, "--page", "source", "--csv", "-k", f"regex:{k}", "--launch-skip", skip,
                      "--launch-count", "1"], capture_output=True, text=True).stdout
rows = list(csv.reader(io.StringIO(out)))
h = rows[1]
data, seen = [], set()
for r in rows[2:]:
    if len(r) == len(h) and r[0].startswith("0x") and r[0] not in seen:
        seen.add(r[0])
        data.append(dict(zip(h, r)))
tot_i = sum(int(d["Instructions Executed"] or 0) for d in data)
tot_s = sum(int(d["Warp Stall Sampling (All Samples)"] or 0) for d in data)
ops = collections.Counter()
stalls = collections.Counter()
for d in data:
    op = d["Source"].split()[0] if d["Source"].split() else "?"
    if op.startswith("@"):
        op = d["Source"].split()[1]
    op = op.split(".")[0]
    ops[op] += int(d["Instructions Executed"] or 0)
    stalls[op] += int(d["Warp Stall Sampling (All Samples)"] or 0)
print(f"{rows[0]}  warp-instr {tot_i}  samples {tot_s}")
print("by opcode (instr%, stall%):")
for op, v in ops.most_common(25):
    print(f"  {op:10s} {100*v/tot_i:5.1f}% {100*stalls[op]/max(tot_s,1):5.1f}%")
print("hottest instructions by stall samples:")
for d in sorted(data, key=lambda d: -int(d["Warp Stall Sampling (All Samples)"] or 0))[:25]:
    print(f"  {d['Address'][-5:]} {int(d['Warp Stall Sampling (All Samples)'] or 0)*100/max(tot_s,1):5.1f}% "
          f"exec {int(d['Instructions Executed'] or 0):9d}  {d['Source'][:70]}")
