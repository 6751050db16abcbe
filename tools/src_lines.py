"""Per-CUDA-source-line totals from `ncu --page source --csv --print-source cuda,sass` output:
python tools/src_lines.py <csv> [top]"""
import collections
import csv
import sys

rows = list(csv.reader(open(sys.argv[1])))
top = int(sys.argv[2]) if len(sys.argv) > 2 else 30
fname, hdr = None, None
inst, samp, text = collections.Counter(), collections.Counter(), {}
cur = None
for r in rows:
    if not r:
        continue
    if r[0] == "File Path":
        fname = r[1].split("/")[-1]
        continue
    if r[0] == "Line No":
        hdr = r
        continue
    if hdr is None or len(r) < 8:
        continue
    if r[0]:  # a CUDA source line
        cur = (fname, int(r[0]))
        text[cur] = r[1].strip()
    if r[2].startswith("0x") and cur is not None:
        d = dict(zip(hdr[2:], r[2:]))
        inst[cur] += int(d.get("Instructions Executed") or 0)
        samp[cur] += int(d.get("Warp Stall Sampling (All Samples)") or 0)
ti, ts = sum(inst.values()), sum(samp.values())
print(f"warp-instr {ti}, stall samples {ts}")
for k, v in sorted(inst.items(), key=lambda x: -x[1])[:top]:
    print(f"{k[0]:>14s}:{k[1]:<5d} inst {100*v/ti:5.1f}%  stall {100*samp[k]/max(ts,1):5.1f}%  {text.get(k, '')[:80]}")
