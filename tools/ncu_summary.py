"""One line per profiled kernel of an ncu raw CSV page + its top stall reasons."""
import csv
import sys
rows = list(csv.reader(open(sys.argv[1])))
hdr = rows[0]
keys = ['gpu__time_duration.sum', 'smsp__issue_active.avg.pct_of_peak_sustained_active',
        'sm__warps_active.avg.pct_of_peak_sustained_active', 'l1tex__throughput.avg.pct_of_peak_sustained_active',
        'dram__bytes_read.sum', 'dram__bytes_write.sum', 'launch__registers_per_thread', 'smsp__inst_executed.sum']
stalls = [h for h in hdr if h.startswith('smsp__pcsamp_warps_issue_stalled_') and not h.endswith('not_issued')]
for r in rows[2:]:
    d = dict(zip(hdr, r))
    name = d.get('Kernel Name', '?')[:48]
    vals = " ".join(f"{k.split('__')[1].split('.')[0][:14]}={d.get(k)}" for k in keys)
    st = sorted(((float(d[h] or 0), h.replace('smsp__pcsamp_warps_issue_stalled_', '')) for h in stalls), reverse=True)[:6]
    print(f"{name} | {vals}\n    stalls: {st}")
