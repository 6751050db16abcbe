#!/bin/bash
# show results of tools/gpu_quick.sh <tag> [prev-tag]
T=$1; P=$2
tail -1 gpurun_out/pt_$T.log; grep -E "^E " gpurun_out/pt_$T.log | head -3
python - "$T" "$P" <<'PY'
import json, sys
for t in [x for x in sys.argv[2:0:-1] if x]:
    try:
        d = json.load(open(f"gpurun_out/bench_{t}.json")); print(t, d["value"], {k: v["ms"] for k, v in d["phases"].items()})
    except Exception as e:
        print(t, "no bench", e)
PY
python tools/summarize_ncu.py launches gpurun_out/launches_$T.csv /tmp/l_$T.md 4 | sed -n 7,30p
