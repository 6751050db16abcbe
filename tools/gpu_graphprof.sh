#!/bin/bash
# gpurun -- bash tools/gpu_graphprof.sh <tag>: warm graph-replay per-kernel list (time, DRAM, instructions)
TAG=${1:-x}
mkdir -p gpurun_out
timeout 900 ncu --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,sm__warps_active.avg.pct_of_peak_sustained_active \
    --clock-control none --cache-control none --csv --log-file gpurun_out/graph_$TAG.csv \
    python tools/prof_iter.py S2r-1M-1280x720-32line 8 > gpurun_out/graph_$TAG.log 2>&1
python tools/graph_table.py gpurun_out/graph_$TAG.csv 8 gpurun_out/graph_$TAG.md
