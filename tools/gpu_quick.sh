#!/bin/bash
# gpurun --timeout 900 -- bash tools/gpu_quick.sh <tag>: GPU tests, bench (no CPU baseline), warm launch list
TAG=${1:-q}
mkdir -p gpurun_out
timeout 600 python -m pytest tests -m gpu -x -q > gpurun_out/pt_$TAG.log 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv \
    --log-file gpurun_out/launches_$TAG.csv python tools/prof_iter.py S2r-1M-1280x720-32line 4 > /dev/null 2>&1
