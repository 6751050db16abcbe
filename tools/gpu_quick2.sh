#!/bin/bash
# gpurun --timeout 1200 -- bash tools/gpu_quick2.sh <tag> [pytest-args]: GPU tests, bench (no CPU
# baseline), warm graph-replay launch list (profiler range = 8 replays)
TAG=${1:-q}; shift; PT=${@:-tests -m gpu -x -q}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest $PT > gpurun_out/pt_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pt_$TAG.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --cache-control none --csv --log-file gpurun_out/graph_$TAG.csv \
    python tools/prof_graph.py S2r-1M-1280x720-32line 8 > gpurun_out/graph_$TAG.log 2>&1
tail -3 gpurun_out/pt_$TAG.log; head -c 700 gpurun_out/bench_$TAG.json
