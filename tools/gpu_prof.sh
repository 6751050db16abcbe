#!/bin/bash
# gpurun --timeout 1800 -- bash tools/gpu_prof.sh <tag> <kernel-regex> [count]
# GPU tests + bench + ncu launch list + full captures of the kernels matching the regex.
TAG=${1:-x}; K=${2:-render_bwd_kernel}; C=${3:-6}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 600 python bench.py --no-cpu-baseline > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --cache-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python tools/prof_iter.py S2r-1M-1280x720-32line 4 > /dev/null 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k "regex:$K" -c $C \
    -o gpurun_out/prof_$TAG python tools/prof_iter.py S2r-1M-1280x720-32line 4 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -3 gpurun_out/pytest_gpu_$TAG.log; cat gpurun_out/bench_$TAG.json | head -c 300
