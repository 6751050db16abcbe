#!/bin/bash
# gpurun --timeout 1500 -- bash tools/gpu_full.sh <tag> <kernel-regex> [count] [pytest-args]
# --set full captures (warm, graph replay) of the kernels matching the regex, after the GPU tests.
TAG=${1:-f}; K=${2:-ssim_fwd_kernel}; C=${3:-6}; shift 3; PT=${@:-tests -m gpu -x -q}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
timeout 900 python -m pytest $PT > gpurun_out/pt_$TAG.log 2>&1; echo "rc=$?" >> gpurun_out/pt_$TAG.log
timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none --cache-control none \
    -k "regex:$K" -c $C -o gpurun_out/full_$TAG python tools/prof_graph.py S2r-1M-1280x720-32line 2 \
    > gpurun_out/full_$TAG.log 2>&1
tail -3 gpurun_out/pt_$TAG.log; tail -3 gpurun_out/full_$TAG.log
