#!/bin/bash
# gpurun -- bash tools/gpu_ncu_kernel.sh <tag> <kernel-regex> [skip] [count]: full ncu captures of the
# matching kernels of the bench iteration (graph replay, steady state), source-mapped, + CSV pages
TAG=${1:-x}; K=${2:-ssim_fwd_kernel}; S=${3:-20}; C=${4:-1}
mkdir -p gpurun_out
timeout 1200 ncu --set full --clock-control none --import-source on -k "regex:$K" --launch-skip $S -c $C \
    -o gpurun_out/full_$TAG python tools/prof_iter.py S2r-1M-1280x720-32line 12 > gpurun_out/ncu_full_$TAG.log 2>&1
ncu -i gpurun_out/full_$TAG.ncu-rep --page raw --csv > gpurun_out/full_$TAG.raw.csv 2>/dev/null
ncu -i gpurun_out/full_$TAG.ncu-rep --page details --csv > gpurun_out/full_$TAG.details.csv 2>/dev/null
