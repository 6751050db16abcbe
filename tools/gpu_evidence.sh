#!/bin/bash
# One gpurun call producing the round's evidence: GPU parity tests, smoke, bench (N=1, with CPU
# baseline), reference arm, ncu launch list, and --set full captures of the top kernels.
#   gpurun --timeout 2400 -- bash tools/gpu_evidence.sh <tag> [kernel-regex] [count]
TAG=${1:-ev}; K=${2:-render_bwd_kernel|preprocess_kernel|ssim_fwd_kernel|ssim_bwd_kernel|chain_kernel|render_fwd_kernel|big_cull|huge_sort|tile_scan}; C=${3:-10}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build_$TAG.log 2>&1
nvidia-smi > gpurun_out/nvidia-smi_$TAG.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu_$TAG.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu_$TAG.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke_$TAG.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke_$TAG.log
timeout 600 python bench.py > gpurun_out/bench_$TAG.json 2> gpurun_out/bench_$TAG.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref_$TAG.json 2> gpurun_out/bench_ref_$TAG.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches_$TAG.csv \
    python tools/prof_iter.py S2r-1M-1280x720-32line 4 > gpurun_out/ncu_launch_$TAG.log 2>&1
timeout 1200 ncu --profile-from-start off --set full --clock-control none --cache-control none --import-source on -k "regex:$K" -c $C \
    -o gpurun_out/prof_$TAG python tools/prof_graph.py S2r-1M-1280x720-32line 1 > gpurun_out/ncu_full_$TAG.log 2>&1
tail -3 gpurun_out/pytest_gpu_$TAG.log; tail -2 gpurun_out/smoke_$TAG.log; head -c 600 gpurun_out/bench_$TAG.json; echo; head -c 400 gpurun_out/bench_ref_$TAG.json
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --cache-control none --csv --log-file gpurun_out/graph_$TAG.csv \
    python tools/prof_graph.py S2r-1M-1280x720-32line 8 > gpurun_out/graph_$TAG.log 2>&1
bash tools/gpu_sweep.sh $TAG
