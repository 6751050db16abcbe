#!/bin/bash
# One gpurun call: GPU parity tests, smoke, bench (N=1), ncu launch list and a full capture of
# the top kernel.  Everything lands in gpurun_out/.
#   gpurun --timeout 1800 -- bash tools/gpu_round.sh [kernel-regex]
set -x
K=${1:-render_bwd_kernel}
mkdir -p gpurun_out
python -c "import __graft_entry__ as g; g.build()" > gpurun_out/build.log 2>&1
nvidia-smi > gpurun_out/nvidia-smi.txt 2>&1
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pytest_gpu.log 2>&1; echo "pytest rc=$?" >> gpurun_out/pytest_gpu.log
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?" >> gpurun_out/smoke.log
timeout 600 python bench.py > gpurun_out/bench.json 2> gpurun_out/bench.err
timeout 600 python bench.py --impl reference --steps 2 --warmup 0 > gpurun_out/bench_ref.json 2> gpurun_out/bench_ref.err
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/launches.csv \
    python tools/prof_iter.py S2r-1M-1280x720-32line 4 > gpurun_out/ncu_launch.log 2>&1
timeout 900 ncu --set full --clock-control none --import-source on -k regex:$K -s 2 -c 1 \
    -o gpurun_out/prof python tools/prof_iter.py S2r-1M-1280x720-32line 4 > gpurun_out/ncu_full.log 2>&1
ls -la gpurun_out
