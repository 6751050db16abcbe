#!/bin/bash
# gpurun -- bash tools/ncu_metrics.sh <tag> <kernel-regex> [skip]: pipe / shared-memory / L1 breakdown of
# one steady-state launch of the bench iteration
TAG=${1:-x}; K=${2:-ssim_fwd_kernel}; S=${3:-6}
mkdir -p gpurun_out
M=gpu__time_duration.sum,smsp__inst_executed.sum,smsp__issue_active.avg.pct_of_peak_sustained_active,\
sm__warps_active.avg.pct_of_peak_sustained_active,l1tex__throughput.avg.pct_of_peak_sustained_active,\
l1tex__data_pipe_lsu_wavefronts_mem_shared_op_ld.sum,l1tex__data_pipe_lsu_wavefronts_mem_shared_op_st.sum,\
l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_ld.sum,l1tex__data_bank_conflicts_pipe_lsu_mem_shared_op_st.sum,\
smsp__inst_executed_op_shared_ld.sum,smsp__inst_executed_op_shared_st.sum,smsp__inst_executed_op_global_ld.sum,\
smsp__inst_executed_op_global_st.sum,l1tex__t_requests_pipe_lsu_mem_global_op_ld.sum,l1tex__t_sectors_pipe_lsu_mem_global_op_ld.sum,\
l1tex__t_sectors_pipe_lsu_mem_global_op_st.sum,smsp__sass_inst_executed_op_ldgsts.sum,l1tex__data_pipe_lsu_wavefronts.sum,\
sm__pipe_fma_cycles_active.avg.pct_of_peak_sustained_active,sm__pipe_alu_cycles_active.avg.pct_of_peak_sustained_active,\
sm__inst_executed_pipe_lsu.avg.pct_of_peak_sustained_active,sm__mio_inst_issued.avg.pct_of_peak_sustained_active,\
smsp__average_warp_latency_issue_stalled_barrier.ratio,smsp__average_warp_latency_issue_stalled_mio_throttle.ratio,\
smsp__average_warp_latency_issue_stalled_short_scoreboard.ratio,smsp__average_warp_latency_issue_stalled_long_scoreboard.ratio,\
smsp__average_warp_latency_issue_stalled_wait.ratio,smsp__average_warp_latency_issue_stalled_math_pipe_throttle.ratio,\
smsp__average_warp_latency_issue_stalled_not_selected.ratio,smsp__average_warp_latency_issue_stalled_lg_throttle.ratio
timeout 900 ncu --metrics $M --clock-control none -k "regex:$K" --launch-skip $S -c 1 --csv \
    python tools/prof_iter.py S2r-1M-1280x720-32line 6 > gpurun_out/metrics_$TAG.csv 2> gpurun_out/metrics_$TAG.err
python - gpurun_out/metrics_$TAG.csv > gpurun_out/metrics_$TAG.txt <<'PY'
import csv, sys
rows = [r for r in csv.reader(open(sys.argv[1])) if len(r) > 10]
h = rows[0]
for r in rows[1:]:
    d = dict(zip(h, r))
    print(d["Kernel Name"][:40], d["Metric Name"], d["Metric Value"])
PY
