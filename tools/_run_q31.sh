timeout 600 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,smsp__inst_executed.sum,sm__warps_active.avg.pct_of_peak_sustained_active,smsp__issue_active.avg.pct_of_peak_sustained_active \
    --clock-control none --cache-control none --csv --log-file gpurun_out/graph_s1.csv \
    python tools/prof_graph.py S1-1M-1280x720 2 > gpurun_out/graph_s1.log 2>&1
tail -2 gpurun_out/graph_s1.log
