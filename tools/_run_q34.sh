timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt_q34.log 2>&1; echo "rc=$?" >> gpurun_out/pt_q34.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_q34.json 2> gpurun_out/bench_q34.err
timeout 300 ncu --profile-from-start off --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum \
    --clock-control none --cache-control none --csv --log-file gpurun_out/graph_q34.csv \
    python tools/prof_graph.py S2r-1M-1280x720-32line 8 > gpurun_out/graph_q34.log 2>&1
tail -2 gpurun_out/pt_q34.log; head -c 300 gpurun_out/bench_q34.json
