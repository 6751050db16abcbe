timeout 600 python tools/debug/big_stats.py > gpurun_out/big_stats.txt 2>&1
cat gpurun_out/big_stats.txt | tail -8
