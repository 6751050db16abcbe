timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/pt_q17.log 2>&1; echo "rc=$?" >> gpurun_out/pt_q17.log
( time timeout 1200 python bench.py --batch --steps 30 --warmup 3 > gpurun_out/bench_q17_batch.json 2> gpurun_out/bench_q17_batch.err ) 2> gpurun_out/time_q17.txt
tail -2 gpurun_out/pt_q17.log; cat gpurun_out/bench_q17_batch.json | head -c 1500; tail -3 gpurun_out/bench_q17_batch.err; cat gpurun_out/time_q17.txt
