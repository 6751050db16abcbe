timeout 900 python -m pytest tests/test_dp_gpu.py tests/test_gpu_parity.py -m gpu -q -k "two_ranks or batch" > gpurun_out/pt_q39.log 2>&1; echo "rc=$?" >> gpurun_out/pt_q39.log
timeout 900 python bench.py --batch --steps 30 --warmup 3 > gpurun_out/bench_q39_batch.json 2> gpurun_out/bench_q39_batch.err
tail -3 gpurun_out/pt_q39.log; head -c 700 gpurun_out/bench_q39_batch.json
