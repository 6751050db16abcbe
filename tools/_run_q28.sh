timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "host_streaming or batch" > gpurun_out/pt_q28.log 2>&1; echo "rc=$?" >> gpurun_out/pt_q28.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_q28.json 2> gpurun_out/bench_q28.err
tail -2 gpurun_out/pt_q28.log; python -c "
import json;d=json.load(open('gpurun_out/bench_q28.json'));print(d['value'], d['e2e'])"
