timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt_q41.log 2>&1; echo "rc=$?" >> gpurun_out/pt_q41.log
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_q41.json 2> gpurun_out/bench_q41.err
tail -2 gpurun_out/pt_q41.log; python -c "
import json;d=json.load(open('gpurun_out/bench_q41.json'));print(d['value'], d['e2e'])"
