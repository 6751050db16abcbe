timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt_q36.log 2>&1; echo "rc=$?" >> gpurun_out/pt_q36.log
timeout 600 python tools/debug/e2e_probe.py > gpurun_out/e2e_probe2.txt 2>&1
timeout 300 python bench.py --no-cpu-baseline > gpurun_out/bench_q36.json 2> gpurun_out/bench_q36.err
tail -2 gpurun_out/pt_q36.log; tail -4 gpurun_out/e2e_probe2.txt; python -c "
import json;d=json.load(open('gpurun_out/bench_q36.json'));print(d['value'], d['e2e']['value'])"
