GSLIC_OVERLAP_PARTS=4 timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "mapping_iterations or host_streaming" > gpurun_out/pt_q16.log 2>&1; echo "rc=$?" >> gpurun_out/pt_q16.log
for P in 0 2 4 8; do
  GSLIC_OVERLAP_PARTS=$P timeout 300 python bench.py --no-cpu-baseline --steps 500 > gpurun_out/bench_q16_$P.json 2>/dev/null
  echo "P=$P $(head -c 230 gpurun_out/bench_q16_$P.json | tail -c 110)"
done
tail -2 gpurun_out/pt_q16.log
