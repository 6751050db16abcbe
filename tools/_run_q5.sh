timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt_q5.log 2>&1; echo "rc=$?" >> gpurun_out/pt_q5.log
bash tools/gpu_sweep.sh sw1
tail -3 gpurun_out/pt_q5.log
