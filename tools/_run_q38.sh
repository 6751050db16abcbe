timeout 900 python -m pytest tests/test_dp_gpu.py -m gpu -q > gpurun_out/pt_q38.log 2>&1; echo "rc=$?" >> gpurun_out/pt_q38.log
tail -30 gpurun_out/pt_q38.log
