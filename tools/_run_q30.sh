timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "mapper or mapping_loop" > gpurun_out/pt_q30.log 2>&1; echo "rc=$?" >> gpurun_out/pt_q30.log
tail -25 gpurun_out/pt_q30.log
