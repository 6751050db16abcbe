timeout 900 python -m pytest tests -m gpu -q > gpurun_out/pt_q29.log 2>&1; echo "rc=$?" >> gpurun_out/pt_q29.log
tail -3 gpurun_out/pt_q29.log
