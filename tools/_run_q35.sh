timeout 600 python tools/debug/e2e_probe.py > gpurun_out/e2e_probe.txt 2>&1; tail -6 gpurun_out/e2e_probe.txt
