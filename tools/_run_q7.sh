timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -q -k "full_size or lazy or binning or forward" > gpurun_out/pt_q7.log 2>&1; echo "rc=$?" >> gpurun_out/pt_q7.log
timeout 300 python bench.py --config S2r-2M-1920x1080-render --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/render_q7.json 2>&1
timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg_render_q7.csv -c 200 \
     python bench.py --config S2r-2M-1920x1080-render --steps 3 --warmup 3 --no-cpu-baseline > /dev/null 2>&1
tail -2 gpurun_out/pt_q7.log; head -c 900 gpurun_out/render_q7.json
