# launch lists (cold ncu) of a few bench steps of the render and S1 configs
for C in S2r-2M-1920x1080-render S1-1M-1280x720; do
  timeout 600 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file gpurun_out/cfg_$C.csv -c 400 \
     python bench.py --config $C --steps 3 --warmup 3 --no-cpu-baseline > gpurun_out/cfg_$C.log 2>&1
done
timeout 300 python bench.py --config S2r-2M-1920x1080-render --steps 300 --warmup 5 --no-cpu-baseline > gpurun_out/render_lazy.json 2>&1
