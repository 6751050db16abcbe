timeout 900 ncu --profile-from-start off --set full --import-source on --clock-control none --cache-control none \
    -k "regex:render_bwd|tile_finish" -c 2 -o gpurun_out/full_s1 python tools/prof_graph.py S1-1M-1280x720 1 > gpurun_out/full_s1.log 2>&1
tail -2 gpurun_out/full_s1.log
