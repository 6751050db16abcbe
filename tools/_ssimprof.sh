mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k "regex:ssim|adam_list|chain_kernel|render_fwd" -c 4 \
    -o gpurun_out/prof_ssim python tools/prof_iter.py S2r-1M-1280x720-32line 2 > gpurun_out/ncu_ssim.log 2>&1
