mkdir -p gpurun_out
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_filter_spectra -s 0 -c 1 -o gpurun_out/p58_fsg python tools/prof_step.py 1 bwd_filter 128,64,128,224,8 > /dev/null 2>&1
timeout 600 ncu --set full --clock-control none --import-source on -k regex:oaa_tile_spectra -s 0 -c 1 -o gpurun_out/p58_ts python tools/prof_step.py 1 fwd 256,96,256,27,5 > /dev/null 2>&1
