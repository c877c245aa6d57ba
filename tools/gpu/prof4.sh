NCU=/usr/local/cuda/bin/ncu
timeout 1200 $NCU --nvtx --nvtx-include "profile/" -k regex:screen_kernel -c 1 --set full --import-source on --clock-control none -o gpurun_out/r2_c4_screen_pass python tools/prof_screen.py --config 4 --iters 2 > gpurun_out/prof4.log 2>&1; echo prof4=$?; tail -3 gpurun_out/prof4.log
