NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --nvtx --nvtx-include "profile/" -k regex:screen_kernel -c 1 --set full --import-source on --clock-control none -o gpurun_out/r2_c3_screen_pass python tools/prof_screen.py --config 3 > gpurun_out/prof3.log 2>&1; echo prof3=$?
timeout 900 $NCU --nvtx --nvtx-include "profile/" -k regex:screen_kernel -c 1 --set full --import-source on --clock-control none -o gpurun_out/r2_c2_screen_pass python tools/prof_screen.py --config 2 > gpurun_out/prof2.log 2>&1; echo prof2=$?
tail -5 gpurun_out/prof3.log
