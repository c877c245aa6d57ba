# bench (driver settings), reference arm, launch list, ncu full captures
python bench.py --impl reference --steps 20 --warmup 5 > gpurun_out/f1_ref.log 2>&1; echo ref=$?; tail -c 1500 gpurun_out/f1_ref.log
python bench.py --steps 20 --warmup 5 > gpurun_out/f1_bench.log 2>&1; echo bench=$?; tail -c 3000 gpurun_out/f1_bench.log
NCU=/usr/local/cuda/bin/ncu
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file gpurun_out/f1_launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --no-traffic --e2e-steps 0 > gpurun_out/f1_ncu_ll.log 2>&1; echo ll=$?
timeout 900 $NCU --nvtx --nvtx-include "profile/" -k regex:screen_kernel -c 1 --set full --import-source on --clock-control none -o gpurun_out/r2_c1_screen python tools/prof_screen.py --config 1 > gpurun_out/f1_prof1.log 2>&1; echo prof1=$?
timeout 900 python tools/bivf_stats.py --config 1 2>&1 | tail -1
timeout 900 python tools/bivf_stats.py --config 3 2>&1 | tail -1
