# round-2 closing artefacts: bench lines (configs 1-4), reference arm, launch
# list, per-iteration kernel table, ncu full capture of the config-1 screen
NCU=/usr/local/cuda/bin/ncu
O=gpurun_out/r2c
mkdir -p $O
python bench.py > $O/bench_c1.json 2> $O/bench_c1.err; echo c1=$?
python bench.py --impl reference > $O/reference_c1.json 2> $O/reference_c1.err; echo ref=$?
timeout 900 $NCU --metrics gpu__time_duration.sum --clock-control none -c 800 --csv --log-file $O/launches.csv python bench.py --steps 5 --warmup 3 --no-cpu-baseline --no-secondary --no-traffic --e2e-steps 0 > $O/ncu_ll.log 2>&1; echo ll=$?
python tools/launch_table.py $O/launches.csv > $O/launch_list.txt
timeout 900 $NCU --nvtx --nvtx-include "iter/" --metrics gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum --clock-control none --csv --log-file $O/iter_c1.csv python tools/prof_iter.py --config 1 > $O/iter_c1.log 2>&1; echo iter=$?
python tools/launch_table.py $O/iter_c1.csv > $O/iteration_kernels.txt
timeout 900 $NCU --nvtx --nvtx-include "profile/" -k regex:screen_kernel -c 1 --set full --import-source on --clock-control none -f -o $O/c1_screen python tools/prof_screen.py --config 1 > $O/prof1.log 2>&1; echo prof1=$?
python bench.py --config 2 --steps 10 --warmup 3 --no-secondary --no-cpu-baseline > $O/bench_c2.json 2> $O/bench_c2.err; echo c2=$?
python bench.py --config 3 --steps 5 --warmup 3 --no-secondary --no-cpu-baseline --e2e-steps 3 > $O/bench_c3.json 2> $O/bench_c3.err; echo c3=$?
python bench.py --config 4 --steps 3 --warmup 3 --no-secondary --no-cpu-baseline --e2e-steps 2 > $O/bench_c4.json 2> $O/bench_c4.err; echo c4=$?
python -c "import __graft_entry__ as g; g.smoke()" > $O/smoke.log 2>&1; echo smoke=$?; tail -1 $O/smoke.log
tools/_build/fhfma_rate > $O/fhfma_rate.txt 2>&1
tools/_build/dram_random 16 > $O/dram_random.txt 2>&1
