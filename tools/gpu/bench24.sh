python bench.py --config 2 --steps 10 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/b_c2.log 2>&1; echo c2=$?; tail -c 600 gpurun_out/b_c2.log
python bench.py --config 4 --steps 3 --warmup 3 --no-secondary --no-cpu-baseline --e2e-steps 2 > gpurun_out/b_c4.log 2>&1; echo c4=$?; tail -c 600 gpurun_out/b_c4.log
python bench.py --config 3 --steps 5 --warmup 3 --no-secondary --no-cpu-baseline --e2e-steps 3 > gpurun_out/b_c3.log 2>&1; echo c3=$?; tail -c 600 gpurun_out/b_c3.log
