timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t11.log 2>&1; echo rc=$?; tail -3 gpurun_out/t11.log
timeout 600 python tools/exp_passes.py --config 2 --passes 0 --reps 2 2>&1 | tail -1
timeout 900 python tools/exp_passes.py --config 3 --passes 0 --reps 2 2>&1 | tail -1
timeout 1500 python tools/exp_passes.py --config 4 --iters 1 --reps 1 --passes 0 2>&1 | tail -1
