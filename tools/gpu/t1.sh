timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t1_parity.log 2>&1; echo parity=$?; tail -3 gpurun_out/t1_parity.log
timeout 600 python tools/exp_passes.py --config 2 --passes 0,1,10,14,20 2>&1 | tail -5
timeout 900 python tools/exp_passes.py --config 3 --passes 0,1,3,4,5,6 2>&1 | tail -6
timeout 1500 python tools/exp_passes.py --config 4 --iters 1 --reps 1 --passes 0,1,12,20,30 2>&1 | tail -5
timeout 2400 python -m pytest tests/test_gpu_configs.py -x -q > gpurun_out/t1_configs.log 2>&1; echo configs=$?; tail -5 gpurun_out/t1_configs.log
