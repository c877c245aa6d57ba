timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t4_parity.log 2>&1; echo parity=$?; tail -3 gpurun_out/t4_parity.log
timeout 600 python tools/exp_passes.py --config 1 --passes 0 2>&1 | tail -1
timeout 600 python tools/exp_passes.py --config 2 --passes 0,8,10,12 2>&1 | tail -4
timeout 900 python tools/exp_passes.py --config 3 --passes 0,4,6 2>&1 | tail -3
timeout 1500 python tools/exp_passes.py --config 4 --iters 1 --reps 1 --passes 0,16 2>&1 | tail -2
