timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "slot_range or ivfd" 2>&1 | tail -2
timeout 600 python tools/exp_passes.py --config 2 --passes 0 --presort 1,0 --reps 2 2>&1 | tail -2
timeout 900 python tools/exp_passes.py --config 3 --passes 0 --presort 1,0 --reps 2 2>&1 | tail -2
timeout 1500 python tools/exp_passes.py --config 4 --iters 1 --reps 1 --passes 0 --presort 1,0 2>&1 | tail -2
