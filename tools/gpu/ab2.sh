timeout 600 python tools/exp_passes.py --config 1 --passes 0 --reps 3 2>&1 | tail -1
timeout 600 python tools/exp_passes.py --config 2 --passes 0 --reps 3 2>&1 | tail -1
timeout 900 python tools/exp_passes.py --config 3 --passes 0 --reps 2 2>&1 | tail -1
timeout 900 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -2
timeout 900 python tools/bivf_stats.py --config 1 2>&1 | tail -1
