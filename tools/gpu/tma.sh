timeout 600 python tools/exp_passes.py --config 1 --passes 0 --tma 0,1 --reps 3 2>&1 | tail -2
timeout 600 python tools/exp_passes.py --config 2 --passes 0 --tma 0,1 --reps 2 2>&1 | tail -2
timeout 900 python tools/exp_passes.py --config 3 --passes 0 --tma 0,1 --reps 2 2>&1 | tail -2
