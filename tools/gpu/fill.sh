timeout 900 python tools/exp_passes.py --config 2 --passes 0 --reps 2 --fill 0.015625,0.03125,0.0625,0.125 2>&1 | tail -4
timeout 1200 python tools/exp_passes.py --config 3 --passes 0 --reps 1 --fill 0.015625,0.03125,0.0625,0.125 2>&1 | tail -4
timeout 2000 python tools/exp_passes.py --config 4 --iters 1 --reps 1 --passes 0 --fill 0.015625,0.03125,0.0625,0.125 2>&1 | tail -4
timeout 600 python tools/exp_passes.py --config 1 --passes 0 --reps 2 --fill 0.015625,0.03125 2>&1 | tail -2
