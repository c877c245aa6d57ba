timeout 900 python tools/exp_passes.py --config 3 --passes 0,4 --warps 0,4,8 2>&1 | tail -6
timeout 600 python tools/exp_passes.py --config 2 --passes 0,16 --warps 0,2,4,8 2>&1 | tail -8
timeout 900 python tools/exp_passes.py --config 4 --iters 1 --reps 1 --passes 0,16 --warps 0,4,8 2>&1 | tail -6
