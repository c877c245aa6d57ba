for c in 3 2; do timeout 900 python tools/exp_passes.py --config $c --passes 0,2,4,8,16,40 2>&1 | tail -8; done
timeout 900 python tools/exp_passes.py --config 4 --iters 1 --reps 1 --passes 0,4,8,16,32 2>&1 | tail -6
