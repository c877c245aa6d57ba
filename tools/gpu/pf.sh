timeout 900 python tools/exp_passes.py --config 3 --passes 0,4 --pf 0,4,8,16,32 2>&1 | tail -10
timeout 600 python tools/exp_passes.py --config 2 --passes 0,16 --pf 0,8,16,32 2>&1 | tail -8
timeout 600 python tools/exp_passes.py --config 1 --passes 0 --pf 0,8,16 2>&1 | tail -3
