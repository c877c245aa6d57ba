timeout 2400 python -m pytest tests/test_gpu_configs.py -x -q > gpurun_out/t3_configs.log 2>&1; echo configs=$?; tail -3 gpurun_out/t3_configs.log
timeout 600 python tools/phase_times.py --config 1 2>&1 | tail -1
timeout 900 python tools/phase_times.py --config 3 --steps 3 2>&1 | tail -1
timeout 600 python tools/phase_times.py --config 2 --steps 3 2>&1 | tail -1
