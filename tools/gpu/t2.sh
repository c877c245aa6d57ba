timeout 1500 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t2_parity.log 2>&1; echo parity=$?; tail -3 gpurun_out/t2_parity.log
timeout 2400 python -m pytest tests/test_gpu_configs.py -x -q > gpurun_out/t2_configs.log 2>&1; echo configs=$?; tail -3 gpurun_out/t2_configs.log
timeout 1200 python bench.py --steps 10 --warmup 3 > gpurun_out/t2_bench.log 2>&1; echo bench=$?; tail -c 6000 gpurun_out/t2_bench.log
