timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q > gpurun_out/t10.log 2>&1; echo rc=$?; tail -1 gpurun_out/t10.log
