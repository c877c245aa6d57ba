timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "multipiece or capacity or ivfd or slot_range" 2>&1 | tail -3
