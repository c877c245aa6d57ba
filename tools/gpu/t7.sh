timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "multipiece" 2>&1 | grep -E "Error|assert|^E " | head -20
