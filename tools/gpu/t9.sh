timeout 1200 python -m pytest tests/test_gpu_parity.py -x -q 2>&1 | tail -1
python bench.py --config 3 --steps 3 --warmup 3 --no-secondary --no-cpu-baseline --no-traffic --e2e-steps 2 > gpurun_out/t9_b3.log 2>&1; echo b3=$?; tail -1 gpurun_out/t9_b3.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['e2e']['run_api']['value'], d['e2e']['run_api']['seconds'])"
