python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/f2_smoke.log 2>&1; echo smoke=$?; tail -1 gpurun_out/f2_smoke.log
timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/f2_pytest.log 2>&1; echo pytest=$?; tail -2 gpurun_out/f2_pytest.log
python bench.py --steps 20 --warmup 5 > gpurun_out/f2_bench.log 2>&1; echo bench=$?; tail -1 gpurun_out/f2_bench.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); print(d['value'], d['e2e']['value'], d['e2e']['run_api'], d['roofline']['frac'], d['roofline'].get('l2',{}).get('frac'), d['secondary']['value'], d['clocks'])"
