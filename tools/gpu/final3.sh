timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/f3_pytest.log 2>&1; echo pytest=$?; tail -1 gpurun_out/f3_pytest.log
python bench.py --config 4 --steps 3 --warmup 3 --no-secondary --no-cpu-baseline --e2e-steps 2 > gpurun_out/f3_c4.log 2>&1; echo c4=$?
python bench.py --config 2 --steps 10 --warmup 3 --no-secondary --no-cpu-baseline > gpurun_out/f3_c2.log 2>&1; echo c2=$?
python bench.py --config 3 --steps 5 --warmup 3 --no-secondary --no-cpu-baseline --e2e-steps 3 > gpurun_out/f3_c3.log 2>&1; echo c3=$?
for c in 2 3 4; do tail -1 gpurun_out/f3_c$c.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['workload'], round(d['value'],4), round(d['ms_per_step'],1), round(d['screen_ms'],1), r['bound'], round(r['frac'],3), r.get('traffic'), r.get('l2',{}).get('frac'), r['hbm'].get('dram_frac'), d['e2e']['value'], d['e2e']['run_api']['value'])"; done
