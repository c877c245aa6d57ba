timeout 2400 python -m pytest tests -m gpu -x -q > gpurun_out/t5_pytest.log 2>&1; echo pytest=$?; tail -3 gpurun_out/t5_pytest.log
timeout 600 python tools/ivfd_vs_ivf.py --config 1 2>&1 | tail -1
timeout 900 python tools/ivfd_vs_ivf.py --config 2 2>&1 | tail -1
for c in 2 3 4; do
timeout 1500 python bench.py --config $c --steps 3 --warmup 3 --no-secondary --no-cpu-baseline --e2e-steps 0 > gpurun_out/t5_b$c.log 2>&1; echo b$c=$?; tail -1 gpurun_out/t5_b$c.log | python -c "
import json,sys; d=json.loads(sys.stdin.read()); r=d['roofline']; print(d['config']['workload'], d['value'], r['bound'], r['frac'], r.get('traffic'), r.get('traffic_launches'), r.get('l2',{}).get('frac'), r['hbm'].get('dram_frac'))"
done
