timeout 900 python -m pytest tests/test_gpu_parity.py -x -q -k "slot_range or cluster or assign_matches" 2>&1 | tail -1
for lib in old new; do
  if [ $lib = old ]; then export IVFKM_LIB=$PWD/paper_2002_09094_b200/_lib/libivfkm_old.so; else unset IVFKM_LIB; fi
  echo "== $lib"
  timeout 600 python tools/exp_passes.py --config 2 --passes 0 --reps 3 2>&1 | tail -1
  timeout 900 python tools/exp_passes.py --config 3 --passes 0 --reps 2 2>&1 | tail -1
  timeout 600 python tools/exp_passes.py --config 1 --passes 0 --reps 3 2>&1 | tail -1
done
unset IVFKM_LIB
timeout 2400 python -m pytest tests/test_gpu_configs.py -x -q 2>&1 | tail -1
