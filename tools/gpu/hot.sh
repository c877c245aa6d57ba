export IVFKM_LIB=$PWD/paper_2002_09094_b200/_lib/libivfkm_old.so
echo "== old"; timeout 600 python tools/exp_passes.py --config 1 --passes 0 --reps 3 2>&1 | tail -1
unset IVFKM_LIB
echo "== new"
timeout 600 python tools/exp_passes.py --config 1 --passes 0 --hot 0,16,64,256,1024 --reps 3 2>&1 | tail -5
timeout 600 python tools/exp_passes.py --config 2 --passes 0 --hot 0,64,256 --reps 2 2>&1 | tail -3
