for c in 2 3 4; do timeout 900 python tools/bivf_stats.py --config $c --iters 2 2>&1 | tail -2; done
