for c in 3 2; do
timeout 900 python tools/sweep_screen.py --config $c --iters 2 --reps 2 --rr 0 --rowcap 512 --fill 0.015625 --order rowlen,label,mindf,meddf > gpurun_out/order_c$c.log 2>&1
echo "config $c rc=$?"; cat gpurun_out/order_c$c.log | grep screen_ms
done
