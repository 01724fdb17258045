out=gpurun_out/prof
mkdir -p $out
for c in 2 3 4; do timeout 900 python tools/sweep.py --config $c --out $out/sweep_c$c.json > $out/sweep_c$c.log 2>&1; done
timeout 1200 python tools/sweep.py --config 5 --quick --reps 5 --out $out/sweep_c5.json > $out/sweep_c5.log 2>&1
