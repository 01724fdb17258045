#!/bin/bash
# Round-2 measurements on one B200 (run under gpurun): full bench lines per
# config, the reference arm, the C5 launch list, and for each config's
# dominant kernel one `ncu --set full` capture (cold: ncu flushes caches) plus
# one warm capture (--cache-control none, the 4th back-to-back launch: the
# state the timed loop runs in). Outputs in gpurun_out/prof/.
cd "$(dirname "$0")/.."
out=gpurun_out/prof
mkdir -p $out
for c in 5 2 3 4 1; do
  timeout 600 python bench.py --config $c > $out/bench_c$c.log 2>&1
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c5.csv \
  python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e --no-cold --iters 0 --no-paper-runs > $out/ncu_launch_c5.log 2>&1
declare -A K=([5]="d8_kernel" [2]="d8_kernel" [3]="nzsplit_kernel" [4]="split_fused_kernel")
WARM="gpu__time_duration.sum,dram__bytes_read.sum,dram__bytes_write.sum,lts__t_sector_hit_rate.pct,dram__throughput.avg.pct_of_peak_sustained_elapsed"
for c in 5 2 3 4; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:${K[$c]} -s 2 -c 1 \
    -o $out/full_c$c python tools/prof_one.py --config $c --reps 3 > $out/ncu_full_c$c.log 2>&1
  timeout 900 ncu --cache-control none --clock-control none -k regex:${K[$c]} -s 3 -c 1 --metrics $WARM --csv \
    --log-file $out/warm_c$c.csv python tools/prof_one.py --config $c --reps 5 > $out/ncu_warm_c$c.log 2>&1
done
# the int32-colind stream kernel on C5 (the round-1 path, D8 off) for comparison
timeout 900 ncu --set full --import-source on --clock-control none -k regex:stream_kernel -s 2 -c 1 \
  -o $out/full_c5_int32 python tools/prof_one.py --config 5 --reps 3 --opts '{"d16": 0}' > $out/ncu_full_c5_int32.log 2>&1
timeout 900 ncu --cache-control none --clock-control none -k regex:stream_kernel -s 3 -c 1 --metrics $WARM --csv \
  --log-file $out/warm_c5_int32.csv python tools/prof_one.py --config 5 --reps 5 --opts '{"d16": 0}' > $out/ncu_warm_c5_int32.log 2>&1
# forced-variant sweeps (selection regret) and the Table V analogue
for c in 2 3 4; do timeout 900 python tools/sweep.py --config $c --quick --out $out/sweep_c$c.json > $out/sweep_c$c.log 2>&1; done
timeout 1200 python tools/sweep.py --config 5 --quick --reps 5 --out $out/sweep_c5.json > $out/sweep_c5.log 2>&1
timeout 900 python tools/table5.py --configs 2,3,4,5 --out $out/table5.json > $out/table5.log 2>&1
# iterated-mode overhead vs back-to-back SpMVs, and the emulated-shard timeline
timeout 600 python tools/exp_iter2.py --config 2 --iters 1000 > $out/iter_overhead.log 2>&1
timeout 600 python tools/exp_iter2.py --config 5 --iters 100 >> $out/iter_overhead.log 2>&1
timeout 600 python tools/timeline_iter.py --n 160 --G 4 --iters 3 > $out/timeline_iter.log 2>&1
python tools/sass_summary.py > $out/sass_summary.txt 2>&1
echo done
