#!/bin/bash
# Round measurements on one B200 (run under gpurun): full bench lines per
# config, the reference arm, the C5 launch list and one `ncu --set full`
# capture of each config's dominant kernel. Outputs in gpurun_out/prof/.
cd "$(dirname "$0")/.."
out=gpurun_out/prof
mkdir -p $out
for c in 5 2 3 4 1; do
  timeout 600 python bench.py --config $c > $out/bench_c$c.log 2>&1
done
timeout 600 python bench.py --impl reference --steps 3 --warmup 1 > $out/bench_ref.log 2>&1
timeout 900 ncu --metrics gpu__time_duration.sum --clock-control none --csv --log-file $out/launches_c5.csv \
  python bench.py --steps 3 --warmup 1 --no-cpu --no-e2e --no-cold --iters 0 > $out/ncu_launch_c5.log 2>&1
declare -A K=([5]="stream_kernel" [2]="stream_kernel" [3]="nzsplit_kernel" [4]="split_fused_kernel" [1]="stream_kernel")
for c in 5 2 3 4; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:${K[$c]} -s 2 -c 1 \
    -o $out/full_c$c python tools/prof_one.py --config $c --reps 3 > $out/ncu_full_c$c.log 2>&1
done
for c in 2 3 4; do timeout 900 python tools/sweep.py --config $c --out $out/sweep_c$c.json > $out/sweep_c$c.log 2>&1; done
timeout 1200 python tools/sweep.py --config 5 --quick --reps 5 --out $out/sweep_c5.json > $out/sweep_c5.log 2>&1
timeout 900 python tools/table5.py --configs 2,3,4,5 --out $out/table5.json > $out/table5.log 2>&1
timeout 1200 python tools/cusparse_context.py --configs 2,3,4,5 --out $out/cusparse.json > $out/cusparse.log 2>&1
echo done
