out=gpurun_out/prof
mkdir -p $out
declare -A K=([5]="stream_kernel" [2]="stream_kernel" [3]="nzsplit_kernel" [4]="split_fused_kernel")
for c in 5 2 3 4; do
  timeout 900 ncu --set full --import-source on --clock-control none -k regex:${K[$c]} -s 2 -c 1 \
    -o $out/full_c$c python tools/prof_one.py --config $c --reps 3 > $out/ncu_full_c$c.log 2>&1
done
