# C4 fused split kernel: occupancy / long-item unroll variants (experiment)
echo "== default"; timeout 120 python tools/exp_c4_parts.py --tma 2>&1 | grep "full.*long_mode': 2"
for v in "lb5 -DSPLIT_LB=5" "lb6 -DSPLIT_LB=6" "lb6u8 -DSPLIT_LB=6 -DLONG_U=8" "lb5u12 -DSPLIT_LB=5 -DLONG_U=12" "u24 -DLONG_U=24" "xb4096 -DLONG_XB=4096"; do
  set -- $v; name=$1; shift
  bash tools/build_variant.sh $name "$@" > /dev/null 2>&1
  grep -h -A1 "split_fused_kernel" exp/$name/*.txt 2>/dev/null | head -2
  echo "== $name"; SPMV_LIB_PATH=exp/$name/libspmv.so timeout 120 python tools/exp_c4_parts.py --tma 2>&1 | grep "long_mode': 2"
done
