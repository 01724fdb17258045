# C4 fused split kernel: block order experiments
echo "== default"; timeout 120 python tools/exp_c4_parts.py --tma 2>&1 | grep "full.*long_mode': 2"
for v in "lf -DSPLIT_LONG_FIRST" "lftpw2 -DSPLIT_LONG_FIRST -DSPLIT_TPW=2" "lftpw8 -DSPLIT_LONG_FIRST -DSPLIT_TPW=8" "lfrg1 -DSPLIT_LONG_FIRST -DLONG_RG=1" "lfrg4 -DSPLIT_LONG_FIRST -DLONG_RG=4"; do
  set -- $v; name=$1; shift
  bash tools/build_variant.sh $name "$@" > /dev/null 2>&1
  echo "== $name"; SPMV_LIB_PATH=exp/$name/libspmv.so timeout 120 python tools/exp_c4_parts.py --tma 2>&1 | grep "full.*long_mode': 2"
done
