make -j32 >/dev/null 2>&1
timeout 300 python tools/dbg_long_tma.py 2>&1 | grep -E "rc|TIMEOUT|case" | head -20
echo "== default"; timeout 120 python tools/exp_c4_parts.py --tma
for v in "ch512d4 -DLT_CH=512 -DLT_D=4" "ch128d8 -DLT_CH=128 -DLT_D=8" "nw16d4 -DLT_NW=16 -DLT_D=4 -DLT_MINB=2"; do
  set -- $v; name=$1; shift
  bash tools/build_variant.sh $name "$@" > /dev/null 2>&1
  echo "== $name"; SPMV_LIB_PATH=exp/$name/libspmv.so timeout 120 python tools/exp_c4_parts.py --tma
done
