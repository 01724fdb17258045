make -j32 >/dev/null 2>&1
timeout 300 python tools/dbg_long_tma.py 2>&1 | grep -E "rc|TIMEOUT|case" | head -20
echo "== default (CH256 D4 NW8 UN8)"; timeout 120 python tools/exp_c4_parts.py --tma
for v in "ch512un16 -DLT_CH=512 -DLT_UN=16 -DLT_MINB=2" "nw16 -DLT_NW=16 -DLT_D=3 -DLT_MINB=2" "nw16ch512 -DLT_NW=16 -DLT_D=2 -DLT_CH=512 -DLT_MINB=2"; do
  set -- $v; name=$1; shift
  bash tools/build_variant.sh $name "$@" > /dev/null 2>&1
  echo "== $name"; SPMV_LIB_PATH=exp/$name/libspmv.so timeout 120 python tools/exp_c4_parts.py --tma
done
