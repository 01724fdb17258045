#!/bin/bash
# Build an experimental libspmv.so with extra -D flags into exp/<name>/:
#   tools/build_variant.sh pf24 -DNZ_HOT_WARPS=24 -DNZ_HOT_PF=1
# then run with SPMV_LIB_PATH=exp/<name>/libspmv.so
set -e
name=$1; shift
ROOT=$(cd "$(dirname "$0")/.." && pwd)
out=$ROOT/exp/$name
mkdir -p $out
objs=()
for f in $ROOT/paper_1711_05487_b200/csrc/*.cu; do
  b=$(basename $f .cu)
  /usr/local/cuda/bin/nvcc -O3 -std=c++17 -gencode arch=compute_100a,code=sm_100a -lineinfo -Xcompiler -fPIC \
    --expt-relaxed-constexpr -I$ROOT/include -I$ROOT/paper_1711_05487_b200/csrc "$@" -c -o $out/$b.o $f &
  objs+=($out/$b.o)
done
wait
/usr/local/cuda/bin/nvcc -gencode arch=compute_100a,code=sm_100a -shared -o $out/libspmv.so "${objs[@]}" -cudart static -lpthread -ldl -lrt
rm -f "${objs[@]}"
echo built $out/libspmv.so
