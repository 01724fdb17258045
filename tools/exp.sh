run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
for v in def hotmask hotmaskpf nomask; do
  if [ $v = def ]; then unset SPMV_LIB_PATH; else export SPMV_LIB_PATH=exp/$v/libspmv.so; fi
  run c3_$v --config 3 --steps 30
  run c4_$v --config 4 --steps 30
done
unset SPMV_LIB_PATH
run c3_def2 --config 3 --steps 30
