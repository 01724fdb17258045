run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/x_pytest.txt 2>&1
for v in def lb4 lb6 lb3 lb8; do
  if [ $v = def ]; then unset SPMV_LIB_PATH; else export SPMV_LIB_PATH=exp/$v/libspmv.so; fi
  run c5_$v --config 5 --steps 10
  run c2_$v --config 2 --steps 30
  run c1_$v --config 1 --steps 30
done
