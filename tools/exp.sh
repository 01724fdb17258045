run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
for r in 1 2; do
run c2_lb5_$r --config 2 --steps 40
SPMV_LIB_PATH=exp/lb6/libspmv.so run c2_lb6_$r --config 2 --steps 40
SPMV_LIB_PATH=exp/lb6/libspmv.so run c5_lb6_$r --config 5 --steps 10
done
