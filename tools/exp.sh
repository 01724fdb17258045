run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --no-cold --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
for r in 1 2; do
run c3_cg_$r --config 3 --steps 40
SPMV_LIB_PATH=exp/na/libspmv.so run c3_na_$r --config 3 --steps 40
run c4_cg_$r --config 4 --steps 40
SPMV_LIB_PATH=exp/na/libspmv.so run c4_na_$r --config 4 --steps 40
done
