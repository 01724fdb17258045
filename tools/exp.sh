run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
for r in 1 2; do
run c3_pf_$r --config 3 --steps 40
SPMV_LIB_PATH=exp/pf0/libspmv.so run c3_nopf_$r --config 3 --steps 40
done
run c5nz_pf --config 5 --steps 5 --variant nnzsplit
SPMV_LIB_PATH=exp/pf0/libspmv.so run c5nz_nopf --config 5 --steps 5 --variant nnzsplit
run c4nz_pf --config 4 --steps 30 --variant nnzsplit
SPMV_LIB_PATH=exp/pf0/libspmv.so run c4nz_nopf --config 4 --steps 30 --variant nnzsplit
