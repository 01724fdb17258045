run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
for r in 1 2; do
run c4_tpw4_$r --config 4 --steps 40
for v in tpw3 tpw5 tpw6 tpw4rg3 tpw4rg1; do SPMV_LIB_PATH=exp/$v/libspmv.so run c4_${v}_$r --config 4 --steps 40; done
done
timeout 900 python -m pytest tests -m gpu -x -q -k "split or long or configs_full or nzsplit_edges" > gpurun_out/x_pytest.txt 2>&1
