export SPMV_LIB_PATH=exp/tma/libspmv.so
timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "hot or nzsplit_edges or configs_full" > gpurun_out/x_pytest.txt 2>&1
run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --no-cold --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
for r in 1 2; do run c3_tma_$r --config 3 --steps 40; done
unset SPMV_LIB_PATH
for r in 1 2; do run c3_def_$r --config 3 --steps 40; done
