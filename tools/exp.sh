run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/x_pytest.txt 2>&1
run c3 --config 3 --steps 30
run c4 --config 4 --steps 30
run c2nz --config 2 --steps 30 --variant nnzsplit
run c5nz --config 5 --steps 10 --variant nnzsplit
SPMV_PLAN_TRACE=1 python tools/dbg_reuse.py > gpurun_out/x_dbg.txt 2>&1
