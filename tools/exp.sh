timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/x_pytest.txt 2>&1
run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --no-cold --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
run c5 --config 5 --steps 5
SPMV_NO_STAGED_UPLOAD=1 run c5_nostage --config 5 --steps 5
run c3 --config 3 --steps 5
