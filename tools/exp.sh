timeout 1200 python -m pytest tests -m gpu -x -q > gpurun_out/x_pytest.txt 2>&1
run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
run c3 --config 3 --steps 40
timeout 600 python tools/exp_parts.py --config 3 --variants auto --parts long > gpurun_out/x_parts_c3.txt 2>&1
