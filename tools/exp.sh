timeout 900 python -m pytest tests -m gpu -x -q -k "iterat or parallel" > gpurun_out/x_pytest.txt 2>&1
run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e "$@" > gpurun_out/x_$name.log 2>&1; }
run c5 --config 5 --steps 5
run c2 --config 2 --steps 20
