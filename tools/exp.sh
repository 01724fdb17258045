timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/x_pytest.txt 2>&1
run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --no-cold --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
for r in 1 2; do run c2_$r --config 2 --steps 40; SPMV_NO_CW6=1 run c2_cw4_$r --config 2 --steps 40; done
run c5 --config 5 --steps 10
