timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "split or long or configs_full" > gpurun_out/x_pytest.txt 2>&1
run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
for r in 1 2; do run c4_$r --config 4 --steps 40; done
timeout 600 python tools/exp_parts.py --config 4 --variants auto --parts long > gpurun_out/x_parts.txt 2>&1
