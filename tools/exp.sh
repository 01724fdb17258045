timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pipelined" > gpurun_out/x_pytest.txt 2>&1
run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-cold --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
run c3 --config 3 --steps 10
SPMV_NO_HOST_PIPE=1 run c3_nopipe --config 3 --steps 10
for nb in 2 4 8; do SPMV_HOST_PIPE_BLOCKS=$nb run c3_nb$nb --config 3 --steps 10; done
