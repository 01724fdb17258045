timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "hot or nzsplit or configs_full or suite" > gpurun_out/x_pytest.txt 2>&1
run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
for r in 1 2; do
run c3_cl2_$r --config 3 --steps 40
SPMV_HOT_CLUSTER=0 run c3_cl1_$r --config 3 --steps 40
done
for h in 20000 24576 28672; do run c3_h$h --config 3 --steps 40 --hot $h; done
