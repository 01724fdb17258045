run() { name=$1; shift; timeout 300 python bench.py --no-cpu --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
for nb in 3 4 6 8; do SPMV_HOST_PIPE_BLOCKS=$nb run c2_nb$nb --config 2 --steps 30; done
for nb in 8 24 32; do SPMV_HOST_PIPE_BLOCKS=$nb run c5_nb$nb --config 5 --steps 10; done
