run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --no-cold --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
for t in 200 400 576 800 1100; do SPMV_ROW_TILE_MIN_NNZ=$t run c2_t$t --config 2 --steps 40; done
for t in 500 1100; do SPMV_ROW_TILE_MIN_NNZ=$t run c5_t$t --config 5 --steps 10; done
