run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
for c in 2 3 4 5; do run c$c --config $c --steps 10; done
