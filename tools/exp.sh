run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-cold --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
for r in 1 2 3; do run c4_$r --config 4 --steps 10; done
run c2 --config 2 --steps 10
