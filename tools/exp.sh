run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
run c2_base --config 2 --steps 50
run c2_d16 --config 2 --steps 50 --d16 1
run c2_nz --config 2 --steps 50 --variant nnzsplit --hot 0
run c2_vec4 --config 2 --steps 50 --variant vector --vs 4
run c2_vec8 --config 2 --steps 50 --variant vector --vs 8
run c5_nz --config 5 --steps 10 --variant nnzsplit --hot 0
run c5_d16 --config 5 --steps 10 --d16 1
