run() { name=$1; shift; timeout 300 python bench.py --no-cpu --no-e2e --iters 0 "$@" > gpurun_out/x_$name.log 2>&1; }
timeout 900 python -m pytest tests -m gpu -x -q > gpurun_out/x_pytest.txt 2>&1
run c2_auto --config 2 --steps 50
run c5_auto --config 5 --steps 10
timeout 600 ncu --set full --import-source on --clock-control none -k regex:stream_kernel -s 2 -c 1 \
    -o gpurun_out/x_full_c2 python tools/prof_one.py --config 2 --reps 3 > gpurun_out/x_ncu_c2.txt 2>&1
