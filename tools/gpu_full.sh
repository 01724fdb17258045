# Round-end style GPU check on the box: build, pytest -m gpu, smoke(), default bench (results under gpurun_out/)
set -x
make -j32 > gpurun_out/make.log 2>&1 || tail -20 gpurun_out/make.log
( time timeout 2400 python -m pytest tests -x -q -m gpu --durations=25 ) > gpurun_out/gputest.log 2>&1; echo "pytest rc=$?"
timeout 300 python -c 'import __graft_entry__ as g; g.smoke()' > gpurun_out/smoke.log 2>&1; echo "smoke rc=$?"
timeout 600 python bench.py > gpurun_out/bench_default.json 2> gpurun_out/bench_default.err; echo "bench rc=$?"
tail -3 gpurun_out/gputest.log; tail -2 gpurun_out/smoke.log; cat gpurun_out/bench_default.json | head -c 600
