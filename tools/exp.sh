timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/x_pytest.txt 2>&1
timeout 300 python -c "import __graft_entry__ as g; g.smoke()" > gpurun_out/x_smoke.txt 2>&1
