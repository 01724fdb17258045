timeout 1500 python -m pytest tests -m gpu -x -q > gpurun_out/x_pytest.txt 2>&1
