timeout 1200 python -m pytest tests -m gpu -x -q -k "d16 or stream or dyadic" > gpurun_out/x_pytest.txt 2>&1
