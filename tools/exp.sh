timeout 900 python -m pytest tests/test_gpu_parity.py -m gpu -x -q -k "pipelined or row_count or execute_norm" > gpurun_out/x_pytest.txt 2>&1
