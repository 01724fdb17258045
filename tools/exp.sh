SPMV_STRESS_SEEDS=40 timeout 2400 python -m pytest tests/test_gpu_stress.py -m gpu -q > gpurun_out/x_pytest.txt 2>&1
