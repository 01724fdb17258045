import os
import subprocess
import sys

import pytest

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
if ROOT not in sys.path:
    sys.path.insert(0, ROOT)


def pytest_configure(config):
    config.addinivalue_line("markers", "gpu: needs a B200 (sm_100a) GPU")
    config.addinivalue_line("markers", "slow: full-size configs")
    # native libs: generators + oracle (CPU) and the product library (nvcc cross-compiles)
    need = [os.path.join(ROOT, p) for p in ("synthgen/libsynthgen.so", "oracle/liboracle.so",
                                           "paper_1711_05487_b200/libspmv.so")]
    if not all(os.path.exists(p) for p in need[:2]):
        subprocess.run(["make", "-C", ROOT, "-j8", "synthgen", "oracle"], check=True)
    if not os.path.exists(need[2]) and os.path.exists("/usr/local/cuda/bin/nvcc"):
        subprocess.run(["make", "-C", ROOT, "-j8", "spmv"], check=False)


def gpu_available():
    try:
        import torch
        return torch.cuda.is_available()
    except Exception:
        return False


def pytest_collection_modifyitems(config, items):
    if gpu_available():
        return
    skip = pytest.mark.skip(reason="no CUDA device")
    for it in items:
        if "gpu" in it.keywords:
            it.add_marker(skip)
