"""GPU test of the distributed iterated mode (parallel.py + libspmv building
blocks) on one GPU with a world-size-1 NCCL process group."""
import os
import socket

import numpy as np
import pytest

import oracle
import synthgen as sg

pytestmark = pytest.mark.gpu
torch = pytest.importorskip("torch")


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def test_native_distributed_iteration_world1():
    import torch.distributed as dist
    import paper_1711_05487_b200 as spmv
    from paper_1711_05487_b200 import parallel
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(_port())
    torch.cuda.set_device(0)
    dist.init_process_group("nccl", rank=0, world_size=1, device_id=torch.device("cuda", 0))
    try:
        m = sg.config(5, small=True)
        K = 100
        plan = spmv.Plan(m.rowptr, m.colind, m.vals)
        b = spmv.shard_bounds(m.rowptr, 1)
        P = spmv.norm_partial_count()
        x = torch.from_numpy(m.x.copy()).cuda()
        x2 = torch.empty(m.n, dtype=torch.float64, device="cuda")
        nn = torch.zeros(2, dtype=torch.float64, device="cuda")
        pl = torch.empty(P, dtype=torch.float64, device="cuda")
        pa = torch.empty(P, dtype=torch.float64, device="cuda")
        nu = torch.empty(K, dtype=torch.float64, device="cuda")
        st = torch.cuda.ExternalStream(plan.stream())
        with torch.cuda.stream(st):
            parallel.iterate(dist, parallel.native_steps(plan), b, 0, 1, x, x2, pl, pa, nu, nn, K)
        torch.cuda.synchronize()
        rc, xr, nur = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, K)
        xg, nug = x.cpu().numpy(), nu.cpu().numpy()
        assert np.max(np.abs(xg - xr)) <= 1e-10 * np.max(np.abs(xr))
        assert np.all(np.abs(nug - nur) <= 1e-12 * nur)
        # same answer as the in-library iterate (same kernels, same order)
        xi, nui = plan.iterate(m.x, K)
        assert np.array_equal(xi, xg) and np.array_equal(nui, nug)
    finally:
        dist.destroy_process_group()


def test_bench_under_torchrun_world1():
    # the launch the driver uses for N > 1 (torchrun, one process per GPU,
    # NCCL), at world size 1 on the one GPU: one JSON line, max-over-ranks
    # timing, the iterated mode through parallel.iterate
    import json
    import subprocess
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", "--nproc-per-node", "1", "--master-addr",
           "127.0.0.1", "--master-port", str(_port()), os.path.join(root, "bench.py"), "--gpus", "1", "--steps", "3",
           "--warmup", "3", "--config", "2", "--no-cpu", "--no-paper-runs", "--iters", "20"]
    out = subprocess.run(cmd, capture_output=True, text=True, timeout=600, cwd=root)
    assert out.returncode == 0, out.stderr[-2000:]
    lines = [l for l in out.stdout.splitlines() if l.startswith("{")]
    assert len(lines) == 1
    d = json.loads(lines[0])
    assert d["n_gpus"] == 1 and d["value"] > 0 and d["gpu_launches"] > 0
    assert d["config"]["d16"] == 2 and d["iterated"]["iters_timed"] == 20
