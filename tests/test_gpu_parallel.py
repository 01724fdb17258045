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


class _HostDist:
    """Collectives of parallel.iterate over gloo for ranks sharing one GPU
    (NCCL refuses two ranks on one device): device tensors go through the
    host, on the current (plan) stream, so each rank's contribution waits for
    its kernels exactly as an NCCL all-gather on that stream would."""

    def __init__(self, dist):
        self.d = dist

    def all_gather_into_tensor(self, out, inp, group=None):
        h = torch.empty(out.numel(), dtype=out.dtype)
        self.d.all_gather_into_tensor(h, inp.cpu(), group=group)
        out.copy_(h)

    def all_gather_object(self, lst, obj, group=None):
        self.d.all_gather_object(lst, obj, group=group)


def _push_worker(rank, world, port, K, d16, out_q):
    import torch.distributed as dist
    import paper_1711_05487_b200 as spmv
    from paper_1711_05487_b200 import parallel
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        torch.cuda.set_device(0)
        m = sg.stencil(24, 27, rp64=True, x_seed=5)
        rp = m.rowptr.astype(np.int64)
        b = spmv.shard_bounds(rp, world)
        b0, b1 = int(b[rank]), int(b[rank + 1])
        lrp = rp[b0:b1 + 1] - rp[b0]
        lci, lva = m.colind[rp[b0]:rp[b1]], m.vals[rp[b0]:rp[b1]]
        plan = spmv.Plan(lrp, np.ascontiguousarray(lci), np.ascontiguousarray(lva), n_cols=m.n,
                         force_variant="stream", d16=d16)
        assert plan.push_capable()
        ra, rb = plan.replicas()
        x, x2 = parallel.device_view(ra, m.n, "cuda:0"), parallel.device_view(rb, m.n, "cuda:0")
        need = torch.tensor([int(lci.min()), int(lci.max()) + 1], dtype=torch.int64)
        needs = [torch.empty(2, dtype=torch.int64) for _ in range(world)]
        dist.all_gather(needs, need)
        layout = parallel.push_plan(b, [n.tolist() for n in needs], world)
        assert layout is not None
        hd = _HostDist(dist)
        push = parallel.open_push(hd, plan, layout, rank, world)
        P = spmv.norm_partial_count()
        nn = torch.zeros(2, dtype=torch.float64, device="cuda")
        pl = torch.empty(P, dtype=torch.float64, device="cuda")
        pa = torch.empty(world * P, dtype=torch.float64, device="cuda")
        nu = torch.empty(K, dtype=torch.float64, device="cuda")
        steps = parallel.native_steps(plan)
        with steps.stream():
            x2.fill_(float("nan"))
            for _ in range(2):  # the second call's first pushes must wait for the peers' unit()
                x.copy_(torch.from_numpy(m.x))
                parallel.iterate(hd, steps, b, rank, world, x, x2, pl, pa, nu, nn, K, push=push)
        torch.cuda.synchronize()
        xs = np.full(m.n, np.nan)
        lo, hi = int(lci.min()), int(lci.max()) + 1
        xh = x.cpu().numpy()
        xs[lo:hi] = xh[lo:hi]
        xs[b0:b1] = xh[b0:b1]
        out_q.put((rank, b.tolist(), xs, nu.cpu().numpy(), plan.info()["sel"]["d16"]))
        dist.barrier()  # no rank unmaps a replica a peer may still store into
        plan.destroy()
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("d16", [2, 0])
def test_halo_push_ipc_two_processes(d16):
    """Halo push across processes (spmv_plan_replicas / spmv_ipc_export /
    spmv_ipc_open / spmv_iter_step_push via parallel.open_push + iterate): two
    ranks, each its own process and CUDA context on the one GPU, each kernel
    storing the rows its neighbour reads into the neighbour's replica through
    a CUDA IPC mapping; no kernel waits on another (the gloo all-gather of the
    partials orders them). x and nu vs the oracle's power iteration, D8 and
    int32 stream kernels."""
    import torch.multiprocessing as mp
    K, world = 30, 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _port()
    procs = [ctx.Process(target=_push_worker, args=(r, world, port, K, d16, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=120)
        assert p.exitcode == 0
    m = sg.stencil(24, 27, rp64=True, x_seed=5)
    rc, xr, nur = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, K)
    assert rc == 0
    for rank, b, x, nu, d in res:
        assert d == d16
        ok = ~np.isnan(x)
        assert ok.sum() > b[rank + 1] - b[rank]  # own block + the pushed halo
        assert np.max(np.abs(x[ok] - xr[ok])) <= 1e-10 * np.max(np.abs(xr))
        assert np.all(np.abs(nu - nur) <= 1e-12 * nur)
