"""World-size-2 gloo tests (CPU) of the one-process-per-GPU orchestration in
paper_1711_05487_b200/parallel.py: shard bounds, the rank-ordered norm
combine and the all-gather(v) of x blocks. The local steps are CPU stubs built
on the oracle (tests may use it; the product never does)."""
import math
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import oracle
import synthgen as sg


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _worker(rank, world, port, K, out_q, use_halo=False, cfg=5, scale=1.0):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_1711_05487_b200 as pkg
        from paper_1711_05487_b200 import parallel
        m = sg.config(cfg, small=True)
        rp = m.rowptr.astype(np.int64)
        b = pkg.shard_bounds(rp, world)
        b0, b1 = int(b[rank]), int(b[rank + 1])
        lrp = rp[b0:b1 + 1] - rp[b0]
        lci, lva = m.colind[rp[b0]:rp[b1]], m.vals[rp[b0]:rp[b1]] * scale
        P = 512
        def norm_step(pa, cnt, nn, nu):  # the spmv_norm_step contract (include/spmv.h)
            n = math.sqrt(math.fsum(pa.numpy()[:cnt]))
            nu.fill_(n / float(nn[0]) if float(nn[0]) > 0 else n)
            e = math.frexp(n)[1] - 1 if n > 0 else 0
            f = math.ldexp(1.0, -e) if abs(e) > 256 else 1.0
            nn[0], nn[1] = n * f, f  # the factor stays pending (applied by the next step / unit)

        def iter_step(x, y, p, nn, nu):  # spmv_iter_step: y = nn[1] * A x, partials, fused norm step
            f = float(nn[1]) if float(nn[1]) != 0 else 1.0
            y.copy_(torch.from_numpy(oracle.spmv(lrp, lci, lva, x.numpy()) * f))
            p.copy_(torch.tensor([float(np.sum(y.numpy()[q * y.numel() // P:(q + 1) * y.numel() // P] ** 2))
                                  for q in range(P)], dtype=torch.float64))
            if nu is not None:
                norm_step(p, P, nn, nu)

        steps = parallel.ShardSteps(
            iter_step=iter_step,
            norm_step=norm_step,
            unit=lambda y, nn, x: x.copy_(y * (float(nn[1]) if float(nn[1]) != 0 else 1.0) / nn[0]),
        )
        x = torch.from_numpy(m.x.copy())
        x2 = torch.full_like(x, float("nan"))
        nn = torch.zeros(2, dtype=torch.float64)
        pl = torch.empty(P, dtype=torch.float64)
        pa = torch.empty(world * P, dtype=torch.float64)
        nu = torch.empty(K, dtype=torch.float64)
        halo = None
        if use_halo:
            need = torch.tensor([int(lci.min()), int(lci.max()) + 1] if lci.size else [0, 0], dtype=torch.int64)
            needs = [torch.empty(2, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(needs, need)
            halo = parallel.halo_plan(b, [n.tolist() for n in needs], rank)
        parallel.iterate(dist, steps, b, rank, world, x, x2, pl, pa, nu, nn, K, halo=halo)
        if use_halo:  # only the range this rank reads is guaranteed: compare that, plus its own block
            lo, hi = int(lci.min()), int(lci.max()) + 1
            xs = np.full(x.numel(), np.nan)
            xs[lo:hi] = x.numpy()[lo:hi]
            xs[b0:b1] = x.numpy()[b0:b1]
            x = torch.from_numpy(xs)
        out_q.put((rank, b.tolist(), x.numpy().copy(), nu.numpy().copy()))
    finally:
        dist.destroy_process_group()


@pytest.mark.parametrize("world", [1, 2])
def test_sharded_power_iteration_gloo(world):
    K = 30
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = sg.config(5, small=True)
    rc, xr, nur = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, K)
    assert rc == 0
    res.sort()
    for rank, b, x, nu in res:
        assert b == oracle.shard_bounds(m.rowptr, world).tolist()
        assert np.max(np.abs(x - xr)) <= 1e-10 * np.max(np.abs(xr))
        assert np.all(np.abs(nu - nur) <= 1e-12 * nur)
    # every rank ends with the identical replica and identical nu (rank-ordered combine)
    for rank, b, x, nu in res[1:]:
        assert np.array_equal(x, res[0][2]) and np.array_equal(nu, res[0][3])



@pytest.mark.parametrize("world,cfg", [(2, 5), (3, 5), (4, 5), (3, 1)])
def test_halo_exchange_power_iteration_gloo(world, cfg):
    """Halo exchange (f2): each rank receives only the x ranges its rows read;
    the iterated result equals the oracle on every rank's own block and on the
    range it reads (banded 27-pt: small halos; random C1: whole blocks)."""
    K = 20
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, q, True, cfg)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = sg.config(cfg, small=True)
    rc, xr, nur = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, K)
    assert rc == 0
    for rank, b, x, nu in res:
        ok = ~np.isnan(x)
        assert ok.sum() >= b[rank + 1] - b[rank]
        assert np.max(np.abs(x[ok] - xr[ok])) <= 1e-10 * np.max(np.abs(xr))
        assert np.all(np.abs(nu - nur) <= 1e-12 * nur)


def test_halo_plan_pure():
    from paper_1711_05487_b200 import parallel
    bounds = [0, 10, 20, 30]
    needs = [(0, 12), (8, 23), (19, 30)]  # banded: each rank reads a little of its neighbours
    s0, r0 = parallel.halo_plan(bounds, needs, 0)
    s1, r1 = parallel.halo_plan(bounds, needs, 1)
    s2, r2 = parallel.halo_plan(bounds, needs, 2)
    assert s0 == [(1, 8, 10)] and r0 == [(1, 10, 12)]
    assert s1 == [(0, 10, 12), (2, 19, 20)] and r1 == [(0, 8, 10), (2, 20, 23)]
    assert s2 == [(1, 20, 23)] and r2 == [(1, 19, 20)]
    # every send has the matching receive on the peer
    plans = [parallel.halo_plan(bounds, needs, g) for g in range(3)]
    for g, (sends, _) in enumerate(plans):
        for peer, lo, hi in sends:
            assert (g, lo, hi) in plans[peer][1]
    assert parallel.halo_bytes(bounds, needs, 1) == 8 * (2 + 3)
    # a rank reading everything receives every other block whole
    s, r = parallel.halo_plan(bounds, [(0, 30)] * 3, 1)
    assert r == [(0, 0, 10), (2, 20, 30)]


@pytest.mark.parametrize("scale", [1e40, 1e-40])
def test_deferred_normalisation_rescale_gloo(scale):
    """Deferred normalisation across ranks (reading 25): the
    unnormalised iterate grows or shrinks by ~1e40 per step, so the exact
    power-of-two rescale fires every few iterations on every rank alike, and
    the exchanged blocks stay consistent; x and nu match the per-step oracle."""
    K, world = 25, 3
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, q, False, 5, scale)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = sg.config(5, small=True)
    rc, xr, nur = oracle.power_iter(m.rowptr, m.colind, m.vals * scale, m.x, K)
    assert rc == 0
    for rank, b, x, nu in res:
        assert np.all(np.isfinite(x)) and np.all(np.isfinite(nu))
        assert np.max(np.abs(x - xr)) <= 1e-10 * np.max(np.abs(xr))
        assert np.all(np.abs(nu - nur) <= 1e-12 * nur)
