"""World-size-2 gloo tests (CPU) of the one-process-per-GPU orchestration in
paper_1711_05487_b200/parallel.py: shard bounds, the rank-ordered norm
combine and the all-gather(v) of x blocks. The local steps are CPU stubs built
on the oracle (tests may use it; the product never does)."""
import ctypes
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


class _ShmPlan:
    """CPU stand-in for the plan's replica / IPC calls (spmv_plan_replicas,
    spmv_ipc_export, spmv_ipc_open): the replicas are shared-memory files, a
    "handle" is the file name, opening one maps the peer's file."""

    def __init__(self, tag, rank, n):
        self.n, self.maps = n, []
        self.files = ["/dev/shm/spmv_push_%s_%d_%s" % (tag, rank, w) for w in "AB"]
        self.rep = [torch.from_file(f, shared=True, size=n, dtype=torch.float64) for f in self.files]

    def replicas(self):
        return self.rep[0].data_ptr(), self.rep[1].data_ptr()

    def ipc_export(self, ptr):
        f = self.files[[r.data_ptr() for r in self.rep].index(ptr)]
        return f.encode().ljust(64, b"\0")

    def ipc_open(self, handle):
        t = torch.from_file(handle.rstrip(b"\0").decode(), shared=True, size=self.n, dtype=torch.float64)
        self.maps.append(t)
        return t.data_ptr()

    def close(self):
        for f in self.files:
            os.unlink(f)


def _store(ptr, rows):
    """Peer store of the push stub: rows (numpy) at the device-pointer stand-in."""
    if ptr is not None and rows.size:
        np.ctypeslib.as_array((ctypes.c_double * rows.size).from_address(ptr))[:] = rows


def _worker(rank, world, port, K, out_q, use_halo=False, cfg=5, scale=1.0, use_push=False):
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

        def iter_step_push(x, y, p, nn, lo, lo_end, hi, hi_begin):  # spmv_iter_step_push
            iter_step(x, y, p, nn, None)
            yv = y.numpy()
            _store(lo, yv[:lo_end])
            if hi is not None:
                _store(hi + 8 * hi_begin, yv[hi_begin:])

        steps = parallel.ShardSteps(
            iter_step=iter_step,
            iter_step_push=iter_step_push,
            norm_step=norm_step,
            unit=lambda y, nn, x: x.copy_(y * (float(nn[1]) if float(nn[1]) != 0 else 1.0) / nn[0]),
        )
        shm = None
        if use_push:  # the iterated mode runs on the plan's replicas, which the peers map
            shm = _ShmPlan(port, rank, m.x.size)
            x, x2 = shm.rep
            x.copy_(torch.from_numpy(m.x))
            x2.fill_(float("nan"))
        else:
            x = torch.from_numpy(m.x.copy())
            x2 = torch.full_like(x, float("nan"))
        nn = torch.zeros(2, dtype=torch.float64)
        pl = torch.empty(P, dtype=torch.float64)
        pa = torch.empty(world * P, dtype=torch.float64)
        nu = torch.empty(K, dtype=torch.float64)
        halo, push = None, None
        if use_halo or use_push:
            need = torch.tensor([int(lci.min()), int(lci.max()) + 1] if lci.size else [0, 0], dtype=torch.int64)
            needs = [torch.empty(2, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(needs, need)
            needs = [n.tolist() for n in needs]
            if use_push:
                layout = parallel.push_plan(b, needs, world)
                assert layout is not None  # banded row blocks
                push = parallel.open_push(dist, shm, layout, rank, world)
            else:
                halo = parallel.halo_plan(b, needs, rank)
        for _ in range(2 if use_push else 1):  # push: a second call starts while peers may still finish the first
            nn.zero_()
            if use_push:
                x.copy_(torch.from_numpy(m.x))
            parallel.iterate(dist, steps, b, rank, world, x, x2, pl, pa, nu, nn, K, halo=halo, push=push)
        if use_push:
            dist.barrier()
            shm.close()
        if use_halo or use_push:  # only the range this rank reads is guaranteed: compare that, plus its own block
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


@pytest.mark.parametrize("world", [2, 3, 4])
def test_halo_push_power_iteration_gloo(world):
    """Halo push (f2, the exchange fused into the SpMV step): each rank's step
    stores the rows its neighbours read straight into their replicas (shared
    memory standing in for the CUDA IPC mappings), no exchange runs, and the
    all-gather of the partials orders the stores; x and nu match the oracle on
    every rank's block and read range, over two back-to-back calls."""
    K = 20
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, K, q, False, 5, 1.0, True)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    m = sg.config(5, small=True)
    rc, xr, nur = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, K)
    assert rc == 0
    for rank, b, x, nu in res:
        ok = ~np.isnan(x)
        assert ok.sum() >= b[rank + 1] - b[rank]
        assert np.max(np.abs(x[ok] - xr[ok])) <= 1e-10 * np.max(np.abs(xr))
        assert np.all(np.abs(nu - nur) <= 1e-12 * nur)


def test_push_plan_pure():
    """push_plan (the in-process rule of api.cu prepare_push): banded blocks
    push prefixes down and suffixes up, the same rows halo_plan sends; a rank
    read by two lower ranks, or a read range that is not a prefix / suffix of
    the block, disables the push for everyone."""
    from paper_1711_05487_b200 import parallel
    bounds = [0, 10, 20, 30]
    needs = [(0, 12), (8, 23), (19, 30)]
    lay = parallel.push_plan(bounds, needs, 3)
    assert lay == [(-1, 0, 1, 8), (0, 2, 2, 9), (1, 3, -1, 10)]
    for g, (lo_peer, lo_end, hi_peer, hi_begin) in enumerate(lay):
        sends = parallel.halo_plan(bounds, needs, g)[0]
        mine = sorted([(lo_peer, bounds[g], bounds[g] + lo_end)] * (lo_peer >= 0) +
                      [(hi_peer, bounds[g] + hi_begin, bounds[g + 1])] * (hi_peer >= 0))
        assert sorted(sends) == mine
    assert parallel.push_plan(bounds, [(0, 12), (8, 23), (5, 30)], 3) is None   # rank 2 reads all of rank 1
    assert parallel.push_plan(bounds, [(0, 12), (8, 23), (0, 30)], 3) is None   # rank 0 read by two ranks
    assert parallel.push_plan(bounds, [(0, 10), (10, 20), (20, 30)], 3) == [(-1, 0, -1, 10), (-1, 0, -1, 10),
                                                                           (-1, 0, -1, 10)]  # block diagonal
