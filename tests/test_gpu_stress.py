"""Seeded randomized GPU parity sweep: random row-length mixes (regular,
power-law, empty runs, a few very long rows), every variant, device and host
buffers (the host path of STREAM / nnz_split plans is the pipelined one),
checked against the oracle's per-row bound; empty rows exactly 0."""
import numpy as np
import pytest

import oracle
import synthgen as sg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
spmv = pytest.importorskip("paper_1711_05487_b200")


def _lengths(g, kind, n):
    if kind == "regular":
        return np.full(n, int(g.integers(1, 40)), np.int64) + g.integers(0, 2, n)
    if kind == "powerlaw":
        return np.minimum((g.pareto(1.1, n) * 2).astype(np.int64), 30000)
    if kind == "empty_runs":
        lens = np.zeros(n, np.int64)
        on = g.random(n) < 0.02
        lens[on] = g.integers(1, 300, on.sum())
        return lens
    # a few very long rows in short ones
    lens = g.integers(0, 12, n).astype(np.int64)
    lens[g.choice(n, 3, replace=False)] = g.integers(5000, 40000, 3)
    return lens


import os

_SEEDS = int(os.environ.get("SPMV_STRESS_SEEDS", "3"))  # more seeds for a longer sweep
CASES = [(seed, kind) for seed in range(_SEEDS) for kind in ("regular", "powerlaw", "empty_runs", "long")]


@pytest.mark.parametrize("seed,kind", CASES)
def test_random_matrices_all_variants(monkeypatch, seed, kind):
    monkeypatch.setenv("SPMV_HOST_PIPE_MIN_BYTES", "1")  # pipelined host path at test sizes
    g = np.random.default_rng(1000 + seed)
    n = int(g.integers(20000, 60000))
    lens = np.minimum(_lengths(g, kind, n), n)  # distinct columns: a row holds at most n
    m = sg.from_lengths(lens, n, g, sg.MODE_U11, sg.MODE_U11)
    yr = oracle.spmv(m.rowptr, m.colind, m.vals, m.x)
    s = oracle.absrow(m.rowptr, m.colind, m.vals, m.x)
    xd = torch.from_numpy(m.x).cuda()
    for v, extra in (("auto", {}), ("vector", {}), ("stream", {"seg": 0}), ("stream", {"seg": 1}), ("merge", {}),
                     ("split", {"l_split": 256}), ("split", {"l_split": 256, "long_mode": 3}), ("nnzsplit", {}),
                     ("nnzsplit", {"hot_x": 512})):
        kw = dict(extra)
        if v != "auto":
            kw["force_variant"] = v
        p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=n, **kw)
        yh = p.execute(m.x, np.full(n, np.nan))
        yd = torch.full((n,), float("nan"), dtype=torch.float64, device="cuda")
        p.execute(xd, yd)
        for y in (yh, yd.cpu().numpy()):
            bad = np.nonzero(~(np.abs(y - yr) <= 1e-12 * s))[0]
            assert bad.size == 0, (v, extra, bad[:5])
            assert np.all(y[lens == 0] == 0.0), (v, extra)
        p.destroy()


@pytest.mark.parametrize("seed", range(_SEEDS))
def test_random_banded_iteration_push(seed):
    """Random banded symmetric-pattern matrices (variable row lengths inside a
    band), 2-8 emulated shards: the iterated mode with the halo push (or the
    copies when a block's halo is not a prefix / suffix) vs the oracle."""
    g = np.random.default_rng(7000 + seed)
    n = int(g.integers(3000, 9000))
    bw = int(g.integers(5, 200))
    G = int(g.integers(2, 9))
    rows, cols = [], []
    for i in range(n):
        lo, hi = max(0, i - bw), min(n, i + bw + 1)
        k = int(g.integers(1, min(12, hi - lo) + 1))
        c = np.unique(np.concatenate([[i], g.choice(np.arange(lo, hi), k, replace=False)]))
        rows.append(np.full(c.size, i))
        cols.append(c)
    lens = np.array([r.size for r in rows], np.int64)
    cols = np.concatenate(cols).astype(np.int32)
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    vals = g.uniform(0.1, 1.0, cols.size)
    x0 = g.uniform(-1, 1, n)
    K = 25
    rc, xr, nur = oracle.power_iter(rp.astype(np.int32), cols, vals, x0, K)
    assert rc == 0
    for d16 in (0, 2):
        p = spmv.Plan(rp.astype(np.int32), cols, vals, ngpus=G, emulate_devices=1, force_variant="stream", d16=d16,
                      seg=0)
        xg, nug = p.iterate(x0, K)
        assert np.max(np.abs(xg - xr)) <= 1e-10 * np.max(np.abs(xr)), (seed, d16, p.info()["iter_push"])
        assert np.all(np.abs(nug - nur) <= 1e-12 * nur), (seed, d16)
        p.destroy()
