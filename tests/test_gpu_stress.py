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
                     ("split", {"l_split": 256}), ("nnzsplit", {}), ("nnzsplit", {"hot_x": 512})):
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
