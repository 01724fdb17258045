"""Maximum sizes: a matrix with more nonzeros than int32 can index.

27-point stencil on 440^3 (N = 85,184,000 rows, nnz = (3*440-2)^3 = 2,289,529,432 > 2^31,
int64 rowptr, int32 colind): every nonzero offset past 2^31 - 1 goes through
the kernels' 64-bit index arithmetic (tile starts, TMA source offsets, warp
tile bases, carries), which C5 (1.52e9 nonzeros) never exercises.

* the feature-guided plan (STREAM + D8, the benchmarked configuration) with
  dyadic x (k/1024): every product and partial sum is exact in any order, so
  y must be bit-equal to the oracle on all 85M rows;
* forced int32-colind STREAM, nnz_split, csr_vector and merge-path plans: A*1 against
  its closed form on every row (exact in any order) and a dyadic x on rows
  sampled across the whole range, past the 2^31-th nonzero included.
"""
import numpy as np
import pytest

import oracle
import synthgen as sg

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")
spmv = pytest.importorskip("paper_1711_05487_b200")

N3 = 440


@pytest.fixture(scope="module")
def big():
    m = sg.stencil(N3, 27, rp64=True, x_seed=11)
    assert m.colind.size > 2 ** 31
    xq = np.random.default_rng(9).integers(-1024, 1025, m.n) / 1024.0
    return m, xq


def _ones_closed_form(n):
    i = np.arange(n, dtype=np.int64)
    prod = np.ones(n)
    for c in (i % N3, (i // N3) % N3, i // (N3 * N3)):
        prod *= 3 - (c == 0).astype(float) - (c == N3 - 1)
    return 27.0 - prod


def test_beyond_int32_auto_d8_dyadic_every_row(big):
    m, xq = big
    p = spmv.Plan(m.rowptr, m.colind, m.vals)
    info = p.info()
    assert info["feat"]["nnz"] == m.colind.size
    assert info["variant"] == "stream" and info["sel"]["d16"] == 2
    xd = torch.from_numpy(xq).cuda()
    yd = torch.empty(m.n, dtype=torch.float64, device="cuda")
    p.execute(xd, yd)
    torch.cuda.synchronize()
    yq, _ = oracle.spmv_omp(m.rowptr, m.colind, m.vals, xq, 0)
    assert np.array_equal(yd.cpu().numpy(), yq)
    # host x and y: the pipelined host execute (tile-range launches per x chunk)
    assert np.array_equal(p.execute(np.ones(m.n)), _ones_closed_form(m.n))
    p.destroy()


@pytest.mark.parametrize("variant,extra", [("stream", {"d16": 0}), ("nnzsplit", {}), ("vector", {}),
                                           ("merge", {})])
def test_beyond_int32_forced_variants(big, variant, extra):
    m, xq = big
    p = spmv.Plan(m.rowptr, m.colind, m.vals, force_variant=variant, **extra)
    assert p.info()["variant"] == variant
    assert np.array_equal(p.execute(np.ones(m.n)), _ones_closed_form(m.n))
    # dyadic x on sampled rows: the first rows, the rows around the 2^31-th
    # nonzero, the last rows and a uniform sample
    r31 = int(np.searchsorted(m.rowptr, 2 ** 31, side="right")) - 1
    g = np.random.default_rng(3)
    rows = np.unique(np.concatenate([np.arange(2000), r31 - 2000 + np.arange(4000), m.n - 1 - np.arange(2000),
                                     g.integers(0, m.n, 200000)]))
    y = p.execute(xq)
    yr = oracle.spmv_rows(m.rowptr, m.colind, m.vals, xq, rows)
    assert np.array_equal(y[rows], yr)
    p.destroy()
