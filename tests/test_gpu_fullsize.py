"""Full-size parity of the headline config C5 (BJ.configs[4]: 27-point
stencil on 384^3, N = 56,623,104, nnz = 1,520,875,000, int64 rowptr) in the
launch configuration bench.py times (the feature-guided plan: STREAM + D8).

* every row of y = A x against the oracle's row-parallel form (bitwise equal
  to the serial oracle) under the per-row bound;
* dyadic x (k/1024): every product and partial sum is exact in any order, so
  y must be bit-equal on every row -- sensitive to any wrong column index;
* the 100-iteration x <- Ax/||Ax|| run (BJ.configs[5]) against
  oracle_power_iter, with the stepwise per-row bound at k in {0, 1, 49, 99}
  and the end-to-end tolerances of SURVEY 8(c3) #21;
* forced non-default variants on the same matrix, sampled rows.
"""
import numpy as np
import pytest

import oracle
import synthgen as sg

pytestmark = [pytest.mark.gpu, pytest.mark.slow]
torch = pytest.importorskip("torch")
spmv = pytest.importorskip("paper_1711_05487_b200")

TOL = 1e-12
N3 = 384


@pytest.fixture(scope="module")
def c5():
    return sg.config(5)


def _all_rows_bound(m, x, y):
    yr, _ = oracle.spmv_omp(m.rowptr, m.colind, m.vals, x, 0)
    s = oracle.absrow(m.rowptr, m.colind, m.vals, x)
    bad = np.nonzero(np.abs(y - yr) > TOL * s)[0]
    assert bad.size == 0, f"{bad.size} rows over the bound, first {bad[:5]}"
    return yr


def test_c5_every_row_and_dyadic(c5):
    m = c5
    p = spmv.Plan(m.rowptr, m.colind, m.vals)
    info = p.info()
    assert info["feat"]["nnz"] == 1520875000 and info["feat"]["n_deltas"] == 15
    assert info["kernel_bytes"] == 8 * m.nnz + m.n + 8 * (info["n_tiles"] + 1) + 16 * m.n
    assert info["variant"] == "stream" and info["sel"]["d16"] == 2  # the benchmarked configuration
    xd = torch.from_numpy(m.x).cuda()
    yd = torch.empty(m.n, dtype=torch.float64, device="cuda")
    p.execute(xd, yd)
    torch.cuda.synchronize()
    _all_rows_bound(m, m.x, yd.cpu().numpy())
    # dyadic x: exact in every summation order -> bit-equal on all 56.6M rows
    xq = np.random.default_rng(8).integers(-1024, 1025, m.n) / 1024.0
    p.execute(torch.from_numpy(xq).cuda(), yd)
    torch.cuda.synchronize()
    yq, _ = oracle.spmv_omp(m.rowptr, m.colind, m.vals, xq, 0)
    assert np.array_equal(yd.cpu().numpy(), yq)
    # plan structures at full size: the 27 row patterns (DESIGN.md reading
    # 31) and every row's pattern equal the oracle's encoding, and the
    # oracle's decoder gives colind back from the device's patterns
    assert info["d8_patterns"] == 27
    ids, lens, ofs = oracle.pat_encode(m.rowptr, m.colind)
    pid, pl, po = p.export("pat_ids"), p.export("pat_len"), p.export("pat_ofs")
    assert np.array_equal(pid, ids) and np.array_equal(pl, lens) and np.array_equal(po, ofs)
    assert np.array_equal(oracle.pat_decode(pid, pl, po), m.colind)
    p.destroy()


def test_c5_power_iteration_100(c5):
    m = c5
    K = 100
    p = spmv.Plan(m.rowptr, m.colind, m.vals)
    xg, nug = p.iterate(m.x, K)
    rc, xr, nur = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, K, nthreads=0)
    assert rc == 0
    # SURVEY 8(c3) #21 end-to-end tolerances
    assert np.max(np.abs(xg - xr)) <= 1e-10 * np.max(np.abs(xr))
    assert np.all(np.abs(nug - nur) <= 1e-12 * nur)
    # nu_k nondecreasing for k >= 1 (symmetric A) and below lambda_max (closed form)
    assert np.all(np.diff(nug[1:]) >= -1e-13 * nug[1:-1])
    assert nug[-1] <= 35.99900125724772 * (1 + 1e-12)
    # stepwise: y_k from the GPU's own x_k obeys the per-row bound on every row
    for k in (0, 1, 49, 99):
        xk = m.x if k == 0 else p.iterate(m.x, k)[0]
        yk = p.execute(xk)
        _all_rows_bound(m, xk, yk)
    p.destroy()


@pytest.mark.parametrize("variant,extra", [("stream", {"d16": 0}), ("nnzsplit", {}), ("vector", {})])
def test_c5_forced_variants_sampled(c5, variant, extra):
    m = c5
    p = spmv.Plan(m.rowptr, m.colind, m.vals, force_variant=variant, **extra)
    y = p.execute(m.x)
    g = np.random.default_rng(1)
    rows = np.unique(np.concatenate([g.integers(0, m.n, 300000), np.arange(3000), m.n - 1 - np.arange(3000)]))
    yr = oracle.spmv_rows(m.rowptr, m.colind, m.vals, m.x, rows)
    s = oracle.absrow(m.rowptr, m.colind, m.vals, m.x, rows)
    assert np.all(np.abs(y[rows] - yr) <= TOL * s)
    # A*1 closed form (exact in any order) on every row: {0, 9, 15, 19} by boundary class
    y1 = p.execute(np.ones(m.n))
    i = np.arange(m.n, dtype=np.int64)
    prod = np.ones(m.n)
    for c in (i % N3, (i // N3) % N3, i // (N3 * N3)):
        prod *= 3 - (c == 0).astype(float) - (c == N3 - 1)
    assert np.array_equal(y1, 27.0 - prod)
    p.destroy()


def test_c5_emulated_shards(c5):
    # the in-process multi-shard path at full size (2 shards on one GPU:
    # nnz-balanced row blocks, x replicated, interior-first iteration with
    # halo peer copies): every row of y, and 10 iterations vs the oracle
    m = c5
    p = spmv.Plan(m.rowptr, m.colind, m.vals, ngpus=2, emulate_devices=1)
    info = p.info()
    assert info["shard_bounds"] == oracle.shard_bounds(m.rowptr, 2).tolist()
    assert info["sel"]["d16"] == 2
    _all_rows_bound(m, m.x, p.execute(m.x))
    K = 10
    xg, nug = p.iterate(m.x, K)
    rc, xr, nur = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, K, nthreads=0)
    assert rc == 0
    assert np.max(np.abs(xg - xr)) <= 1e-10 * np.max(np.abs(xr))
    assert np.all(np.abs(nug - nur) <= 1e-12 * nur)
    p.destroy()
