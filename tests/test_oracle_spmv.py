"""Pins for the oracle's SpMV and iterated mode (CPU only).

Each check pins the oracle to something other than itself: dense brute force,
closed forms, exact rational arithmetic, scipy, eigvalsh. Citations: P:n =
PAPER.md line, S:n = SPEC.md line, SURVEY 8(c4) = the pin table.
"""
import json
import os
from fractions import Fraction

import numpy as np
import pytest
import scipy.sparse as sp

import oracle
import synthgen as sg

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def dense_of(m):
    """Dense matrix built from CSR triplets with numpy scatter (independent of the oracle)."""
    rp = m.rowptr.astype(np.int64)
    rows = np.repeat(np.arange(m.n), np.diff(rp))
    A = np.zeros((m.n, m.x.size))
    np.add.at(A, (rows, m.colind), m.vals)
    return A


def small_cases(val_mode=sg.MODE_U11, x_mode=sg.MODE_U11, seed=0):
    cases = [c for c in sg.small_suite(seed, val_mode, x_mode) if c[1].n * c[1].x.size <= 4e7]
    return cases


@pytest.mark.parametrize("name,m", small_cases())
def test_spmv_vs_dense_bruteforce(name, m):
    # brute-force dense matvec on tiny matrices
    A = dense_of(m)
    y = oracle.spmv(m.rowptr, m.colind, m.vals, m.x)
    yd = A @ m.x
    bound = np.abs(A) @ np.abs(m.x)
    assert np.all(np.abs(y - yd) <= 1e-12 * bound)
    # the oracle's own bound denominator agrees with the dense one
    s = oracle.absrow(m.rowptr, m.colind, m.vals, m.x)
    assert np.allclose(s, bound, rtol=1e-12, atol=0)


def test_identity_spec_example():
    g = GOLD["spmv_identity"]  # S:196 identity . [3,4] -> [3,4]
    y = oracle.spmv(np.array([0, 1, 2]), np.array([0, 1], np.int32), np.array([1.0, 1.0]), np.array(g["x"]))
    assert y.tolist() == g["y"]


def test_empty_rows_exact_zero():
    # a row with no nonzeros gives exactly 0.0
    rp = np.array([0, 0, 2, 2, 3])
    y = oracle.spmv(rp, np.array([1, 3, 0], np.int32), np.array([1.5, -2.0, 4.0]), np.array([1.0, 2, 3, 4]))
    assert y[0] == 0.0 and y[2] == 0.0 and y[1] == 1.5 * 2 - 8.0 and y[3] == 4.0


def test_diagonal_exact():
    # y_i = d_i x_i exactly (single product per row)
    g = np.random.default_rng(1)
    n = 5000
    d, x = g.standard_normal(n), g.standard_normal(n)
    y = oracle.spmv(np.arange(n + 1), np.arange(n, dtype=np.int32), d, x)
    assert np.array_equal(y, d * x)


@pytest.mark.parametrize("c", [1, 2, 4])
def test_unit_vector_gives_column(c):
    # A e_j equals column j of A bit-exactly
    m = sg.config(c, small=True)
    csc = sp.csr_matrix((m.vals, m.colind, m.rowptr.astype(np.int64)), shape=(m.n, m.n)).tocsc()
    for j in [0, 1, m.n // 3, m.n - 1]:
        e = np.zeros(m.n); e[j] = 1.0
        y = oracle.spmv(m.rowptr, m.colind, m.vals, e)
        col = np.zeros(m.n)
        col[csc.indices[csc.indptr[j]:csc.indptr[j + 1]]] = csc.data[csc.indptr[j]:csc.indptr[j + 1]]
        assert np.array_equal(y, col)


def missing_neighbours(n, pts):
    """Closed form of (stencil) * ones from grid coordinates."""
    i = np.arange(n ** 3)
    c = [i % n, (i // n) % n, i // (n * n)]
    if pts == 7:
        return sum((ci == 0).astype(float) + (ci == n - 1) for ci in c)
    prod = np.ones(i.size)
    for ci in c:
        prod *= 3 - (ci == 0).astype(float) - (ci == n - 1)
    return 27.0 - prod


@pytest.mark.parametrize("n,pts", [(2, 7), (5, 7), (24, 7), (2, 27), (5, 27), (20, 27)])
def test_stencil_times_ones_closed_form(n, pts):
    m = sg.stencil(n, pts, rp64=(pts == 27))
    y = oracle.spmv(m.rowptr, m.colind, m.vals, np.ones(m.n))
    exp = missing_neighbours(n, pts)
    assert np.array_equal(y, exp)
    vals = set(np.unique(y).tolist())
    if n >= 3:
        assert vals == ({0.0, 1.0, 2.0, 3.0} if pts == 7 else {0.0, 9.0, 15.0, 19.0})
    # structure closed forms: nnz = 7n^3 - 6n^2 and (3n-2)^3
    assert m.nnz == (7 * n ** 3 - 6 * n ** 2 if pts == 7 else (3 * n - 2) ** 3)


@pytest.mark.parametrize("name,m", small_cases(sg.MODE_DYADIC, sg.MODE_DYADIC, seed=3))
def test_dyadic_exact_vs_rational(name, m):
    # dyadic k/1024 inputs make every summation order exact;
    # compare with exact integer arithmetic.
    kv = np.rint(m.vals * 1024).astype(np.int64)
    kx = np.rint(m.x * 1024).astype(np.int64)
    rp = m.rowptr.astype(np.int64)
    prods = kv * kx[m.colind]
    exact = np.add.reduceat(np.append(prods, 0), rp[:-1]) if m.nnz else np.zeros(m.n, np.int64)
    exact = np.where(np.diff(rp) > 0, exact, 0)
    y = oracle.spmv(m.rowptr, m.colind, m.vals, m.x)
    assert np.array_equal(y, exact.astype(np.float64) / 2.0 ** 20)
    # spot check one row with Fraction arithmetic
    i = int(np.argmax(np.diff(rp)))
    fr = sum(Fraction(int(a), 1024) * Fraction(int(b), 1024) for a, b in zip(kv[rp[i]:rp[i + 1]], kx[m.colind[rp[i]:rp[i + 1]]]))
    assert Fraction(y[i]) == fr


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_scipy_and_neumaier_selfcheck_small_configs(c):
    m = sg.config(c, small=True)
    y = oracle.spmv(m.rowptr, m.colind, m.vals, m.x)
    s = oracle.absrow(m.rowptr, m.colind, m.vals, m.x)
    A = sp.csr_matrix((m.vals, m.colind, m.rowptr.astype(np.int64)), shape=(m.n, m.n))
    assert np.all(np.abs(y - A @ m.x) <= 1e-12 * s)
    yc = oracle.spmv_neumaier(m.rowptr, m.colind, m.vals, m.x)
    assert np.all(np.abs(y - yc) <= 1e-13 * s)


@pytest.mark.slow
@pytest.mark.parametrize("c", [1, 2, 4])
def test_neumaier_selfcheck_full_configs(c):
    m = sg.config(c)
    y = oracle.spmv(m.rowptr, m.colind, m.vals, m.x)
    s = oracle.absrow(m.rowptr, m.colind, m.vals, m.x)
    yc = oracle.spmv_neumaier(m.rowptr, m.colind, m.vals, m.x)
    assert np.all(np.abs(y - yc) <= 1e-13 * s)


def test_omp_form_bitwise_equal():
    # per-row sequential order -> bit-identical for any thread count
    m = sg.config(4, small=True)
    y = oracle.spmv(m.rowptr, m.colind, m.vals, m.x)
    for t in (1, 2, 3, 8):
        yo, used = oracle.spmv_omp(m.rowptr, m.colind, m.vals, m.x, t)
        assert used == t and np.array_equal(yo, y)


def lambda_max_27(n):
    mu = 1 + 2 * np.cos(np.arange(1, n + 1) * np.pi / (n + 1))
    return 27 - mu.max() ** 2 * mu.min()


@pytest.mark.parametrize("n,pts", [(5, 27), (6, 7), (4, 27)])
def test_power_iteration_pins(n, pts):
    m = sg.stencil(n, pts, rp64=True)
    rc, xK, nu = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, 100)
    assert rc == 0
    A = dense_of(m)
    lam = np.abs(np.linalg.eigvalsh(A)).max()
    if pts == 27:
        assert abs(lam - lambda_max_27(n)) < 1e-12 * lam  # closed form
    # nu_k nondecreasing for k >= 1 (Cauchy-Schwarz, symmetric A)
    assert np.all(np.diff(nu[1:]) >= -1e-13 * nu[1:-1])
    assert np.all(nu[1:] <= lam * (1 + 1e-13))  # k = 0 excluded: x_0 is not a unit vector
    assert abs(nu[-1] - lam) < 1e-4 * lam
    # x_K is a unit vector and satisfies x_K = A x_{K-1} / nu
    assert abs(np.linalg.norm(xK) - 1) < 1e-14
    # recompute one step independently with dense algebra
    rc2, x99, nu99 = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, 99)
    y = A @ x99
    assert np.allclose(y / np.sqrt(np.sum(y * y)), xK, rtol=0, atol=1e-14)


def test_power_iteration_zero_norm():
    rp = np.zeros(11, np.int64)
    rc, _, nu = oracle.power_iter(rp, np.zeros(0, np.int32), np.zeros(0), np.ones(10), 5)
    assert rc == -7 and nu[0] == 0.0


# ---- Neumaier self-check pinned to exact rational sums ------
def _exact_row_sums(rp, ci, va, x):
    return [sum((Fraction(float(va[j])) * Fraction(float(x[ci[j]])) for j in range(rp[i], rp[i + 1])), Fraction(0))
            for i in range(rp.size - 1)]


def test_neumaier_exact_on_cancellation_rows():
    # products {1e16, 1, -1e16} -> 1; {1, 1e100, 1, -1e100} -> 2 (Neumaier's
    # example); {3, 1e16, -1e16, -2**-30}: a plain left-to-right sum gives 0 / -2^-30,
    # the compensated sum the exact value
    rows = [[1e16, 1.0, -1e16], [1.0, 1e100, 1.0, -1e100], [3.0, 1e16, -1e16, -2.0 ** -30], [0.5, 0.25, -0.125]]
    rp = np.zeros(len(rows) + 1, np.int64)
    np.cumsum([len(r) for r in rows], out=rp[1:])
    va = np.concatenate([np.array(r) for r in rows])
    ci = np.arange(va.size, dtype=np.int32)
    x = np.ones(va.size)
    yc = oracle.spmv_neumaier(rp, ci, va, x)
    exact = _exact_row_sums(rp, ci, va, x)
    assert yc.tolist() == [float(e) for e in exact] == [1.0, 2.0, 3.0 - 2.0 ** -30, 0.625]
    yp = oracle.spmv(rp, ci, va, x)
    assert yp[0] != 1.0 and yp[1] != 2.0  # the plain sum loses them: the pin is not vacuous


@pytest.mark.parametrize("seed", range(3))
def test_neumaier_error_bound_vs_exact(seed):
    # |y_neu - S| <= u|S| + 2 n u^2 sum|p| (compensated summation bound), on rows
    # with heavy cancellation where the plain sum's error is far larger
    g = np.random.default_rng(seed)
    n, L = 60, 200
    rp = np.arange(n + 1, dtype=np.int64) * L
    big = g.uniform(-1, 1, n * L) * 10.0 ** g.integers(0, 16, n * L)
    va = np.concatenate([np.concatenate([b, -b[::-1]])[: L] + g.uniform(-1, 1, L) for b in big.reshape(n, L)[:, :L // 2]])
    ci = np.arange(va.size, dtype=np.int32)
    x = np.ones(va.size)
    yc = oracle.spmv_neumaier(rp, ci, va, x)
    exact = _exact_row_sums(rp, ci, va, x)
    u = 2.0 ** -53
    worst_plain = 0.0
    yp = oracle.spmv(rp, ci, va, x)
    for i in range(n):
        S = exact[i]
        a = float(sum(abs(Fraction(float(v))) for v in va[rp[i]:rp[i + 1]]))
        assert abs(Fraction(float(yc[i])) - S) <= u * abs(S) + Fraction(2 * L * u * u * a)
        worst_plain = max(worst_plain, float(abs(Fraction(float(yp[i])) - S)) / a)
    assert worst_plain > 4 * L * u * u  # the plain sum does not meet the compensated bound
