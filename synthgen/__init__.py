"""Seeded synthetic inputs for BASELINE.json's five configs.

Inputs only: this package holds none of the SpMV method's arithmetic, so the
oracle and the CUDA product path may both consume it. Heavy generators are in
``synthgen.cpp`` (OpenMP, counter-based SplitMix64, thread-count independent);
small structured test matrices are drawn with numpy's seeded Generator.

Config recipe (BASELINE.json configs C1..C5; seeds matrix 1711054870+c,
x 1711054880+c, value seed = matrix seed + 1000003, long-row pick seed =
matrix seed + 2000003):
  C1 n=10,000: diagonal + 8 distinct uniform off-diagonal columns, U[-1,1]
  C2 7-point Laplacian 128^3 (diag 6, off -1), Dirichlet, lexicographic
  C3 R-MAT scale 22, edge factor 16, (a,b,c,d)=(.57,.19,.19,.05), dedup,
     self-loops kept, values U(0,1]
  C4 n=1e6: 15 distinct uniform columns per row; 100 random rows instead
     hold 200,000 distinct uniform columns; U[-1,1]
  C5 27-point stencil 384^3 (diag 26, off -1), int64 rowptr
  x is U[-1,1] for every config.
"""
from __future__ import annotations

import ctypes
import os
from dataclasses import dataclass, field

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

MODE_CONST, MODE_U11, MODE_DYADIC, MODE_U01 = 0, 1, 2, 3


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "libsynthgen.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make synthgen` (or __graft_entry__.build())")
        L = ctypes.CDLL(path)
        vp, i64, u64, d, ci = ctypes.c_void_p, ctypes.c_int64, ctypes.c_uint64, ctypes.c_double, ctypes.c_int
        L.sg_rng.argtypes = [u64, u64]; L.sg_rng.restype = u64
        L.sg_u01.argtypes = [u64, u64]; L.sg_u01.restype = d
        L.sg_below.argtypes = [u64, u64, u64]; L.sg_below.restype = u64
        L.sg_num_threads.restype = ci
        L.sg_vector.argtypes = [i64, i64, u64, ci, d, vp]
        L.sg_stencil_nnz_range.argtypes = [i64, ci, i64, i64]; L.sg_stencil_nnz_range.restype = i64
        L.sg_stencil_fill.argtypes = [i64, ci, d, d, ci, u64, i64, i64, i64, vp, ci, vp, vp]
        L.sg_stencil_rowptr.argtypes = [i64, ci, i64, i64, vp, ci]
        L.sg_pick_rows.argtypes = [i64, i64, u64, vp]
        L.sg_randrows_nnz.argtypes = [i64, ci, i64, i64, i64]; L.sg_randrows_nnz.restype = i64
        L.sg_randrows_fill.argtypes = [i64, ci, i64, vp, i64, i64, u64, ci, u64, vp, ci, vp, vp]
        L.sg_rmat_make.argtypes = [ci, i64, d, d, d, u64]; L.sg_rmat_make.restype = vp
        L.sg_rmat_n.argtypes = [vp]; L.sg_rmat_n.restype = i64
        L.sg_rmat_nnz.argtypes = [vp]; L.sg_rmat_nnz.restype = i64
        L.sg_rmat_fill.argtypes = [vp, ci, u64, vp, ci, vp, vp]
        L.sg_rmat_free.argtypes = [vp]
        L.sg_checksum.argtypes = [vp, i64]; L.sg_checksum.restype = u64
        _LIB = L
    return _LIB


def _p(a):
    return a.ctypes.data_as(ctypes.c_void_p)


def checksum(a: np.ndarray) -> int:
    a = np.ascontiguousarray(a)
    return int(_lib().sg_checksum(_p(a), a.nbytes))


def rng(s, k):
    return int(_lib().sg_rng(s, k))


@dataclass
class CSR:
    n: int
    rowptr: np.ndarray
    colind: np.ndarray
    vals: np.ndarray
    x: np.ndarray
    name: str = ""
    meta: dict = field(default_factory=dict)

    @property
    def nnz(self) -> int:
        return int(self.rowptr[-1])

    def checksums(self):
        return {k: hex(checksum(getattr(self, k))) for k in ("rowptr", "colind", "vals", "x")}


def _empty(shape, dtype, out=None):
    if out is not None:
        assert out.dtype == dtype and out.size >= shape, (out.dtype, dtype, out.size, shape)
        return out[:shape]
    return np.empty(shape, dtype)


def vector(n, seed, mode=MODE_U11, i0=0, out=None):
    v = _empty(n, np.float64, out)
    _lib().sg_vector(n, i0, seed, mode, 0.0, _p(v))
    return v


def stencil(n, pts, diag=None, off=-1.0, rp64=False, val_mode=MODE_CONST, val_seed=0, x_seed=0,
            x_mode=MODE_U11, rows=None, outs=None):
    """pts in {7, 27}; rows=(rb, re) generates that row block (rowptr rebased)."""
    assert pts in (7, 27)
    if diag is None:
        diag = 6.0 if pts == 7 else 26.0
    N = n ** 3
    rb, re = rows if rows is not None else (0, N)
    L = _lib()
    nz0 = L.sg_stencil_nnz_range(n, pts, 0, rb) if rb > 0 else 0
    nnz = L.sg_stencil_nnz_range(n, pts, rb, re)
    outs = outs or {}
    rp = _empty(re - rb + 1, np.int64 if rp64 else np.int32, outs.get("rowptr"))
    ci = _empty(max(nnz, 1), np.int32, outs.get("colind"))[:nnz]
    va = _empty(max(nnz, 1), np.float64, outs.get("vals"))[:nnz]
    L.sg_stencil_fill(n, pts, diag, off, val_mode, val_seed, rb, re, nz0, _p(rp), 8 if rp64 else 4, _p(ci), _p(va))
    x = vector(N, x_seed, x_mode, out=outs.get("x"))
    return CSR(N, rp, ci, va, x, name=f"stencil{pts}_{n}", meta={"rows": (rb, re), "nz0": nz0})


def stencil_rowptr(n, pts, rp64=True, rows=None):
    """Global rowptr of the pts-point stencil on n^3 (or of a row block, rebased)."""
    N = n ** 3
    rb, re = rows if rows is not None else (0, N)
    rp = np.empty(re - rb + 1, np.int64 if rp64 else np.int32)
    _lib().sg_stencil_rowptr(n, pts, rb, re, _p(rp), 8 if rp64 else 4)
    return rp


def randrows(n, k, diag=True, long_rows=None, k_long=0, col_seed=1, val_mode=MODE_U11, val_seed=2,
             x_seed=3, x_mode=MODE_U11, rp64=False):
    lr = np.ascontiguousarray(long_rows if long_rows is not None else np.zeros(0), np.int64)
    L = _lib()
    nnz = L.sg_randrows_nnz(n, int(diag), k, lr.size, k_long)
    rp = np.empty(n + 1, np.int64 if rp64 else np.int32)
    ci = np.empty(nnz, np.int32)
    va = np.empty(nnz, np.float64)
    L.sg_randrows_fill(n, int(diag), k, _p(lr), lr.size, k_long, col_seed, val_mode, val_seed,
                       _p(rp), 8 if rp64 else 4, _p(ci), _p(va))
    x = vector(n, x_seed, x_mode)
    return CSR(n, rp, ci, va, x, name=f"randrows_{n}_{k}")


def pick_rows(n, count, seed):
    out = np.empty(count, np.int64)
    _lib().sg_pick_rows(n, count, seed, _p(out))
    return out


def rmat(scale, edge_factor, a=0.57, b=0.19, c=0.19, seed=1, val_mode=MODE_U01, val_seed=2, x_seed=3,
         x_mode=MODE_U11, rp64=False):
    L = _lib()
    h = L.sg_rmat_make(scale, edge_factor, a, b, c, seed)
    try:
        n, nnz = L.sg_rmat_n(h), L.sg_rmat_nnz(h)
        rp = np.empty(n + 1, np.int64 if rp64 else np.int32)
        ci = np.empty(nnz, np.int32)
        va = np.empty(nnz, np.float64)
        L.sg_rmat_fill(h, val_mode, val_seed, _p(rp), 8 if rp64 else 4, _p(ci), _p(va))
    finally:
        L.sg_rmat_free(h)
    x = vector(n, x_seed, x_mode)
    return CSR(n, rp, ci, va, x, name=f"rmat_{scale}_{edge_factor}")


# --------------------------------------------------------------------------
# BASELINE.json configs. `scale` shrinks the sizes for
# parity tests while keeping each config's structure.
# --------------------------------------------------------------------------
def seeds(c):
    ms = 1711054870 + c
    return {"matrix": ms, "x": 1711054880 + c, "value": ms + 1000003, "pick": ms + 2000003}


def config(c, small=False, rp64=None, val_mode=None, x_mode=MODE_U11, outs=None, rows=None):
    """Build config c in 1..5. small=True gives the same structure at sizes the
    oracle finishes in seconds (C2: 24^3, C3: scale 14, C4: n=20000 with
    10 long rows of 4500, C5: 27-pt 20^3)."""
    s = seeds(c)
    if c == 1:
        m = randrows(10000, 8, diag=True, col_seed=s["matrix"], val_mode=val_mode or MODE_U11,
                     val_seed=s["value"], x_seed=s["x"], x_mode=x_mode, rp64=bool(rp64))
        m.name = "C1_uniform_random_10k"
        return m
    if c == 2:
        n = 24 if small else 128
        m = stencil(n, 7, rp64=bool(rp64), val_mode=val_mode or MODE_CONST, val_seed=s["value"],
                    x_seed=s["x"], x_mode=x_mode, rows=rows, outs=outs)
        m.name = f"C2_lap7_{n}^3"
        return m
    if c == 3:
        scale = 14 if small else 22
        m = rmat(scale, 16, seed=s["matrix"], val_mode=val_mode or MODE_U01, val_seed=s["value"],
                 x_seed=s["x"], x_mode=x_mode, rp64=bool(rp64))
        m.name = f"C3_rmat_s{scale}_ef16"
        return m
    if c == 4:
        n, nl, kl = (20000, 10, 4500) if small else (1000000, 100, 200000)
        lr = pick_rows(n, nl, s["pick"])
        m = randrows(n, 15, diag=False, long_rows=lr, k_long=kl, col_seed=s["matrix"],
                     val_mode=val_mode or MODE_U11, val_seed=s["value"], x_seed=s["x"], x_mode=x_mode,
                     rp64=bool(rp64))
        m.name = f"C4_longrow_{n}"
        m.meta["long_rows"] = lr
        return m
    if c == 5:
        n = 20 if small else 384
        m = stencil(n, 27, rp64=True if rp64 is None else rp64, val_mode=val_mode or MODE_CONST,
                    val_seed=s["value"], x_seed=s["x"], x_mode=x_mode, rows=rows, outs=outs)
        m.name = f"C5_st27_{n}^3"
        return m
    raise ValueError(c)


# --------------------------------------------------------------------------
# Small structured matrices for parity tests (numpy Generator, seeded)
# --------------------------------------------------------------------------
def from_lengths(lens, n_cols, rng_, val_mode=MODE_U11, x_mode=MODE_U11, rp64=False):
    """Random sorted distinct columns per row with the given row lengths."""
    lens = np.asarray(lens, np.int64)
    n = lens.size
    rp = np.zeros(n + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    ci = np.empty(int(rp[-1]), np.int32)
    for i in range(n):
        L_ = int(lens[i])
        if L_:
            ci[rp[i]:rp[i + 1]] = np.sort(rng_.choice(n_cols, size=L_, replace=False))
    va = _draw(rng_, ci.size, val_mode)
    x = _draw(rng_, n_cols, x_mode)
    return CSR(n, rp.astype(np.int64 if rp64 else np.int32), ci, va, x)


def _draw(rng_, m, mode):
    if mode == MODE_DYADIC:
        return rng_.integers(-1024, 1025, size=m).astype(np.float64) / 1024.0
    if mode == MODE_U01:
        return 1.0 - rng_.random(m)
    return rng_.uniform(-1.0, 1.0, size=m)


def small_suite(seed=0, val_mode=MODE_U11, x_mode=MODE_U11):
    """A list of (name, CSR) covering the structures the method distinguishes:
    uniform short rows, empty rows, power-law lengths, a dense row, long rows,
    diagonal, single row, all-empty, banded."""
    g = np.random.default_rng(seed)
    out = []

    def add(name, lens, ncols=None):
        lens = np.asarray(lens, np.int64)
        out.append((name, from_lengths(lens, ncols or max(int(lens.max(initial=0)), lens.size), g,
                                       val_mode, x_mode)))

    add("uniform9", np.full(3000, 9))
    add("len1", np.ones(1000, np.int64))
    add("empty_mix", g.choice([0, 0, 0, 3, 17], size=4000))
    add("powerlaw", np.minimum((g.pareto(1.2, size=5000) * 3).astype(np.int64), 4999))
    lens = np.full(2000, 5); lens[777] = 2000
    add("one_dense_row", lens)
    lens = np.full(6000, 7); lens[[5, 100, 4000]] = [5000, 6000, 5500]
    add("long_rows", lens)
    add("all_empty", np.zeros(500, np.int64), ncols=500)
    add("single_row", np.array([4096]), ncols=5000)
    add("two_rows_long_short", np.array([9000, 1]), ncols=9000)
    add("mixed_32_64", g.choice([31, 33, 64, 65, 128], size=2500), ncols=3000)
    out.append(("diag", _diag(2048, g, val_mode, x_mode)))
    out.append(("banded", _banded(5000, 3, g, val_mode, x_mode)))
    return out


def _diag(n, g, val_mode, x_mode):
    rp = np.arange(n + 1, dtype=np.int32)
    ci = np.arange(n, dtype=np.int32)
    return CSR(n, rp, ci, _draw(g, n, val_mode), _draw(g, n, x_mode))


def _banded(n, bw, g, val_mode, x_mode):
    rows, cols = [], []
    for i in range(n):
        for c in range(max(0, i - bw), min(n, i + bw + 1)):
            rows.append(i); cols.append(c)
    rows = np.asarray(rows); cols = np.asarray(cols, np.int32)
    rp = np.zeros(n + 1, np.int64)
    np.add.at(rp, rows + 1, 1)
    rp = np.cumsum(rp).astype(np.int32)
    return CSR(n, rp, cols, _draw(g, cols.size, val_mode), _draw(g, n, x_mode))
