"""Plain CPU oracle for the SpMV hot path -- TEST INFRASTRUCTURE ONLY.

Only ``tests/``, ``__graft_entry__.smoke()`` and ``bench.py``'s
``cpu_baseline`` / ``--impl reference`` legs may import this package. The
product path (``paper_1711_05487_b200``) never imports it and shares no code
with it (no kernels, headers, helpers, tables or constants).

Heavy loops live in ``oracle.c`` (fp64, no FMA, serial); the small pure
functions (selection rule, analytic bounds, amortisation, harmonic mean) are
written out here in Python. Every function cites the passage it follows:
``P:n`` = reference PAPER.md line n, ``S:n`` = SPEC.md line n, ``SURVEY 8(x)``
= the reading this build takes.

Pins (tests/test_oracle_*.py, ``-m "not gpu"``) -- no function is
"parity unpinned":
  spmv            dense brute-force matvec, identity/diagonal exact, A e_j =
                  column j exact, stencil A*1 closed forms, dyadic exactness
                  vs Fraction arithmetic, scipy csr @ x, Neumaier self-check
  spmv_neumaier   exact Fraction row sums on cancellation rows (the plain sum
                  fails them), the compensated-summation error bound
  power_iter      monotone nu_k (k>=1) for symmetric A, nu <= lambda_max closed
                  form, nu -> lambda_max vs numpy eigvalsh on a small grid
  shard_bounds    SPEC S:254-255 examples, linear-scan definition, coverage
  tile_rows       linear-scan definition, ownership cover
  merge_splits    binary-search split vs the sequential merge, path invariants
  long_chunks     coverage / exact tiling of long rows
  nonempty_rows   numpy flatnonzero of the row lengths, coverage
  nz_tiles        binary-search (searchsorted) re-derivation, ownership cover
  hot_columns     hand example, maximality of the count threshold
  classify_profile SPEC S:469-474 examples, strictness, monotonicity in P_ML
  table1          SPEC S:415-417 worked rows, diagonal closed form, brute-force per-row loops
  d16 encode/dec  SPEC S:134-136 widths, round trip, stencil gap closed forms
  features        SPEC S:415 sd example, stencil closed forms, short-row
                  statistics / n_empty / long rows vs numpy incl. L_split edges
  d8 dict/enc/dec stencil dictionaries from the grid geometry (7-pt: 10, 27-pt:
                  15 codes), hand example, 256/257 and 255/256 limits, round trip
  pat enc/dec     stencil patterns from the grid geometry (27 boundary classes,
                  interior offsets dz n^2 + dy n + dx), hand example, first-
                  occurrence order vs a dict-based re-derivation, 256/257 and
                  offset limits, round trip
  select          hand-evaluated rule table on the configs' closed-form features
"""
from __future__ import annotations

import ctypes
import math
import os
from dataclasses import dataclass

import numpy as np

_HERE = os.path.dirname(os.path.abspath(__file__))
_LIB = None

_i64p = ctypes.POINTER(ctypes.c_int64)


def _lib():
    global _LIB
    if _LIB is None:
        path = os.path.join(_HERE, "liboracle.so")
        if not os.path.exists(path):
            raise RuntimeError(f"{path} missing: run `make oracle` (or __graft_entry__.build())")
        L = ctypes.CDLL(path)
        vp = ctypes.c_void_p
        i64 = ctypes.c_int64
        L.oracle_spmv.argtypes = [i64, vp, vp, vp, vp, vp]
        L.oracle_spmv_rows.argtypes = [vp, vp, vp, vp, vp, i64, vp]
        L.oracle_absrow_rows.argtypes = [vp, vp, vp, vp, vp, i64, vp]
        L.oracle_spmv_neumaier.argtypes = [i64, vp, vp, vp, vp, vp]
        L.oracle_spmv_omp.argtypes = [i64, vp, vp, vp, vp, vp, ctypes.c_int]
        L.oracle_spmv_omp.restype = ctypes.c_int
        L.oracle_power_iter.argtypes = [i64, vp, vp, vp, vp, ctypes.c_int, vp, vp, ctypes.c_int]
        L.oracle_power_iter.restype = ctypes.c_int
        L.oracle_shard_bounds.argtypes = [i64, vp, i64, i64, vp]
        L.oracle_validate.argtypes = [i64, i64, vp, vp, _i64p]
        L.oracle_validate.restype = ctypes.c_int
        L.oracle_features.argtypes = [i64, vp, vp, i64, i64, vp]
        L.oracle_tile_rows.argtypes = [i64, vp, i64, i64, vp]
        L.oracle_merge_splits.argtypes = [i64, vp, i64, i64, i64, vp, vp]
        L.oracle_long_chunks.argtypes = [i64, vp, i64, i64, vp, vp, vp]
        L.oracle_nonempty_rows.argtypes = [i64, vp, vp, vp]
        L.oracle_nonempty_rows.restype = i64
        L.oracle_nz_tiles.argtypes = [i64, vp, i64, i64, vp]
        L.oracle_long_chunks.restype = i64
        L.oracle_d16_encode.argtypes = [i64, vp, vp, vp, vp, _i64p]
        L.oracle_d16_encode.restype = ctypes.c_int
        L.oracle_d16_decode.argtypes = [i64, vp, vp, vp, vp]
        L.oracle_d16_encode_esc.argtypes = [i64, vp, vp, vp, vp, _i64p, vp, ctypes.POINTER(ctypes.c_int)]
        L.oracle_d16_encode_esc.restype = ctypes.c_int
        L.oracle_d16_decode_esc.argtypes = [i64, vp, vp, vp, vp, vp]
        L.oracle_tile_anchor.argtypes = [vp, i64, i64, i64, vp]
        L.oracle_d8_dict.argtypes = [i64, vp, vp, vp]
        L.oracle_d8_dict.restype = ctypes.c_int
        L.oracle_d8_encode.argtypes = [i64, vp, vp, vp, vp, vp]
        L.oracle_d8_encode.restype = ctypes.c_int
        L.oracle_d8_decode.argtypes = [i64, vp, vp, vp, vp]
        L.oracle_pat_encode.argtypes = [i64, vp, vp, i64, i64, vp, vp, vp]
        L.oracle_pat_encode.restype = i64
        L.oracle_pat_decode.argtypes = [i64, vp, i64, vp, vp, vp]
        _LIB = L
    return _LIB


def _p(a):
    return None if a is None else a.ctypes.data_as(ctypes.c_void_p)


def _rp64(rowptr):
    return np.ascontiguousarray(rowptr, dtype=np.int64)


def _c32(colind):
    return np.ascontiguousarray(colind, dtype=np.int32)


def _f64(v):
    return np.ascontiguousarray(v, dtype=np.float64)


# --------------------------------------------------------------------------
# SpMV (Fig. 2, accumulation reading SURVEY 8(c3) #1)
# --------------------------------------------------------------------------
def spmv(rowptr, colind, vals, x):
    rp = _rp64(rowptr)
    n = rp.size - 1
    y = np.empty(n, np.float64)
    ci, v, xx = _c32(colind), _f64(vals), _f64(x)
    _lib().oracle_spmv(n, _p(rp), _p(ci), _p(v), _p(xx), _p(y))
    return y


def spmv_omp(rowptr, colind, vals, x, nthreads=0):
    """Row-parallel form (P:708-711 static nnz-balanced partition); bitwise == spmv."""
    rp = _rp64(rowptr)
    n = rp.size - 1
    y = np.empty(n, np.float64)
    ci, v, xx = _c32(colind), _f64(vals), _f64(x)
    used = _lib().oracle_spmv_omp(n, _p(rp), _p(ci), _p(v), _p(xx), _p(y), int(nthreads))
    return y, used


def spmv_rows(rowptr, colind, vals, x, rows):
    rp, ci, v, xx = _rp64(rowptr), _c32(colind), _f64(vals), _f64(x)
    r = np.ascontiguousarray(rows, dtype=np.int64)
    out = np.empty(r.size, np.float64)
    _lib().oracle_spmv_rows(_p(rp), _p(ci), _p(v), _p(xx), _p(r), r.size, _p(out))
    return out


def absrow(rowptr, colind, vals, x, rows=None):
    """s_i = sum_j |a_ij x_j|, the right side of BJ.north_star's per-row bound."""
    rp, ci, v, xx = _rp64(rowptr), _c32(colind), _f64(vals), _f64(x)
    if rows is None:
        m = rp.size - 1
        out = np.empty(m, np.float64)
        _lib().oracle_absrow_rows(_p(rp), _p(ci), _p(v), _p(xx), None, m, _p(out))
    else:
        r = np.ascontiguousarray(rows, dtype=np.int64)
        out = np.empty(r.size, np.float64)
        _lib().oracle_absrow_rows(_p(rp), _p(ci), _p(v), _p(xx), _p(r), r.size, _p(out))
    return out


def spmv_neumaier(rowptr, colind, vals, x):
    rp = _rp64(rowptr)
    n = rp.size - 1
    y = np.empty(n, np.float64)
    ci, v, xx = _c32(colind), _f64(vals), _f64(x)
    _lib().oracle_spmv_neumaier(n, _p(rp), _p(ci), _p(v), _p(xx), _p(y))
    return y


def power_iter(rowptr, colind, vals, x0, K, nthreads=1):
    """Iterated mode x <- Ax/||Ax|| (BJ.configs[5]). Returns (rc, x_K, nu[K])."""
    rp = _rp64(rowptr)
    n = rp.size - 1
    ci, v, x = _c32(colind), _f64(vals), _f64(x0)
    xo = np.empty(n, np.float64)
    nu = np.zeros(K, np.float64)
    rc = _lib().oracle_power_iter(n, _p(rp), _p(ci), _p(v), _p(x), int(K), _p(xo), _p(nu), int(nthreads))
    return rc, xo, nu


# --------------------------------------------------------------------------
# Plan structures; bit-exact definitions
# --------------------------------------------------------------------------
def shard_bounds(rowptr, G):
    rp = _rp64(rowptr)
    b = np.empty(G + 1, np.int64)
    _lib().oracle_shard_bounds(rp.size - 1, _p(rp), int(rp[-1]), int(G), _p(b))
    return b


VALIDATE_CODES = {0: "ok", 1: "rowptr[0] != 0", 2: "rowptr[n] != nnz", 3: "rowptr decreasing",
                  4: "colind out of range", 5: "colind not strictly increasing in row"}


def validate(n, nnz, rowptr, colind):
    rp, ci = _rp64(rowptr), _c32(colind)
    where = ctypes.c_int64(-1)
    code = _lib().oracle_validate(int(n), int(nnz), _p(rp), _p(ci), ctypes.byref(where))
    return code, where.value


class _Feat(ctypes.Structure):
    _fields_ = [(k, ctypes.c_int64) for k in
                ("n", "nnz", "nnz_min", "nnz_max", "n_empty", "n_long", "nnz_long", "n_short", "max_short")] + \
               [(k, ctypes.c_uint64) for k in ("s1", "s2", "s1_short", "s2_short")] + \
               [(k, ctypes.c_int64) for k in ("maxgap", "misses")] + \
               [(k, ctypes.c_double) for k in ("nnz_avg", "nnz_sd", "avg_short", "sd_short")]


def features(rowptr, colind, L_split=4096, line_elems=16, n_cols=None):
    """Theta(N) Table I features + counts for selection.
    n_cols (default: square, = rows) is carried for the long-row density test."""
    rp, ci = _rp64(rowptr), _c32(colind)
    f = _Feat()
    _lib().oracle_features(rp.size - 1, _p(rp), _p(ci), int(L_split), int(line_elems), ctypes.byref(f))
    d = {k: getattr(f, k) for k, _ in _Feat._fields_}
    d["n_cols"] = int(rp.size - 1 if n_cols is None else n_cols)
    d["n_big_gaps"] = big_gap_count(rp, ci)
    c = np.asarray(colind)
    d["col_min"], d["col_max"] = (int(c.min()), int(c.max())) if c.size else (0, -1)
    d["n_deltas"] = d8_dict(rp, ci)[0]
    return d


ESC0, ESC_MAX, BIG_TAB = 65472, 64, 128


def big_gap_count(rowptr, colind):
    """Distinct in-row gaps >= 65472 (the escape-coded D16 candidates),
    BIG_TAB + 1 when there are more than BIG_TAB (reading 21)."""
    rp, ci = _rp64(rowptr), np.asarray(colind, np.int64)
    if ci.size < 2:
        return 0
    g = np.diff(ci)
    head = np.zeros(ci.size, bool)
    starts = rp[:-1][np.diff(rp) > 0]
    head[starts] = True
    g = g[~head[1:]]
    u = np.unique(g[g >= ESC0])
    return int(u.size) if u.size <= BIG_TAB else BIG_TAB + 1


def tile_count(nnz, C):
    return max(1, -(-int(nnz) // int(C)))


def tile_rows(rowptr, C):
    rp = _rp64(rowptr)
    T = tile_count(rp[-1], C)
    R = np.empty(T + 1, np.int64)
    _lib().oracle_tile_rows(rp.size - 1, _p(rp), int(C), T, _p(R))
    return R


NZ_TILE = 256  # nnz_split warp tile (nonzeros)


def nonempty_rows(rowptr):
    """(rowmap[mc+1], rpc[mc+1]) of the non-empty rows (reading 19)."""
    rp = _rp64(rowptr)
    n = rp.size - 1
    mc = _lib().oracle_nonempty_rows(n, _p(rp), None, None)
    rowmap = np.empty(mc + 1, np.int64)
    rpc = np.empty(mc + 1, np.int64)
    _lib().oracle_nonempty_rows(n, _p(rp), _p(rowmap), _p(rpc))
    return rowmap, rpc


def nz_tiles(rpc, W=NZ_TILE):
    """tile_q[k] = largest q with rpc[q] <= k*W (k < T = ceil(nnz/W)), tile_q[T] = mc."""
    rpc = _rp64(rpc)
    mc, nnz = rpc.size - 1, int(rpc[-1])
    T = -(-nnz // int(W))
    tq = np.empty(T + 1, np.int64)
    _lib().oracle_nz_tiles(mc, _p(rpc), int(W), T, _p(tq))
    return tq


HOT_BUCKETS = 4096


def hot_columns(colind, n_cols, K, buckets=HOT_BUCKETS):
    """nnz_split hot-x set (reading 20): column counts cnt, count
    histogram H[min(cnt, buckets-1)]; t = the smallest count >= 1 such that the
    columns with cnt >= t number <= K (the top bucket is taken whole); the hot
    columns are those with cnt >= t in column order, the first min(#, K)
    rounded down to even. Returns (hot columns, coverage = their nonzeros)."""
    cnt = np.bincount(np.asarray(colind, np.int64), minlength=int(n_cols))
    H = np.bincount(np.minimum(cnt, buckets - 1), minlength=buckets)
    acc, t = 0, buckets - 1
    for v in range(buckets - 1, 0, -1):
        if v < buckets - 1 and acc + H[v] > K:
            break
        acc += int(H[v])
        t = v
    hot = np.flatnonzero(cnt >= t)
    k2 = min(hot.size, K) & ~1
    hot = hot[:k2]
    return hot, int(cnt[hot].sum())


def merge_splits(rowptr, items):
    rp = _rp64(rowptr)
    n, nnz = rp.size - 1, int(rp[-1])
    T = max(1, -(-(n + nnz) // int(items)))
    si = np.empty(T + 1, np.int64)
    sj = np.empty(T + 1, np.int64)
    _lib().oracle_merge_splits(n, _p(rp), nnz, int(items), T, _p(si), _p(sj))
    return si, sj


def long_chunks(rowptr, L_split, C):
    rp = _rp64(rowptr)
    n = rp.size - 1
    q = _lib().oracle_long_chunks(n, _p(rp), int(L_split), int(C), None, None, None)
    crow, cb, ce = (np.empty(q, np.int64) for _ in range(3))
    if q:
        _lib().oracle_long_chunks(n, _p(rp), int(L_split), int(C), _p(crow), _p(cb), _p(ce))
    return crow, cb, ce


def d16_encode(rowptr, colind):
    """Returns (width, maxgap, dcol u16[nnz] | None, head i32[n] | None)."""
    rp, ci = _rp64(rowptr), _c32(colind)
    n, nnz = rp.size - 1, int(rp[-1])
    dcol = np.zeros(max(nnz, 1), np.uint16)
    head = np.zeros(max(n, 1), np.int32)
    mg = ctypes.c_int64(0)
    w = _lib().oracle_d16_encode(n, _p(rp), _p(ci), _p(dcol), _p(head), ctypes.byref(mg))
    if w == 0:
        return 0, mg.value, None, None
    return w, mg.value, dcol[:nnz], head[:n]


def d16_encode_esc(rowptr, colind):
    """d16_encode extended with escape codes (reading 21). Returns
    (width, maxgap, dcol | None, head | None, esc table)."""
    rp, ci = _rp64(rowptr), _c32(colind)
    n, nnz = rp.size - 1, int(rp[-1])
    dcol = np.zeros(max(nnz, 1), np.uint16)
    head = np.zeros(max(n, 1), np.int32)
    esc = np.zeros(64, np.int32)
    mg = ctypes.c_int64(0)
    ne = ctypes.c_int(0)
    w = _lib().oracle_d16_encode_esc(n, _p(rp), _p(ci), _p(dcol), _p(head), ctypes.byref(mg), _p(esc),
                                     ctypes.byref(ne))
    if w == 0:
        return 0, mg.value, None, None, esc[:0]
    return w, mg.value, dcol[:nnz], head[:n], esc[:ne.value].copy()


def d16_decode_esc(rowptr, dcol, head, esc):
    rp = _rp64(rowptr)
    out = np.empty(max(int(rp[-1]), 1), np.int32)
    e = np.zeros(64, np.int32)
    e[:len(esc)] = esc
    _lib().oracle_d16_decode_esc(rp.size - 1, _p(rp), _p(np.ascontiguousarray(dcol, np.uint16)),
                                 _p(np.ascontiguousarray(head, np.int32)), _p(e), _p(out))
    return out[:int(rp[-1])]


def d16_decode(rowptr, dcol, head):
    rp = _rp64(rowptr)
    n, nnz = rp.size - 1, int(rp[-1])
    out = np.empty(max(nnz, 1), np.int32)
    _lib().oracle_d16_decode(n, _p(rp), _p(np.ascontiguousarray(dcol, np.uint16)),
                             _p(np.ascontiguousarray(head, np.int32)), _p(out))
    return out[:nnz]


def d8_dict(rowptr, colind):
    """Distinct row-relative deltas in ascending order (reading 26;
    P:589-597): head delta colind[rowptr[i]] - i, in-row gaps
    colind[j] - colind[j-1]. Returns (count, dict) with count = 257 (and a
    partial dict) when more than 256 distinct deltas exist."""
    rp, ci = _rp64(rowptr), _c32(colind)
    d = np.zeros(257, np.int64)
    nd = _lib().oracle_d8_dict(rp.size - 1, _p(rp), _p(ci), _p(d))
    return nd, d[:min(nd, 256)].copy()


def d8_encode(rowptr, colind):
    """Dictionary-coded 8-bit deltas. Returns (dict int64[nd], codes u8[nnz],
    rlen u8[n]) or None when not D8-codable (> 256 distinct deltas or a row
    longer than 255)."""
    rp, ci = _rp64(rowptr), _c32(colind)
    n, nnz = rp.size - 1, int(rp[-1])
    d = np.zeros(256, np.int64)
    codes = np.zeros(max(nnz, 1), np.uint8)
    rlen = np.zeros(max(n, 1), np.uint8)
    nd = _lib().oracle_d8_encode(n, _p(rp), _p(ci), _p(d), _p(codes), _p(rlen))
    if nd == 0 and nnz > 0:
        return None
    return d[:nd].copy(), codes[:nnz], rlen[:n]


def d8_decode(dict_, codes, rlen):
    rl = np.ascontiguousarray(rlen, np.uint8)
    cd = np.ascontiguousarray(codes, np.uint8)
    d = np.zeros(256, np.int64)
    d[:len(dict_)] = dict_
    out = np.empty(max(cd.size, 1), np.int32)
    _lib().oracle_d8_decode(rl.size, _p(rl), _p(cd), _p(d), _p(out))
    return out[:cd.size]


PAT_MAX = 256       # DESIGN.md reading 31: at most 256 row patterns (one byte per row) ...
PAT_MAX_OFS = 4096  # ... holding at most 4096 column offsets in total


def pat_encode(rowptr, colind, maxp=PAT_MAX, maxofs=PAT_MAX_OFS):
    """Row-pattern codes (reading 31): pattern of row i = (len_i;
    colind[j] - i for j in row i), numbered by first occurrence. Returns
    (ids u8[n], lens int64[np], ofs int64[sum lens]) or None when not codable
    (a row longer than 255, > maxp patterns or > maxofs offsets)."""
    rp, ci = _rp64(rowptr), _c32(colind)
    n = rp.size - 1
    ids = np.zeros(max(n, 1), np.uint8)
    lens = np.zeros(max(maxp, 1), np.int64)
    ofs = np.zeros(max(maxofs, 1), np.int64)
    npat = _lib().oracle_pat_encode(n, _p(rp), _p(ci), int(maxp), int(maxofs), _p(ids), _p(lens), _p(ofs))
    if npat < 0:
        return None
    return ids[:n], lens[:npat].copy(), ofs[:int(lens[:npat].sum())].copy()


def pat_decode(ids, lens, ofs):
    ids_ = np.ascontiguousarray(ids, np.uint8)
    ln = np.ascontiguousarray(lens, np.int64)
    of = np.ascontiguousarray(ofs, np.int64)
    nnz = int(ln[ids_].sum()) if ids_.size else 0
    out = np.empty(max(nnz, 1), np.int32)
    _lib().oracle_pat_decode(ids_.size, _p(ids_), ln.size, _p(ln), _p(of), _p(out))
    return out[:nnz]


def tile_anchor(colind, C):
    ci = _c32(colind)
    T = tile_count(ci.size, C)
    out = np.empty(T, np.int32)
    _lib().oracle_tile_anchor(_p(ci), ci.size, int(C), T, _p(out))
    return out


# --------------------------------------------------------------------------
# Analytic bounds (Sec. III-B) and methodology helpers
# --------------------------------------------------------------------------
def p_mb(nnz, n, bmax, rowptr_bytes=4, colind_bytes=4):
    """P_MB = 2 NNZ / ((S_CSR + S_x + S_y)/B_max), S_CSR = 8NNZ + 4NNZ + 4(N+1)."""
    s = 8 * nnz + colind_bytes * nnz + rowptr_bytes * (n + 1) + 16 * n
    return 2.0 * nnz / (s / bmax)


def p_peak(nnz, n, bmax):
    """P_peak = 2 NNZ / ((S_values + S_x + S_y)/B_max)."""
    return 2.0 * nnz / ((8 * nnz + 16 * n) / bmax)


def algorithmic_bytes(n, nnz, rowptr_bytes):
    """BJ.metric bytes: values + colind + rowptr + x + y, uncompressed CSR."""
    return 8 * nnz + 4 * nnz + rowptr_bytes * (n + 1) + 8 * n + 8 * n


def n_iters_min(t_pre, t_base, t_sel):
    """N_iters,min = t_pre / (t_spmv - t'_spmv) (SPEC example S:627)."""
    d = t_base - t_sel
    return math.inf if d <= 0 else t_pre / d


def harmonic_mean(rates):
    """Paper methodology: runs summarised by the harmonic mean."""
    return len(rates) / sum(1.0 / r for r in rates)


# --------------------------------------------------------------------------
# Selection (Table II). A pure function of the
# features and device properties. Rule constants are readings.
# --------------------------------------------------------------------------
VARIANT_VECTOR, VARIANT_STREAM, VARIANT_MERGE, VARIANT_SPLIT, VARIANT_NNZSPLIT = 1, 2, 3, 4, 5
CLASS_MB, CLASS_ML, CLASS_IMB, CLASS_CMP = 1, 2, 4, 8


D8_MAX, D8_MAX_ROW = 256, 255  # one byte per code / per row length


@dataclass
class Selection:
    variant: int
    vs: int
    d16: int  # 0 int32 colind, 1 16-bit deltas, 2 dictionary-coded 8-bit deltas (D8)
    xwin: bool
    classes: int


def _pow2ceil(v):
    p = 1
    while p < v:
        p *= 2
    return p


def select(f, l2_bytes, window_max, rowptr_bytes, K_long=100, skew_sd=1.0, empty_frac=0.25):
    """Feature-guided selection. f = features(..) dict.

    IMB: long rows (n_long > 0 and nnz_max > K_long*nnz_avg) ->
    long_row_split when they are dense enough for column-tiled x blocks
    (nnz_long >= 64 * n_long * ceil(n_cols/2048)), else nnz_split; skew
    (sd_s/avg_s > skew_sd or empty/N > empty_frac) -> nnz_split. Tiny
    matrices (<= 2^20 nonzeros, launch-bound) -> csr_vector. Scattered
    columns (misses/nnz > 0.75: most nonzeros open a new x line, the ML access
    pattern of Table I) -> nnz_split (L1 x gathers, 8 per lane; DESIGN.md
    reading 24). Other regular rows -> cta_stream for avg_s <= 32, else
    csr_vector (CMP analogue: lane group sized to the row, VS =
    clamp(pow2ceil(avg_s), 2, 32)). MB: working set > L2/2 (the
    D16 colind it maps to is available but not auto-selected: slower on
    B200, reading 9). ML:
    misses/nnz > 0.75 and x larger than L2/16 -> x persistence window when it
    fits the access-policy window.
    """
    n, nnz = f["n"], f["nnz"]
    avg_s = f["avg_short"]
    sd_s = f["sd_short"]
    ws = algorithmic_bytes(n, nnz, rowptr_bytes)
    classes = 0
    skew = n > 0 and ((avg_s > 0 and sd_s / avg_s > skew_sd) or f["n_empty"] > empty_frac * n)
    longr = f["n_long"] > 0 and f["nnz_max"] > K_long * f["nnz_avg"]
    if skew or longr:
        classes |= CLASS_IMB
    vs = min(32, max(2, _pow2ceil(int(math.ceil(avg_s))) if avg_s > 0 else 2))
    nblk = -(-int(f.get("n_cols", n)) // 2048)
    dense_long = f["n_long"] > 0 and f["nnz_long"] >= 64 * f["n_long"] * nblk
    if longr:  # long rows first: the decomposition also absorbs skew
        variant = VARIANT_SPLIT if dense_long else VARIANT_NNZSPLIT
    elif skew:
        variant = VARIANT_NNZSPLIT
    elif nnz <= (1 << 20):  # tiny matrices: launch-bound, plain csr_vector
        variant = VARIANT_VECTOR
    elif nnz > 0 and f["misses"] > 0.75 * nnz:  # scattered columns (ML access pattern, Table I misses)
        variant = VARIANT_NNZSPLIT
    elif avg_s <= 32:
        variant = VARIANT_STREAM
    else:
        variant = VARIANT_VECTOR
    if variant == VARIANT_STREAM:
        # cta_stream: one lane per row up to 32 nonzeros, else pow2ceil(avg_s/32)
        vs = min(32, _pow2ceil(int(math.ceil(avg_s / 32.0)))) if avg_s > 32 else 1
    if avg_s <= 4:
        classes |= CLASS_CMP
    mb = ws > l2_bytes // 2
    if mb and not (classes & CLASS_IMB):
        classes |= CLASS_MB
    # MB delta colind: 16-bit deltas (or escape codes) only when forced
    # (measured slower on B200, reading 9); dictionary-coded 8-bit
    # deltas (D8, reading 26) for MB stream plans with regular rows, one lane
    # per row, <= 256 distinct row-relative deltas and rows <= 255 nonzeros
    d8_ok = f.get("n_deltas", D8_MAX + 1) <= D8_MAX and f["nnz_max"] <= D8_MAX_ROW and nnz > 0
    regular = f["nnz_max"] > 0 and f["nnz_max"] <= 1.25 * f["nnz_avg"] + 1.0
    d16 = 2 if (variant == VARIANT_STREAM and (classes & CLASS_MB) and d8_ok and regular and vs == 1) else 0
    ml = nnz > 0 and f["misses"] > 0.75 * nnz and 8 * n > l2_bytes // 16
    if ml:
        classes |= CLASS_ML
    xwin = bool(ml and 8 * n <= window_max)
    return Selection(variant, vs, d16, xwin, classes)


# ---- profile-guided selection (reading 22) --------------
T_IMB, T_ML, APPROX_TOL = 1.24, 1.25, 0.10  # Fig. 4 caption
# The same hyperparameters re-tuned for B200 by the paper's procedure, a grid
# search maximising the average gain of the selected optimisation,
# over a synthetic matrix set (tools/tune_profile.py -> profiles/
# r02_profile_tuning.json; reading 29): the library's defaults.
T_IMB_B200, T_ML_B200, APPROX_TOL_B200 = 2.54, 1.08, 0.10


def classify_profile(p_csr, p_mb, p_ml, p_imb, p_cmp, p_peak, t_imb=T_IMB, t_ml=T_ML, tol=APPROX_TOL):
    """Fig. 4, written out: multilabel, strict '>', 'P_CSR ~ P_MB'
    read as P_CSR >= (1 - tol) P_MB. Returns a CLASS_* bitmask."""
    c = 0
    if p_csr <= 0:
        return 0
    if p_imb / p_csr > t_imb:
        c |= CLASS_IMB
    if p_ml / p_csr > t_ml:
        c |= CLASS_ML
    if p_csr >= (1 - tol) * p_mb and p_mb < p_cmp < p_peak:
        c |= CLASS_MB
    if p_mb > p_cmp or p_cmp > p_peak:
        c |= CLASS_CMP
    return c


def profile_select(f, bounds, window_max, K_long=100, t_imb=T_IMB_B200, t_ml=T_ML_B200, tol=APPROX_TOL_B200,
                   classes=None, p_stream=None):
    """Table II for the GPU variants: IMB -> long_row_split (dense
    long rows) or nnz_split; ML -> nnz_split with the x window; MB / CMP ->
    cta_stream (MB adds D8 codes when codable, else 16-bit deltas when the
    gaps fit); no class -> the CSR
    baseline (csr_vector), "not worth applying any". Precedence
    IMB > ML > MB/CMP. bounds: dict with p_csr, p_mb, p_ml, p_imb, p_cmp, p_peak;
    t_imb / t_ml / tol: Fig. 4's hyperparameters (default: the B200 grid
    search); classes: a given CLASS_* set instead of Fig. 4 (bounds unused);
    p_stream: the second stage (reading 30) -- the measured rate of
    the plain cta_stream kernel a CMP matrix was mapped to: if its indices
    are D8-codable and it reaches (1 - tol) P_MB, Fig. 4's MB test holds for
    the optimised kernel and MB (D8) is applied jointly."""
    forced = classes is not None
    if classes is None:
        classes = classify_profile(*(bounds[k] for k in ("p_csr", "p_mb", "p_ml", "p_imb", "p_cmp", "p_peak")),
                                   t_imb=t_imb, t_ml=t_ml, tol=tol)
    avg_s = f["avg_short"]
    longr = f["n_long"] > 0 and f["nnz_max"] > K_long * f["nnz_avg"]
    nblk = -(-int(f.get("n_cols", f["n"])) // 2048)
    dense_long = f["n_long"] > 0 and f["nnz_long"] >= 64 * f["n_long"] * nblk
    if classes & CLASS_IMB:
        variant = VARIANT_SPLIT if (longr and dense_long) else VARIANT_NNZSPLIT
    elif classes & CLASS_ML:
        variant = VARIANT_NNZSPLIT
    elif classes & (CLASS_MB | CLASS_CMP):
        variant = VARIANT_STREAM
    else:
        variant = VARIANT_VECTOR
    vs = min(32, max(2, _pow2ceil(int(math.ceil(avg_s))))) if avg_s > 0 else 2
    if variant == VARIANT_STREAM:
        vs = min(32, _pow2ceil(int(math.ceil(avg_s / 32.0)))) if avg_s > 32 else 1
    d16 = 0
    if classes & CLASS_MB and variant == VARIANT_STREAM:  # MB -> deltas: D8 when codable, else 16-bit
        d8_ok = f.get("n_deltas", D8_MAX + 1) <= D8_MAX and f["nnz_max"] <= D8_MAX_ROW and vs == 1
        d16 = 2 if d8_ok else (1 if f["maxgap"] <= 65535 else 0)
    if (p_stream and not forced and variant == VARIANT_STREAM and d16 == 0 and vs == 1
            and f.get("n_deltas", D8_MAX + 1) <= D8_MAX and 0 < f["nnz_max"] <= D8_MAX_ROW
            and f["nnz_max"] <= 1.25 * f["nnz_avg"] + 1.0 and p_stream >= (1 - tol) * bounds["p_mb"]):
        classes |= CLASS_MB
        d16 = 2
    xwin = bool(classes & CLASS_ML) and 8 * f["n"] <= window_max
    return Selection(variant, vs, d16, xwin, classes)


# ---- full Table I (reading 23) ------------------
def table1(rowptr, colind, n_cols=None, l2_bytes=126 * 2 ** 20, rp_bytes=None, line=16):
    """Every Table I feature, from the definitions (numpy): size (1 iff CSR +
    x + y fit in L2), density NNZ/(N*M), nnz_{min,max,avg,sd} over all rows,
    bw_i = last - first + 1 (inclusive), scatter_i = nnz_i/bw_i,
    clustering_i = ngroups_i/nnz_i (groups of consecutive columns),
    bw/scatter/clustering statistics over the non-empty rows,
    misses_avg = in-row gaps > line elements / N (all rows); population sd."""
    rp = _rp64(rowptr)
    ci = np.asarray(colind, np.int64)
    n = rp.size - 1
    m = int(n if n_cols is None else n_cols)
    nnz = int(rp[-1])
    lens = np.diff(rp)
    rpb = (np.asarray(rowptr).dtype.itemsize if rp_bytes is None else rp_bytes)
    ws = 12 * nnz + rpb * (n + 1) + 8 * m + 8 * n
    out = {"size_fits_l2": int(ws <= l2_bytes), "density": nnz / (n * m) if n and m else 0.0}
    out["nnz_min"] = float(lens.min()) if n else 0.0
    out["nnz_max"] = float(lens.max()) if n else 0.0
    out["nnz_avg"] = float(lens.mean()) if n else 0.0
    out["nnz_sd"] = float(np.sqrt(((lens - lens.mean()) ** 2).mean())) if n else 0.0
    ne = lens > 0
    first = ci[rp[:-1][ne]]
    last = ci[rp[1:][ne] - 1]
    bw = (last - first + 1).astype(np.float64)
    sc = lens[ne] / bw
    row_of = np.repeat(np.arange(n), lens)
    head = np.zeros(nnz, bool)
    head[rp[:-1][ne]] = True
    g = np.diff(ci)
    nh = ~head[1:]
    new_group = np.zeros(nnz, bool)
    new_group[1:] = nh & (g > 1)
    groups = 1 + np.bincount(row_of[new_group], minlength=n)
    cl = groups[ne] / lens[ne]
    misses = int(np.count_nonzero(nh & (g > line)))
    k = int(ne.sum())
    def stat(v):
        if k == 0:
            return 0.0, 0.0
        a = v.sum() / k
        return float(a), float(np.sqrt(((v - a) ** 2).sum() / k))
    out["bw_min"] = float(bw.min()) if k else 0.0
    out["bw_max"] = float(bw.max()) if k else 0.0
    out["bw_avg"], out["bw_sd"] = stat(bw)
    out["scatter_avg"], out["scatter_sd"] = stat(sc)
    out["clustering_avg"] = float(cl.sum() / k) if k else 0.0
    out["misses_avg"] = misses / n if n else 0.0
    out["n_nonempty"] = k
    return out
