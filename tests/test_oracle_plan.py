"""Pins for the oracle's plan structures, features, selection and formulas (CPU)."""
import json
import math
import os

import numpy as np
import pytest

import oracle
import synthgen as sg

GOLD = json.load(open(os.path.join(os.path.dirname(__file__), "golden", "spec_examples.json")))


def rp_of(lens):
    rp = np.zeros(len(lens) + 1, np.int64)
    np.cumsum(lens, out=rp[1:])
    return rp


def random_rowptrs(count=60, seed=7):
    g = np.random.default_rng(seed)
    out = []
    for t in range(count):
        n = int(g.integers(1, 300))
        kind = t % 4
        if kind == 0:
            lens = g.integers(0, 20, n)
        elif kind == 1:
            lens = g.choice([0, 0, 0, 1, 50], n)
        elif kind == 2:
            lens = np.minimum((g.pareto(1.1, n) * 4).astype(np.int64), 3000)
        else:
            lens = np.zeros(n, np.int64)
        out.append(rp_of(lens))
    return out


# ---- partition -------------------------
@pytest.mark.parametrize("ex", GOLD["partition"])
def test_partition_spec_examples(ex):
    assert oracle.shard_bounds(rp_of(ex["lengths"]), ex["G"]).tolist() == ex["bounds"]


def test_partition_vs_linear_scan():
    for rp in random_rowptrs():
        n, nnz = rp.size - 1, int(rp[-1])
        for G in (1, 2, 3, 8, 17):
            b = oracle.shard_bounds(rp, G)
            exp = [0] + [next((r for r in range(n + 1) if rp[r] >= -(-g * nnz // G)), n) for g in range(1, G)] + [n]
            assert b.tolist() == exp
            assert np.all(np.diff(b) >= 0)


def test_tile_rows_vs_linear_scan_and_ownership():
    for rp in random_rowptrs():
        n, nnz = rp.size - 1, int(rp[-1])
        for C in (1, 4, 16, 64):
            R = oracle.tile_rows(rp, C)
            T = oracle.tile_count(nnz, C)
            assert R.size == T + 1 and R[0] == 0 and R[-1] == n
            for k in range(1, T):
                assert R[k] == next((r for r in range(n + 1) if rp[r] >= k * C), n)
            # each row owned by exactly one tile, and its start lies in its tile window
            for k in range(T - 1):
                for r in range(R[k], R[k + 1]):
                    assert k * C <= rp[r] < (k + 1) * C


# ---- merge path ------------------------------------------------
def split_binary_search(rp, d):
    """The survey's binary-search split rule (a different algorithm from the oracle's merge)."""
    n, nnz = rp.size - 1, int(rp[-1])
    lo, hi = max(0, d - nnz), min(d, n)
    while lo < hi:
        mid = (lo + hi) // 2
        if rp[mid + 1] <= d - mid - 1:
            lo = mid + 1
        else:
            hi = mid
    return lo, d - lo


def test_merge_splits_vs_binary_search_and_invariants():
    for rp in random_rowptrs():
        n, nnz = rp.size - 1, int(rp[-1])
        for items in (1, 3, 7, 64):
            si, sj = oracle.merge_splits(rp, items)
            T = si.size - 1
            assert si[0] == 0 and sj[0] == 0 and si[-1] == n and sj[-1] == nnz
            for k in range(T + 1):
                d = min(k * items, n + nnz)
                assert (si[k], sj[k]) == split_binary_search(rp, d)
                i, j = si[k], sj[k]
                if i > 0 and j < nnz:
                    assert rp[i] <= j  # A[i-1] <= B[j] (ties to A)
                if i < n and j > 0:
                    assert j - 1 < rp[i + 1]  # B[j-1] < A[i]


# ---- long-row chunks -----------------------------------
@pytest.mark.parametrize("ex", GOLD["decompose"])
def test_decompose_examples_long_rows(ex):
    crow, cb, ce = oracle.long_chunks(rp_of(ex["lengths"]), ex["threshold"], 4)
    assert sorted(set(crow.tolist())) == ex["long_rows"]


def test_long_chunks_cover_long_rows_exactly():
    for rp in random_rowptrs():
        lens = np.diff(rp)
        for L, C in ((10, 4), (0, 1), (30, 64)):
            crow, cb, ce = oracle.long_chunks(rp, L, C)
            covered = []
            for r, b, e in zip(crow, cb, ce):
                assert rp[r] <= b < e <= rp[r + 1] and e - b <= C
                covered.extend(range(b, e))
            exp = [j for i in np.nonzero(lens > L)[0] for j in range(rp[i], rp[i + 1])]
            assert covered == exp  # disjoint, ordered, complete (decomposition conservation S:149)


# ---- D16 delta colind -------------------------
def test_delta_width_spec_examples():
    for ex in GOLD["delta_width"]:
        if ex["rows"] == "banded bandwidth 3":
            m = sg.small_suite(0)[-1][1]  # banded
            w, mg, _, _ = oracle.d16_encode(m.rowptr, m.colind)
            assert mg <= 2
        else:
            rows = ex["rows"]
            rp = rp_of([len(r) for r in rows])
            w, mg, _, _ = oracle.d16_encode(rp, np.concatenate([np.array(r, np.int32) for r in rows]))
        assert w == ex["width"]


@pytest.mark.parametrize("name,m", sg.small_suite(5))
def test_d16_round_trip(name, m):
    w, mg, dcol, head = oracle.d16_encode(m.rowptr, m.colind)
    if w == 0:
        assert mg > 65535
        return
    assert np.array_equal(oracle.d16_decode(m.rowptr, dcol, head), m.colind)
    rp = m.rowptr.astype(np.int64)
    empty = np.diff(rp) == 0
    assert np.all(head[empty] == m.n)  # sentinel
    assert np.all(dcol[rp[:-1][~empty]] == 0)  # placeholder delta at heads


@pytest.mark.parametrize("n", [3, 5, 24])
def test_stencil_maxgap_closed_forms(n):
    m7 = sg.stencil(n, 7)
    m27 = sg.stencil(n, 27)
    assert oracle.d16_encode(m7.rowptr, m7.colind)[1] == n * n
    assert oracle.d16_encode(m27.rowptr, m27.colind)[1] == n * n - n - 1
    w, _, dcol, head = oracle.d16_encode(m7.rowptr, m7.colind)
    assert np.array_equal(oracle.d16_decode(m7.rowptr, dcol, head), m7.colind)


def test_config_widths():
    # C2 (128^3): maxgap 128^2 = 16384 -> 16-bit; C5 (384^3): 384^2-384-1 = 147071 -> none
    assert 128 * 128 <= 65535 < 384 * 384 - 384 - 1
    m = sg.config(1)
    assert oracle.d16_encode(m.rowptr, m.colind)[0] == 16


def test_tile_anchor():
    ci = np.arange(100, dtype=np.int32) * 3
    assert oracle.tile_anchor(ci, 16).tolist() == (np.arange(0, 100, 16) * 3).tolist()


# ---- features (Table I) -------------------------------------------
def test_features_spec_example():
    g = GOLD["features_sd"]
    rp = rp_of(g["lengths"])
    f = oracle.features(rp, np.array([0, 0, 1, 0, 1, 2], np.int32))
    assert (f["nnz_min"], f["nnz_max"], f["nnz_avg"]) == (g["nnz_min"], g["nnz_max"], g["nnz_avg"])
    assert abs(f["nnz_sd"] - math.sqrt(g["nnz_sd_sq_num"] / g["nnz_sd_sq_den"])) < 1e-15
    r = GOLD["features_row"]
    f = oracle.features(rp_of([4]), np.array(r["colind"], np.int32), line_elems=r["line_elems"])
    assert f["misses"] == r["misses"] and f["maxgap"] == r["maxgap"]


@pytest.mark.parametrize("n", [2, 3, 10])
def test_features_stencil_closed_forms(n):
    f = oracle.features(sg.stencil(n, 7).rowptr, sg.stencil(n, 7).colind)
    N = n ** 3
    assert f["nnz"] == 7 * N - 6 * n * n and f["nnz_min"] == 4 and f["nnz_max"] == (7 if n >= 3 else 4)
    assert f["nnz_avg"] == f["nnz"] / N
    # sd from the closed-form length histogram: lengths 7 - #boundary faces
    i = np.arange(N)
    lens = 7 - sum(((c == 0).astype(int) + (c == n - 1)) for c in (i % n, (i // n) % n, i // (n * n)))
    assert abs(f["nnz_sd"] - lens.std()) < 1e-12
    f27 = oracle.features(sg.stencil(n, 27).rowptr, sg.stencil(n, 27).colind)
    assert f27["nnz"] == (3 * n - 2) ** 3 and f27["nnz_min"] == 8 and f27["nnz_max"] == (27 if n >= 3 else 8)


def test_features_configs_small():
    f1 = oracle.features(sg.config(1).rowptr, sg.config(1).colind)
    assert f1["nnz_min"] == f1["nnz_max"] == 9 and f1["nnz_sd"] == 0.0
    m4 = sg.config(4, small=True)
    f4 = oracle.features(m4.rowptr, m4.colind)
    assert f4["nnz_min"] == 15 and f4["nnz_max"] == 4500 and f4["n_long"] == 10 and f4["nnz_long"] == 45000


# ---- validation ------------------------------------------
@pytest.mark.parametrize("rp,ci,n,nnz,code,where", [
    ([0, 1, 2], [0, 1], 2, 2, 0, -1),
    ([1, 1, 2], [0, 1], 2, 2, 1, 0),
    ([0, 1, 3], [0, 1], 2, 2, 2, 2),
    ([0, 2, 1, 2], [0, 1], 3, 2, 3, 1),
    ([0, 1, 2], [0, 2], 2, 2, 4, 1),
    ([0, 1, 2], [-1, 0], 2, 2, 4, 0),
    ([0, 2, 4], [0, 1, 1, 1], 2, 4, 5, 3),
    ([0, 2, 4], [1, 0, 0, 1], 2, 4, 5, 1),
    ([0, 0, 0], [], 2, 0, 0, -1),
])
def test_validate_hand_cases(rp, ci, n, nnz, code, where):
    assert oracle.validate(n, nnz, np.array(rp), np.array(ci, np.int32)) == (code, where)


# ---- selection (Table II) ---------------------------
L2 = 126 * 2 ** 20
WIN = 128 * 2 ** 20


def test_select_rule_table_on_closed_form_features():
    def feat(n, nnz, avg_s, sd_s, n_empty=0, n_long=0, nnz_max=0, maxgap=0, misses=0, nnz_long=0, n_big_gaps=129,
             n_deltas=257):
        return dict(n=n, nnz=nnz, avg_short=avg_s, sd_short=sd_s, n_empty=n_empty, n_long=n_long,
                    nnz_max=nnz_max, nnz_avg=nnz / n, maxgap=maxgap, misses=misses, nnz_long=nnz_long, n_cols=n,
                    n_big_gaps=n_big_gaps, n_deltas=n_deltas)
    S = oracle
    # C2: 7-pt 128^3 (closed forms above): regular, 217 MB > L2/2, maxgap 16384,
    # 10 distinct row-relative deltas (test_d8_config_dictionaries) -> stream + D8
    s = S.select(feat(2097152, 14581760, 6.953125, 0.2148, nnz_max=7, maxgap=16384, misses=8323072, n_deltas=10),
                 L2, WIN, 4)
    assert (s.variant, s.d16, s.xwin, s.vs) == (S.VARIANT_STREAM, 2, False, 1) and s.classes & S.CLASS_MB
    # C5: 27-pt 384^3: regular, 15 deltas -> D8 (maxgap 147071: no 16-bit deltas;
    # 4 distinct gaps >= 65472: escape codes possible but forced only, reading 21)
    s = S.select(feat(56623104, 1520875000, 26.86, 0.5, nnz_max=27, maxgap=147071, misses=10 ** 8, n_big_gaps=4,
                      n_deltas=15), L2, WIN, 8)
    assert (s.variant, s.d16, s.vs) == (S.VARIANT_STREAM, 2, 1)  # rows <= 32 nnz: one lane per row
    # the same without a codable dictionary (> 256 deltas) keeps int32 colind:
    # 16-bit deltas are never auto-selected (reading 9)
    s = S.select(feat(5832000, 155235000, 26.6, 0.6, nnz_max=27, maxgap=32219, misses=10 ** 7, n_big_gaps=0), L2,
                 WIN, 8)
    assert s.d16 == 0 and s.variant == S.VARIANT_STREAM
    # irregular rows (longest > 1.25 x average + 1): no D8 even when codable
    s = S.select(feat(15625000, 109000000, 6.98, 0.2, nnz_max=12, maxgap=62250, misses=10 ** 7, n_big_gaps=0,
                      n_deltas=40), L2, WIN, 4)
    assert s.d16 == 0
    # rows longer than 255: no D8
    s = S.select(feat(1000000, 300000000, 300.0, 0.0, nnz_max=300, maxgap=100, misses=0, n_deltas=5), L2, WIN, 8)
    assert s.d16 == 0
    # uniform random rows (4M x 8/row: every nonzero opens a new x line) ->
    # scattered columns -> nnz_split (reading 24), not the row-walking stream
    s = S.select(feat(4000000, 36000000, 9.0, 0.3, maxgap=3999000, misses=35900000), L2, WIN, 4)
    assert s.variant == S.VARIANT_NNZSPLIT and s.classes & S.CLASS_ML and not s.classes & S.CLASS_IMB
    # the same pattern below 2^20 nonzeros stays on the launch-bound csr_vector
    s = S.select(feat(100000, 900000, 9.0, 0.3, maxgap=99000, misses=899000), L2, WIN, 4)
    assert s.variant == S.VARIANT_VECTOR
    # C1: 1.28 MB working set, 90,000 nonzeros -> launch-bound: csr_vector VS 16, no MB, no D16
    s = S.select(feat(10000, 90000, 9.0, 0.0, maxgap=9000, misses=80000), L2, WIN, 4)
    assert (s.variant, s.vs, s.d16, s.classes & S.CLASS_MB) == (S.VARIANT_VECTOR, 16, 0, 0)
    # C3-like: half the rows empty, sparse long rows (11.4M nnz over 1794 rows of
    # 4.2M columns: far below 64 per 2048-column block) -> nnz_split, IMB + ML
    s = S.select(feat(4194304, 65244537, 12.8, 78.5, n_empty=2185429, n_long=1794, nnz_max=97958,
                      maxgap=4165791, misses=56437921, nnz_long=11392466), L2, WIN, 4)
    assert s.variant == S.VARIANT_NNZSPLIT and s.classes & S.CLASS_IMB and s.xwin and s.classes & S.CLASS_ML
    # skew without long rows -> nnz_split
    s = S.select(feat(4194304, 20000000, 4.8, 9.0, n_empty=2185429, n_long=0, nnz_max=3000,
                      maxgap=4165791, misses=19000000), L2, WIN, 4)
    assert s.variant == S.VARIANT_NNZSPLIT and s.classes & S.CLASS_IMB
    # C4-like: 100 dense long rows (200,000 of 1M columns: ~410 per 2048-column
    # block) -> long_row_split (column-tiled long rows + nnz_split bin)
    s = S.select(feat(1000000, 34998500, 15.0, 0.0, n_long=100, nnz_max=200000, maxgap=900000,
                      misses=34000000, nnz_long=20000000), L2, WIN, 4)
    assert (s.variant, s.vs) == (S.VARIANT_SPLIT, 16) and s.classes & S.CLASS_IMB
    # the same long rows 10x sparser (41 per block) -> nnz_split
    s = S.select(feat(1000000, 16998500, 15.0, 0.0, n_long=100, nnz_max=20000, maxgap=900000,
                      misses=16000000, nnz_long=2000000), L2, WIN, 4)
    assert s.variant == S.VARIANT_NNZSPLIT
    # medium regular rows -> csr_vector with VS = pow2ceil(avg)
    s = S.select(feat(100000, 4000000, 40.0, 2.0, maxgap=10), L2, WIN, 4)
    assert (s.variant, s.vs) == (S.VARIANT_VECTOR, 32)


# ---- formulas ----------------------------------------------------------------
def test_bounds_spec_numbers():
    b = GOLD["bounds"]
    assert abs(oracle.p_mb(b["nnz"], b["n"], b["bmax"]) / b["p_mb"] - 1) < b["p_mb_rel_tol"]
    assert oracle.p_peak(b["nnz"], b["n"], b["bmax"]) >= oracle.p_mb(b["nnz"], b["n"], b["bmax"])
    # NNZ -> inf limit of P_peak / P_MB is 1.5
    assert abs(oracle.p_peak(10 ** 12, 10, 1.0) / oracle.p_mb(10 ** 12, 10, 1.0) - 1.5) < 1e-9


def test_amortization_and_harmonic_mean():
    a = GOLD["amortization"]
    assert round(oracle.n_iters_min(a["t_pre"], a["t_base"], a["t_sel"]), 9) == a["n_iters_min"]
    assert oracle.n_iters_min(1.0, 0.005, 0.010) == math.inf
    for h in GOLD["harmonic_mean"]:
        assert abs(oracle.harmonic_mean(h["rates"]) - h["hm"]) < 1e-15


def test_algorithmic_bytes_configs():
    # C2 216,924,164 B; C4 439,982,004 B; C5 19,609,454,504 B
    assert oracle.algorithmic_bytes(2097152, 14581760, 4) == 216924164
    assert oracle.algorithmic_bytes(1000000, 34998500, 4) == 439982004
    assert oracle.algorithmic_bytes(56623104, 1520875000, 8) == 19609454504


# ---- nnz_split structures (reading 19) ---------------------------------
def test_nonempty_rows_and_nz_tiles_hand_example():
    # lengths [0, 3, 0, 0, 1, 300, 0, 2]: non-empty rows 1, 4, 5, 7
    lens = np.array([0, 3, 0, 0, 1, 300, 0, 2])
    rp = np.concatenate([[0], np.cumsum(lens)])
    rowmap, rpc = oracle.nonempty_rows(rp)
    assert rowmap.tolist() == [1, 4, 5, 7, 8] and rpc.tolist() == [0, 3, 4, 304, 306]
    # nonzero 256 lies in row 5 (q = 2), so tile 1 starts inside it
    assert oracle.nz_tiles(rpc).tolist() == [0, 2, 4]
    assert oracle.nz_tiles(rpc, W=4).tolist()[:3] == [0, 2, 2]


@pytest.mark.parametrize("seed", range(6))
def test_nz_structures_rederived(seed):
    g = np.random.default_rng(seed)
    n = int(g.integers(1, 3000))
    lens = g.integers(0, 40, n) * (g.random(n) < 0.6)
    lens[g.integers(0, n, 3)] = g.integers(0, 2000, 3)
    rp = np.concatenate([[0], np.cumsum(lens)])
    rowmap, rpc = oracle.nonempty_rows(rp)
    nz = np.flatnonzero(lens > 0)
    assert np.array_equal(rowmap[:-1], nz) and rowmap[-1] == n
    assert np.array_equal(rpc[:-1], rp[nz]) and rpc[-1] == rp[-1]
    for W in (256, 7):
        tq = oracle.nz_tiles(rpc, W)
        T = -(-int(rp[-1]) // W)
        assert tq.size == T + 1 and tq[-1] == rpc.size - 1
        k = np.arange(T)
        # searchsorted re-derivation: last q with rpc[q] <= k*W
        assert np.array_equal(tq[:-1], np.searchsorted(rpc, k * W, side="right") - 1)
        # ownership: nonzero k*W lies in row rowmap[tq[k]]
        for kk in k[:: max(1, T // 50)]:
            q = tq[kk]
            assert rpc[q] <= kk * W < rpc[q + 1]


# ---- nnz_split hot-x set (reading 20) ------------------------------------
def test_hot_columns_hand_example():
    # column counts: c0:5, c1:1, c2:3, c3:3, c4:0, c5:2
    ci = np.array([0, 0, 0, 0, 0, 1, 2, 2, 2, 3, 3, 3, 5, 5], np.int32)
    hot, cov = oracle.hot_columns(ci, 6, K=4)   # cnt >= 2: columns 0, 2, 3, 5
    assert hot.tolist() == [0, 2, 3, 5] and cov == 13
    hot, cov = oracle.hot_columns(ci, 6, K=6)   # cnt >= 1: 5 columns -> 4
    assert hot.tolist() == [0, 1, 2, 3] and cov == 12
    hot, cov = oracle.hot_columns(ci, 6, K=2)   # cnt >= 5 only c0 -> 0 columns (even)
    assert hot.tolist() == [] and cov == 0


@pytest.mark.parametrize("seed", range(4))
def test_hot_columns_threshold_maximal(seed):
    g = np.random.default_rng(seed)
    n = 5000
    ci = np.minimum((g.pareto(1.1, 40000) * 10).astype(np.int64), n - 1).astype(np.int32)
    cnt = np.bincount(ci, minlength=n)
    for K in (16, 256, 1000):
        hot, cov = oracle.hot_columns(ci, n, K)
        assert hot.size <= K and hot.size % 2 == 0 and np.all(np.diff(hot) > 0)
        assert cov == cnt[hot].sum()
        # brute force: t = the smallest count >= 1 whose columns (cnt >= t)
        # number <= K, unless even the top bucket exceeds K
        t = next((v for v in range(1, 4096) if np.count_nonzero(cnt >= v) <= K), 4095)
        cand = np.flatnonzero(cnt >= t)
        assert np.array_equal(hot, cand[:min(cand.size, K) & ~1])


# ---- escape-coded D16 (reading 21) --------------------------------------
def test_d16_escape_hand_example():
    rp = np.array([0, 4, 6])
    ci = np.array([0, 70000, 70001, 140001, 5, 100005], np.int32)  # gaps 70000, 1, 70000 | 100000
    assert oracle.d16_encode(rp, ci)[0] == 0  # plain 16-bit deltas cannot hold 70000
    w, mg, dcol, head, esc = oracle.d16_encode_esc(rp, ci)
    assert (w, mg) == (16, 100000) and esc.tolist() == [70000, 100000]
    assert dcol.tolist() == [0, 65472, 1, 65472, 0, 65473] and head.tolist() == [0, 5]
    assert np.array_equal(oracle.d16_decode_esc(rp, dcol, head, esc), ci)
    assert oracle.big_gap_count(rp, ci) == 2


def test_d16_escape_limits_and_stencil():
    # 65 distinct large gaps -> not encodable; 64 -> encodable
    for k, ok in ((64, True), (65, False)):
        ci = np.cumsum(np.concatenate([[0], 65472 + np.arange(k)])).astype(np.int32)
        rp = np.array([0, ci.size])
        w = oracle.d16_encode_esc(rp, ci)[0]
        assert (w == 16) == ok and oracle.big_gap_count(rp, ci) == k
    # 27-point stencil n = 260: exactly the 4 closed-form large gaps, round trip
    m = sg.stencil(260, 27, rp64=True, rows=(0, 200000))
    n = 260
    w, mg, dcol, head, esc = oracle.d16_encode_esc(m.rowptr, m.colind)
    assert w == 16 and esc.tolist() == [n * n - 2 * n - 2, n * n - 2 * n - 1, n * n - n - 2, n * n - n - 1]
    assert np.array_equal(oracle.d16_decode_esc(m.rowptr, dcol, head, esc), m.colind)


# ---- profile-guided classifier (Fig. 4) ------------------
def test_classify_profile_spec_examples():
    C = oracle
    neutral = dict(p_csr=1.0, p_mb=2.0, p_ml=1.0, p_imb=1.0, p_cmp=3.0, p_peak=4.0)
    assert C.classify_profile(**neutral) == 0                              # no rule fires
    assert C.classify_profile(**{**neutral, "p_ml": 1.30}) == C.CLASS_ML   # 1.30 > 1.25
    assert C.classify_profile(**{**neutral, "p_imb": 1.24}) == 0           # strict >
    assert C.classify_profile(**{**neutral, "p_imb": 1.2401}) == C.CLASS_IMB
    assert C.classify_profile(**{**neutral, "p_cmp": 5.0}) & C.CLASS_CMP   # P_CMP > P_peak
    assert C.classify_profile(**{**neutral, "p_cmp": 1.5}) == C.CLASS_CMP  # P_MB > P_CMP
    # MB: P_CSR within 10 % of P_MB and P_MB < P_CMP < P_peak
    assert C.classify_profile(**{**neutral, "p_csr": 1.8}) == C.CLASS_MB
    assert C.classify_profile(**{**neutral, "p_csr": 1.79}) == 0
    # all four at once is impossible only for MB + (P_MB > P_CMP) CMP; MB + IMB + ML is fine
    assert C.classify_profile(p_csr=1.8, p_mb=2.0, p_ml=3.0, p_imb=3.0, p_cmp=3.0, p_peak=4.0) == \
        C.CLASS_MB | C.CLASS_ML | C.CLASS_IMB


def test_classify_profile_properties():
    g = np.random.default_rng(3)
    for _ in range(2000):
        b = dict(zip(("p_csr", "p_mb", "p_ml", "p_imb", "p_cmp", "p_peak"), g.uniform(0.5, 3.0, 6)))
        c = oracle.classify_profile(**b)
        # monotone in P_ML
        assert (oracle.classify_profile(**{**b, "p_ml": b["p_ml"] * 2}) & oracle.CLASS_ML) >= (c & oracle.CLASS_ML)
        # MB and the P_MB > P_CMP branch of CMP exclude each other
        if b["p_mb"] > b["p_cmp"]:
            assert not (c & oracle.CLASS_MB)


def test_profile_select_table2_mapping():
    f = dict(n=1000, nnz=20000, avg_short=20.0, n_long=0, nnz_max=30, nnz_avg=20.0, n_cols=1000, nnz_long=0,
             maxgap=100)
    b = dict(p_csr=1.0, p_mb=2.0, p_ml=1.0, p_imb=1.0, p_cmp=3.0, p_peak=4.0)
    S = oracle

    def ps(f, b, w):  # the mapping under the paper's Fig. 4 thresholds
        return oracle.profile_select(f, b, w, t_imb=oracle.T_IMB, t_ml=oracle.T_ML, tol=oracle.APPROX_TOL)
    assert ps(f, b, 1 << 27).variant == S.VARIANT_VECTOR                     # no class: baseline
    assert ps(f, {**b, "p_imb": 2.0}, 1 << 27).variant == S.VARIANT_NNZSPLIT  # IMB, no long rows
    s = ps(f, {**b, "p_ml": 2.0}, 1 << 27)
    assert s.variant == S.VARIANT_NNZSPLIT and s.xwin                                       # ML
    s = ps(f, {**b, "p_csr": 1.9}, 1 << 27)
    assert (s.variant, s.d16, s.vs) == (S.VARIANT_STREAM, 1, 1)                             # MB -> stream + D16
    s = ps({**f, "n_deltas": 12}, {**b, "p_csr": 1.9}, 1 << 27)
    assert (s.variant, s.d16, s.vs) == (S.VARIANT_STREAM, 2, 1)                             # MB, codable -> D8
    s = ps(f, {**b, "p_cmp": 1.0}, 1 << 27)
    assert (s.variant, s.d16) == (S.VARIANT_STREAM, 0)                                      # CMP
    fl = {**f, "n_long": 10, "nnz_max": 5000, "nnz_long": 50000}
    assert ps(fl, {**b, "p_imb": 2.0}, 1 << 27).variant == S.VARIANT_SPLIT    # dense long rows


# ---- full Table I (reading 23) --------------------------------
def test_table1_spec_worked_rows():
    rp = np.array([0, 4])
    ci = np.array([4, 5, 6, 20], np.int32)
    t = oracle.table1(rp, ci, n_cols=30, line=8)
    assert t["bw_avg"] == 17 and abs(t["scatter_avg"] - 4 / 17) < 1e-15 and t["clustering_avg"] == 0.5
    assert t["misses_avg"] == 1.0  # gap 14 > 8 elements (S:416, 64-B lines)
    assert oracle.table1(rp, ci, n_cols=30)["misses_avg"] == 0.0  # 128-B lines: 14 <= 16
    # lengths [1, 2, 3]: nnz_sd = sqrt(2/3)
    t = oracle.table1(np.array([0, 1, 3, 6]), np.array([0, 0, 1, 0, 1, 2], np.int32), n_cols=3)
    # consecutive columns: one group per row, clustering_i = 1 / nnz_i
    assert abs(t["nnz_sd"] - math.sqrt(2 / 3)) < 1e-15 and abs(t["clustering_avg"] - (1 + 1 / 2 + 1 / 3) / 3) < 1e-15
    # diagonal: bw 1, scatter 1, clustering 1, no misses
    n = 50
    t = oracle.table1(np.arange(n + 1), np.arange(n, dtype=np.int32))
    assert (t["bw_min"], t["bw_max"], t["scatter_avg"], t["scatter_sd"], t["clustering_avg"], t["misses_avg"]) == \
        (1.0, 1.0, 1.0, 0.0, 1.0, 0.0)
    assert t["density"] == 1 / n and t["size_fits_l2"] == 1


def test_table1_bruteforce_rows():
    for name, m in sg.small_suite(seed=11)[:6]:
        t = oracle.table1(m.rowptr, m.colind, n_cols=m.x.size)
        rp = m.rowptr.astype(np.int64)
        bws, scs, cls, miss = [], [], [], 0
        for i in range(rp.size - 1):
            row = m.colind[rp[i]:rp[i + 1]].astype(np.int64)
            if row.size == 0:
                continue
            bws.append(row[-1] - row[0] + 1)
            scs.append(row.size / bws[-1])
            gaps = np.diff(row)
            cls.append((1 + int(np.sum(gaps > 1))) / row.size)
            miss += int(np.sum(gaps > 16))
        if bws:
            assert t["bw_min"] == min(bws) and t["bw_max"] == max(bws)
            assert abs(t["bw_avg"] - np.mean(bws)) <= 1e-12 * max(1.0, np.mean(bws))
            assert abs(t["scatter_sd"] - np.std(scs)) <= 1e-12
            assert abs(t["clustering_avg"] - np.mean(cls)) <= 1e-12
        assert t["misses_avg"] == miss / (rp.size - 1), name


# ---- D8: dictionary-coded 8-bit deltas (reading 26) ------
def _d8_stencil_dict(n, pts):
    """Closed form from the stencil geometry (not the delta formula): heads =
    -(smallest present neighbour offset) over the boundary cases; in-row gaps
    between consecutive present offsets (7-pt: sums of adjacent base gaps; 27-pt:
    1 inside an x-run, n + xmin - xmax on a y step, n^2 + (ymin-ymax) n +
    (xmin-xmax) on a z step, with xmin-xmax, ymin-ymax in {-2, -1})."""
    if pts == 7:
        heads = {-n * n, -n, -1, 0}
        gaps = {1, n - 1, n, n * n - n, n * n - 1, n * n}
    else:
        heads = {-(a * n * n + b * n + c) for a in (0, 1) for b in (0, 1) for c in (0, 1)}
        gaps = {1, n - 2, n - 1} | {n * n + dy * n + dx for dy in (-2, -1) for dx in (-2, -1)}
    return sorted(heads | gaps)


@pytest.mark.parametrize("n", [3, 4, 7, 16])
@pytest.mark.parametrize("pts", [7, 27])
def test_d8_stencil_dictionary_closed_form(n, pts):
    m = sg.stencil(n, pts)
    want = _d8_stencil_dict(n, pts)
    nd, d = oracle.d8_dict(m.rowptr, m.colind)
    assert nd == len(want) and d.tolist() == want
    enc = oracle.d8_encode(m.rowptr, m.colind)
    assert enc is not None and enc[0].tolist() == want
    assert np.array_equal(enc[2], np.diff(m.rowptr.astype(np.int64)))
    assert np.array_equal(oracle.d8_decode(*enc), m.colind)  # round trip


def test_d8_config_dictionaries():
    # C2 7-pt 128^3: 10 codes; C5 27-pt 384^3: 15 codes (closed forms above)
    assert _d8_stencil_dict(128, 7) == [-16384, -128, -1, 0, 1, 127, 128, 16256, 16383, 16384]
    assert len(_d8_stencil_dict(384, 27)) == 15
    m = sg.stencil(128, 7, rows=(0, 40000))
    assert oracle.d8_dict(m.rowptr, m.colind)[0] <= 10
    # C1 (uniform random columns): far more than 256 distinct deltas
    m1 = sg.config(1)
    assert oracle.d8_dict(m1.rowptr, m1.colind)[0] == 257 and oracle.d8_encode(m1.rowptr, m1.colind) is None


def test_d8_hand_example_and_limits():
    # rows: [2, 5, 6], [], [0, 3] (row ids 0, 1, 2): deltas 2,3,1 | - | -2,3
    rp = rp_of([3, 0, 2])
    ci = np.array([2, 5, 6, 0, 3], np.int32)
    d, codes, rlen = oracle.d8_encode(rp, ci)
    assert d.tolist() == [-2, 1, 2, 3]
    assert codes.tolist() == [2, 3, 1, 0, 3] and rlen.tolist() == [3, 0, 2]
    assert oracle.d8_decode(d, codes, rlen).tolist() == ci.tolist()
    # diagonal: one delta (0), every code 0
    n = 50
    d, codes, _ = oracle.d8_encode(np.arange(n + 1), np.arange(n, dtype=np.int32))
    assert d.tolist() == [0] and not codes.any()
    # exactly 256 distinct head deltas: codable; 257: not
    for k, ok in ((256, True), (257, False)):
        ci = (np.arange(k) * 2).astype(np.int32)  # row i -> column 2i: head delta i
        enc = oracle.d8_encode(np.arange(k + 1), ci)
        assert (enc is not None) == ok
        if ok:
            assert enc[0].tolist() == list(range(k)) and enc[1].tolist() == list(range(k))
    # row lengths: 255 codable, 256 not (u8 lengths), even with 2 distinct deltas
    for L_, ok in ((255, True), (256, False)):
        enc = oracle.d8_encode(rp_of([L_]), np.arange(L_, dtype=np.int32))
        assert (enc is not None) == ok


@pytest.mark.parametrize("seed", range(6))
def test_d8_round_trip_random_banded(seed):
    # banded rows drawn from a small gap alphabet: codable, decode(encode) == colind
    g = np.random.default_rng(seed)
    n = 3000
    lens = g.integers(0, 30, n)
    rp = rp_of(lens)
    ci = np.empty(int(rp[-1]), np.int32)
    for i in range(n):
        if lens[i] == 0:
            continue
        steps = g.choice([1, 2, 7, 40, 333], lens[i])
        steps[0] = g.integers(-min(i, 60), 60)
        ci[rp[i]:rp[i + 1]] = i + np.cumsum(steps)
    enc = oracle.d8_encode(rp, ci)
    nd = oracle.d8_dict(rp, ci)[0]
    if nd > 256:
        assert enc is None
        return
    d, codes, rlen = enc
    assert np.all(np.diff(d) > 0)  # strictly ascending, distinct
    assert np.array_equal(oracle.d8_decode(d, codes, rlen), ci)


# ---- short-row statistics and empty rows (Table I nnz stats over len <= L_split) ----
@pytest.mark.parametrize("seed", range(4))
def test_features_short_row_stats_vs_numpy(seed):
    g = np.random.default_rng(seed)
    n = 2000
    lens = g.choice([0, 0, 1, 3, 9, 40, 700], n).astype(np.int64)
    # L_split edge rows: exactly 4096 (short) and 4097 (long), plus longer ones
    lens[g.choice(n, 6, replace=False)] = [4096, 4096, 4097, 4097, 5000, 9000]
    rp = rp_of(lens)
    ci = np.concatenate([np.arange(L, dtype=np.int32) for L in lens])
    f = oracle.features(rp, ci, n_cols=10000)
    short = lens[lens <= 4096]
    assert f["n_short"] == short.size and f["max_short"] == short.max()
    assert f["n_empty"] == int((lens == 0).sum())
    assert f["n_long"] == int((lens > 4096).sum()) and f["nnz_long"] == int(lens[lens > 4096].sum())
    assert f["s1_short"] == short.sum() and f["s2_short"] == int((short * short).sum())
    assert abs(f["avg_short"] - short.mean()) <= 1e-15 * short.mean()
    assert abs(f["sd_short"] - short.std()) <= 1e-12 * short.std()
    assert abs(f["nnz_sd"] - lens.std()) <= 1e-12 * lens.std()
    for L in (4096, 4097, 100):
        fl = oracle.features(rp, ci, L_split=L, n_cols=10000)
        sh = lens[lens <= L]
        assert fl["n_short"] == sh.size and fl["max_short"] == sh.max()
        assert abs(fl["sd_short"] - sh.std()) <= 1e-12 * max(sh.std(), 1)


def test_features_all_empty_and_all_long():
    f = oracle.features(np.zeros(6, np.int64), np.zeros(0, np.int32))
    assert f["n_empty"] == 5 and f["n_short"] == 5 and f["avg_short"] == 0.0 and f["sd_short"] == 0.0
    lens = np.array([5000, 6000])
    f = oracle.features(rp_of(lens), np.concatenate([np.arange(L, dtype=np.int32) for L in lens]), n_cols=6000)
    assert f["n_short"] == 0 and f["n_long"] == 2 and f["avg_short"] == 0.0 and f["max_short"] == 0


# ---- B200 grid search of Fig. 4's hyperparameters (reading 29) -------
def test_tuned_thresholds_reproduce_the_recorded_search():
    """profiles/r02_profile_tuning.json holds the measured bounds and plan times
    of the grid search (tools/tune_profile.py); its chosen point is the
    oracle's (and the library's) B200 default, every matrix's recorded classes
    follow from Fig. 4 on its bounds, and the tool's Fig. 4 is the oracle's."""
    import json, sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    d = json.load(open(os.path.join(root, "profiles", "r02_profile_tuning.json")))
    assert (d["chosen"]["t_imb"], d["chosen"]["t_ml"], d["chosen"]["tol"]) == \
        (oracle.T_IMB_B200, oracle.T_ML_B200, oracle.APPROX_TOL_B200)
    assert (d["paper_knc"]["t_imb"], d["paper_knc"]["t_ml"], d["paper_knc"]["tol"]) == (oracle.T_IMB, oracle.T_ML, oracle.APPROX_TOL)
    names = {"MB": oracle.CLASS_MB, "ML": oracle.CLASS_ML, "IMB": oracle.CLASS_IMB, "CMP": oracle.CLASS_CMP}
    for r in d["matrices"]:
        b = r["bounds_gflops"]
        args = [b[k] for k in ("p_csr", "p_mb", "p_ml", "p_imb", "p_cmp", "p_peak")]
        for tag, t in (("b200", (oracle.T_IMB_B200, oracle.T_ML_B200, oracle.APPROX_TOL_B200)), ("paper", (oracle.T_IMB, oracle.T_ML, oracle.APPROX_TOL))):
            c = oracle.classify_profile(*args, t_imb=t[0], t_ml=t[1], tol=t[2])
            assert c == sum(names[n] for n in r["classes_" + tag]), (r["name"], tag)
            assert r["plan_" + tag] == r["plan_of_classes"][str(c)]
    # the tuned point scores at least the paper's on the recorded set
    assert d["score_chosen"]["geomean"] >= d["score_paper"]["geomean"]
    sys.path.insert(0, os.path.join(root, "tools"))
    import tune_profile as T
    rng = np.random.default_rng(29)
    for _ in range(2000):
        v = rng.uniform(0.2, 5.0, 6)
        t = (rng.uniform(1, 3), rng.uniform(1, 3), rng.uniform(0.05, 0.9))
        b = dict(zip(("p_csr", "p_mb", "p_ml", "p_imb", "p_cmp", "p_peak"), v))
        assert T.classify(b, *t) == oracle.classify_profile(*v, t_imb=t[0], t_ml=t[1], tol=t[2])


def test_profile_select_forced_classes_follow_table2():
    """classes= bypasses Fig. 4: the Table II mapping of a given class set
    (IMB > ML > MB/CMP precedence)."""
    f = oracle.features(np.array([0, 2, 4, 6]), np.array([0, 1, 1, 2, 0, 2], np.int32))
    assert oracle.profile_select(f, None, 1 << 30, classes=0).variant == oracle.VARIANT_VECTOR
    assert oracle.profile_select(f, None, 1 << 30, classes=oracle.CLASS_CMP).variant == oracle.VARIANT_STREAM
    assert oracle.profile_select(f, None, 1 << 30, classes=oracle.CLASS_ML | oracle.CLASS_CMP).variant == oracle.VARIANT_NNZSPLIT
    assert oracle.profile_select(f, None, 1 << 30, classes=oracle.CLASS_IMB | oracle.CLASS_ML).variant == oracle.VARIANT_NNZSPLIT
    for c in range(16):
        assert oracle.profile_select(f, None, 1 << 30, classes=c).classes == c


def test_profile_select_second_stage():
    """Reading 30: a CMP matrix mapped to the plain stream kernel gets MB and
    D8 when that kernel reaches (1 - tol) P_MB and its indices are codable."""
    f = dict(n=1000, nnz=7000, avg_short=7.0, n_long=0, nnz_max=7, nnz_avg=7.0, n_cols=1000, nnz_long=0,
             maxgap=100, n_deltas=7)
    b = dict(p_csr=1.0, p_mb=3.0, p_ml=1.0, p_imb=1.0, p_cmp=1.3, p_peak=4.0)  # P_MB > P_CMP: CMP
    w = 1 << 27
    base = oracle.profile_select(f, b, w)
    assert (base.variant, base.d16, base.classes) == (oracle.VARIANT_STREAM, 0, oracle.CLASS_CMP)
    s = oracle.profile_select(f, b, w, p_stream=2.7)  # 2.7 >= 0.9 * 3.0
    assert (s.variant, s.d16, s.classes) == (oracle.VARIANT_STREAM, 2, oracle.CLASS_CMP | oracle.CLASS_MB)
    assert oracle.profile_select(f, b, w, p_stream=2.69).d16 == 0          # below (1 - tol) P_MB
    assert oracle.profile_select({**f, "n_deltas": 257}, b, w, p_stream=3.5).d16 == 0   # not codable
    assert oracle.profile_select({**f, "nnz_max": 20}, b, w, p_stream=3.5).d16 == 0     # irregular rows
    assert oracle.profile_select(f, b, w, p_stream=3.5, classes=oracle.CLASS_CMP).d16 == 0  # forced classes


def test_tune_profile_search_picks_the_widest_margin():
    """tools/tune_profile.search on synthetic records: a stencil-like matrix
    (IMB ratio 1.5: IMB would pick a 2x slower plan) and an R-MAT-like one
    (ratio 6: IMB gains 4x) leave T_IMB optimal in [1.5, 6); the chosen point
    sits at the geometric middle of that gap (widest log-margin), and T_ML /
    tol, which no record's decision depends on, keep the paper's values."""
    import sys
    root = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
    sys.path.insert(0, os.path.join(root, "tools"))
    import tune_profile as T

    def rec(name, ratio_imb, gains):
        b = dict(p_csr=1.0, p_mb=5.0, p_ml=0.97, p_imb=ratio_imb, p_cmp=1.3, p_peak=8.0)
        us, poc = {}, {}
        for c in range(16):
            key = f"plan{c & T.IMB}"
            poc[str(c)] = key
            us[key] = 100.0 / gains.get(c & T.IMB, 1.0)
        return dict(name=name, us=us, plan_of_classes=poc), b
    r1, b1 = rec("stencil", 1.5, {0: 1.0, T.IMB: 0.5})
    r2, b2 = rec("rmat", 6.0, {0: 1.0, T.IMB: 4.0})
    res, chosen = T.search([r1, r2], [b1, b2])
    lo, hi = res["optimal_region_bbox"]["t_imb"]
    assert 1.5 <= lo <= 1.51 and 5.98 <= hi < 6.0
    assert abs(chosen[0] - 3.0) <= 0.02            # sqrt(1.5 * 6) = 3: equal log-margins
    assert (chosen[1], chosen[2]) == (T.PAPER[1], T.PAPER[2])
    assert T.score([r1, r2], [b1, b2], chosen)[1] > T.score([r1, r2], [b1, b2], T.PAPER)[1]


# ---- row-pattern codes (reading 31) ------------------------------
def _pat_stencil_closed_form(n, pts):
    """Patterns of a pts-point stencil on n^3 (n >= 3) from the grid geometry:
    one per boundary class (low / interior / high in each dimension), offsets
    dz n^2 + dy n + dx over the neighbours that exist, ascending."""
    out = {}
    for cz in (0, 1, 2):
        for cy in (0, 1, 2):
            for cx in (0, 1, 2):
                def rng(c):
                    return [d for d in (-1, 0, 1) if not (c == 0 and d == -1) and not (c == 2 and d == 1)]
                if pts == 27:
                    o = [dz * n * n + dy * n + dx for dz in rng(cz) for dy in rng(cy) for dx in rng(cx)]
                else:
                    o = [0] + [dz * n * n for dz in rng(cz) if dz] + [dy * n for dy in rng(cy) if dy] + \
                        [dx for dx in rng(cx) if dx]
                out[(cz, cy, cx)] = sorted(o)
    return out


@pytest.mark.parametrize("n", [3, 4, 7, 12])
@pytest.mark.parametrize("pts", [7, 27])
def test_pat_stencil_closed_form(n, pts):
    m = sg.stencil(n, pts)
    ids, lens, ofs = oracle.pat_encode(m.rowptr, m.colind)
    want = _pat_stencil_closed_form(n, pts)
    assert len(lens) == 27  # one pattern per boundary class
    starts = np.concatenate([[0], np.cumsum(lens)])
    got = {tuple(ofs[starts[p]:starts[p + 1]].tolist()) for p in range(len(lens))}
    assert got == {tuple(v) for v in want.values()}
    # every row carries the pattern of its class
    i = np.arange(m.n)
    cls = lambda c: np.where(c == 0, 0, np.where(c == n - 1, 2, 1))  # noqa: E731
    for r in np.random.default_rng(n).integers(0, m.n, 200):
        key = (int(cls(i[r] // (n * n))), int(cls((i[r] // n) % n)), int(cls(i[r] % n)))
        p = ids[r]
        assert ofs[starts[p]:starts[p + 1]].tolist() == want[key]
    assert int(lens.sum()) == (343 if pts == 27 else 135)  # (2+3+2)^3; 8*4 + 12*5 + 6*6 + 7
    assert np.array_equal(oracle.pat_decode(ids, lens, ofs), m.colind)


def test_pat_hand_example_and_limits():
    # rows: [0, 1], [1, 2], [0]: offsets (0, 1), (0, 1), (-2) -> ids 0, 0, 1
    ids, lens, ofs = oracle.pat_encode(rp_of([2, 2, 1]), np.array([0, 1, 1, 2, 0], np.int32))
    assert ids.tolist() == [0, 0, 1] and lens.tolist() == [2, 1] and ofs.tolist() == [0, 1, -2]
    # empty rows are the length-0 pattern; ids by first occurrence
    ids, lens, ofs = oracle.pat_encode(rp_of([0, 1, 0, 1]), np.array([3, 0], np.int32))
    assert ids.tolist() == [0, 1, 0, 2] and lens.tolist() == [0, 1, 1] and ofs.tolist() == [2, -3]
    # 256 patterns codable, 257 not: row i -> column 0 (offset -i)
    for k, ok in ((256, True), (257, False)):
        enc = oracle.pat_encode(np.arange(k + 1), np.zeros(k, np.int32))
        assert (enc is not None) == ok
        if ok:
            assert enc[0].tolist() == list(range(k)) and enc[2].tolist() == [-i for i in range(k)]
    # offsets limit (total over the patterns) and the 255 row-length limit
    rp, ci = rp_of([3, 3]), np.array([0, 1, 2, 0, 2, 3], np.int32)  # offsets (0,1,2), (-1,1,2): 6
    assert oracle.pat_encode(rp, ci, maxofs=6) is not None and oracle.pat_encode(rp, ci, maxofs=5) is None
    for L_, ok in ((255, True), (256, False)):
        assert (oracle.pat_encode(rp_of([L_]), np.arange(L_, dtype=np.int32)) is not None) == ok


@pytest.mark.parametrize("seed", range(4))
def test_pat_first_occurrence_vs_dict(seed):
    # banded rows from a few templates: ids equal a dict-based re-derivation
    # (first occurrence of each (length, offsets) tuple), round trip exact
    g = np.random.default_rng(seed)
    n = 2000
    tmpl = [np.array(sorted(set(g.integers(-40, 40, g.integers(1, 12)).tolist()))) for _ in range(9)]
    rows = [tmpl[t] for t in g.integers(0, 9, n)]
    rows = [r[(r + i >= 0) & (r + i < n)] + i for i, r in enumerate(rows)]
    rp = rp_of([len(r) for r in rows])
    ci = np.concatenate(rows).astype(np.int32)
    ids, lens, ofs = oracle.pat_encode(rp, ci)
    seen, want = {}, []
    for i, r in enumerate(rows):
        want.append(seen.setdefault(tuple((r - i).tolist()), len(seen)))
    assert ids.tolist() == want and len(lens) == len(seen)
    assert np.array_equal(oracle.pat_decode(ids, lens, ofs), ci)
