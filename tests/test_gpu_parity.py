"""GPU parity: the CUDA path (through the C ABI) against the oracle.

Bar (BJ.north_star): |y_gpu[i] - y_ref[i]| <= 1e-12 * sum_j |a_ij x_j| for
every row; bit-exact for integer work (plan structures, D16 round trip,
features, validation codes) and for dyadic inputs where every summation
order is exact.
"""
import os

import numpy as np
import pytest

import oracle
import synthgen as sg

pytestmark = pytest.mark.gpu

torch = pytest.importorskip("torch")
spmv = pytest.importorskip("paper_1711_05487_b200")

TOL = 1e-12


def assert_bound(y, m, rows=None, tol=TOL):
    if rows is None:
        yr = oracle.spmv(m.rowptr, m.colind, m.vals, m.x)
        s = oracle.absrow(m.rowptr, m.colind, m.vals, m.x)
        yy = y
    else:
        yr = oracle.spmv_rows(m.rowptr, m.colind, m.vals, m.x, rows)
        s = oracle.absrow(m.rowptr, m.colind, m.vals, m.x, rows)
        yy = y[rows]
    err = np.abs(yy - yr)
    bad = np.nonzero(err > tol * s)[0]
    assert bad.size == 0, f"{bad.size} rows over the bound, first {bad[:5]}, err {err[bad[:5]]}, s {s[bad[:5]]}"
    # empty rows must be exactly zero (bound RHS is 0)
    return err


def m_maxlen(m):
    return int(np.diff(m.rowptr.astype(np.int64)).max(initial=0))


VARIANTS = [("vector", 1), ("vector", 2), ("vector", 8), ("vector", 32), ("stream", 1), ("stream", 4),
            ("stream", 8), ("stream", 32), ("stream_seg", 1), ("stream_nnz_tiles", 1), ("merge", 0), ("split", 4),
    ("split_seg", 32), ("split_chunks", 16), ("split_tiled", 8), ("split_tma", 8), ("split_bins", 8), ("nnzsplit", 0),
    ("nnzsplit_hot", 0), ("nnzsplit_nohot", 0)]
ALL = ("vector", "stream", "merge", "split", "nnzsplit")

SUITE = sg.small_suite(seed=21)


def variant_kw(variant):
    """test variant name -> (force_variant, extra options)"""
    if variant == "stream_seg":
        return "stream", {"seg": 1}
    if variant == "stream_d16":
        return "stream", {"d16": 1}
    if variant == "split_seg":
        return "split", {"seg": 1, "split_bins": 0}
    if variant == "split_bins":
        return "split", {"split_bins": 0}
    if variant == "nnzsplit_hot":
        return "nnzsplit", {"hot_x": 64}
    if variant == "nnzsplit_nohot":
        return "nnzsplit", {"hot_x": 0}
    if variant == "split_chunks":
        return "split", {"long_mode": 1}
    if variant == "split_tiled":
        return "split", {"long_mode": 2}
    if variant == "split_tma":
        return "split", {"long_mode": 3}
    if variant == "stream_nnz_tiles":
        return "stream", {"no_aligned": 1}
    return variant, {}


@pytest.mark.parametrize("variant,vs", VARIANTS)
@pytest.mark.parametrize("name,m", SUITE, ids=[n for n, _ in SUITE])
def test_small_suite_all_variants(name, m, variant, vs):
    fv, extra = variant_kw(variant)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, force_variant=fv, force_vs=vs, l_split=64,
                  tile_nnz=512, **extra)
    y = p.execute(m.x)
    assert_bound(y, m)
    assert p.info()["variant"] == fv


LONG_TMA_CASES = [  # (n, k per short row, long rows, nonzeros per long row, l_split)
    (5001, 6, 300, 1500, 64),     # 300 long rows: > 32 rows per warp at rg = 1, so rg > 1; odd n: odd last x block
    (20000, 15, 10, 4500, 64),    # C4 small
    (3000, 4, 3, 2990, 64),       # nearly dense long rows
    (70001, 3, 5, 60000, 4096),   # long segments: several chunks per (row, x block)
    (9000, 5, 40, 300, 64),       # sparse long rows: many empty (row, x block) segments
]


@pytest.mark.parametrize("case", LONG_TMA_CASES)
@pytest.mark.parametrize("dyadic", [False, True])
def test_split_long_tma(case, dyadic):
    """long_mode 3: TMA-staged column-tiled long rows on the side stream
    (long_tma.cu) next to the nnz_split bin; every row within the per-row
    bound, dyadic inputs bit-equal to the oracle, and x at an address that is
    not 16-B aligned takes the register-staged kernel."""
    import torch
    n, k, nl, kl, ls = case
    mode = sg.MODE_DYADIC if dyadic else sg.MODE_U11
    m = sg.randrows(n, k, diag=False, long_rows=sg.pick_rows(n, nl, 77 + n), k_long=kl, col_seed=5 + n,
                    val_mode=mode, val_seed=6, x_seed=7, x_mode=mode)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=n, force_variant="split", long_mode=3, l_split=ls)
    info = p.info()
    assert info["variant"] == "split" and info["long_mode"] == 3 and info["long_rg"] >= 1
    assert -(-nl // (info["long_rg"] * 8)) <= 32  # rows of a warp inside an item fit the lanes
    y = p.execute(m.x)
    if dyadic:
        assert np.array_equal(y, oracle.spmv(m.rowptr, m.colind, m.vals, m.x))
    else:
        assert_bound(y, m)
    xb = torch.zeros(n + 1, dtype=torch.float64, device="cuda")
    xb[1:] = torch.from_numpy(m.x)
    yd = torch.empty(n, dtype=torch.float64, device="cuda")
    for _ in range(2):
        p.execute(xb[1:], yd)  # 8-B offset: the fallback kernel (its own summation order)
        if dyadic:
            assert np.array_equal(yd.cpu().numpy(), y)
        else:
            assert_bound(yd.cpu().numpy(), m)
    xa = torch.from_numpy(m.x).cuda()
    for _ in range(3):  # back-to-back launches on the plan's streams
        p.execute(xa, yd)
    assert np.array_equal(yd.cpu().numpy(), y)


@pytest.mark.parametrize("tile", [128, 384, 1024])
@pytest.mark.parametrize("name,m", SUITE, ids=[n for n, _ in SUITE])
def test_seg_mode_tiles(name, m, tile):
    for fv in ("stream", "split"):
        p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, force_variant=fv, seg=1, tile_nnz=tile,
                      l_split=256, split_bins=0)
        assert p.info()["sel"]["seg"] == 1
        assert_bound(p.execute(m.x), m)


@pytest.mark.parametrize("variant,vs", VARIANTS + [("stream_d16", 8)])
@pytest.mark.parametrize("name,m", sg.small_suite(seed=4, val_mode=sg.MODE_DYADIC, x_mode=sg.MODE_DYADIC),
                         ids=[n for n, _ in SUITE])
def test_dyadic_bit_exact(name, m, variant, vs):
    kw = dict(force_vs=vs, l_split=64, tile_nnz=512)
    variant, extra = variant_kw(variant)
    kw.update(extra)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, force_variant=variant, **kw)
    y = p.execute(m.x)
    assert np.array_equal(y, oracle.spmv(m.rowptr, m.colind, m.vals, m.x))


@pytest.mark.parametrize("tile", [512, 1024, 4096])
@pytest.mark.parametrize("vs", [1, 4])
@pytest.mark.parametrize("name,m", SUITE, ids=[n for n, _ in SUITE])
def test_stream_d16_and_structures(name, m, tile, vs):
    w, mg, dcol, head, esc = oracle.d16_encode_esc(m.rowptr, m.colind)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, force_variant="stream", d16=1, tile_nnz=tile,
                  force_vs=vs)
    info = p.info()
    stride = info["tile_stride"]  # tile_nnz, or tile_nnz - longest row for row-aligned tiles
    assert stride == (tile - m_maxlen(m) if info["tiles_row_aligned"] else tile)
    assert np.array_equal(p.export("tile_rows"), oracle.tile_rows(m.rowptr, stride))
    if w == 0:
        assert info["sel"]["d16"] == 0
    else:
        assert info["sel"]["d16"] == 1 and info["d16_width"] == (8 if mg <= 255 else 16)
        assert info["d16_n_esc"] == esc.size
        if m.nnz:
            assert np.array_equal(p.export("dcol"), dcol)
            assert np.array_equal(p.export("head"), head)
            assert np.array_equal(p.export("anchor"), oracle.tile_anchor(m.colind, stride))
            assert np.array_equal(p.export("decoded"), m.colind)  # round trip
    assert_bound(p.execute(m.x), m)


@pytest.mark.parametrize("name,m", SUITE, ids=[n for n, _ in SUITE])
def test_plan_structures_bit_exact(name, m):
    pm = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, force_variant="merge")
    si, sj = oracle.merge_splits(m.rowptr, 2048)
    assert np.array_equal(pm.export("merge_rows"), si) and np.array_equal(pm.export("merge_nnz"), sj)
    for L, C in ((64, 256), (4096, 8192), (0, 256)):
        ps = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, force_variant="split", l_split=L,
                       long_chunk=C)
        crow, cb, ce = oracle.long_chunks(m.rowptr, L if L else 4096, C)
        assert np.array_equal(ps.export("chunk_row"), crow)
        assert np.array_equal(ps.export("chunk_begin"), cb)
        assert np.array_equal(ps.export("chunk_end"), ce)
        assert_bound(ps.execute(m.x), m)
    # nnz_split structures (reading 19)
    pz = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, force_variant="nnzsplit")
    rowmap, rpc = oracle.nonempty_rows(m.rowptr)
    assert np.array_equal(pz.export("nz_rowmap"), rowmap)
    assert np.array_equal(pz.export("nz_rpc"), rpc)
    assert np.array_equal(pz.export("nz_tile_q"), oracle.nz_tiles(rpc) if m.nnz else np.array([0]))
    assert pz.info()["n_nz_rows"] == rowmap.size - 1
    ph = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, force_variant="nnzsplit", hot_x=100)
    hot, cov = oracle.hot_columns(m.colind, m.x.size, 100)
    assert np.array_equal(ph.export("nz_hot_cols"), hot) and ph.info()["n_hot"] == hot.size
    if m.nnz:
        assert abs(ph.info()["hot_cover"] - cov / m.nnz) < 1e-15
    assert_bound(ph.execute(m.x), m)
    # features: exact integers, identical doubles (same formula, IEEE sqrt)
    f = oracle.features(m.rowptr, m.colind, n_cols=m.x.size)
    g = pm.info()["feat"]
    for k, v in f.items():
        assert g[k] == v, k


@pytest.mark.parametrize("rp,ci,n,nnz", [
    ([1, 1, 2], [0, 1], 2, 2),
    ([0, 1, 3], [0, 1], 2, 2),
    ([0, 2, 1, 2], [0, 1], 3, 2),
    ([0, 1, 2], [0, 2], 2, 2),
    ([0, 1, 2], [-1, 0], 2, 2),
    ([0, 2, 4], [0, 1, 1, 1], 2, 4),
    ([0, 2, 4], [1, 0, 0, 1], 2, 4),
    ([0, 3, 6], [0, 1, 1, 0, 5, 1], 2, 6),
])
def test_validation_matches_oracle(rp, ci, n, nnz):
    code, where = oracle.validate(n, nnz, np.array(rp), np.array(ci, np.int32))
    assert code != 0
    rp64 = np.array(rp, np.int64)
    with pytest.raises(spmv.SpmvError) as e:
        spmv.Plan(rp64[: n + 1] if rp64.size > n + 1 else rp64, np.array(ci[:max(nnz, 0)], np.int32),
                  np.ones(len(ci)), n_cols=n)
    assert e.value.status == -2
    assert f"code {code} " in e.value.msg and e.value.msg.endswith(f" {where}"), e.value.msg


def test_valid_edge_cases():
    # all-empty matrix, single row, zero rows
    for rp, ci, n in (([0, 0, 0, 0], [], 3), ([0, 1], [0], 1), ([0], [], 0)):
        for v in ALL:
            p = spmv.Plan(np.array(rp, np.int64), np.array(ci, np.int32), np.ones(len(ci)), n_cols=max(n, 1),
                          force_variant=v)
            y = p.execute(np.full(max(n, 1), 3.0), np.full(n, 7.0) if n else np.zeros(0))
            assert np.array_equal(y, oracle.spmv(np.array(rp), np.array(ci, np.int32), np.ones(len(ci)),
                                                 np.full(max(n, 1), 3.0)))


@pytest.mark.parametrize("c", [1, 2, 3, 4])
def test_configs_full_auto_selection(c):
    m = sg.config(c)
    p = spmv.Plan(m.rowptr, m.colind, m.vals)
    y = p.execute(m.x)
    assert_bound(y, m)
    info = p.info()
    f = oracle.features(m.rowptr, m.colind)
    props = spmv.device_query(0)
    o = oracle.select(f, props["l2_bytes"], props["access_window_max"], m.rowptr.dtype.itemsize)
    assert (info["sel"]["variant"], info["sel"]["vs"], info["sel"]["d16"], bool(info["sel"]["xwin"])) == \
        (o.variant, o.vs, o.d16, o.xwin)


@pytest.mark.parametrize("c", [2, 3, 4])
@pytest.mark.parametrize("variant", list(ALL) + ["split_bins"])
def test_configs_full_forced_variants(c, variant):
    variant, extra = variant_kw(variant)
    m = sg.config(c)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, force_variant=variant, **extra)
    assert_bound(p.execute(m.x), m)


def test_split_long_rows_16bit_columns(monkeypatch):
    """SPLIT's column-tiled long rows read 16-bit in-block columns (colind mod
    the 2048-column x block) on full C4: the plan reports it, its compulsory
    bytes drop by 2 B per long-row nonzero, and y is bit-identical to the
    int32-colind long rows (same arithmetic, same order) and within the bound."""
    m = sg.config(4)
    p = spmv.Plan(m.rowptr, m.colind, m.vals)
    info = p.info()
    assert info["variant"] == "split" and info["long_c16"] == 1
    monkeypatch.setenv("SPMV_LONG_C16", "0")
    q = spmv.Plan(m.rowptr, m.colind, m.vals)
    monkeypatch.delenv("SPMV_LONG_C16")
    iq = q.info()
    assert iq["long_c16"] == 0
    assert iq["kernel_bytes"] - info["kernel_bytes"] == 2 * info["feat"]["nnz_long"]
    y = p.execute(m.x)
    assert np.array_equal(y, q.execute(m.x))
    assert_bound(y, m)
    p.destroy()
    q.destroy()


def test_stencil_ones_bit_exact():
    # 7-pt A*1 counts missing neighbours exactly -> bit-equal
    m = sg.config(2)
    ones = np.ones(m.n)
    ref = oracle.spmv(m.rowptr, m.colind, m.vals, ones)
    for v in ALL:
        for d16 in (0, 1):
            p = spmv.Plan(m.rowptr, m.colind, m.vals, force_variant=v, d16=d16)
            assert np.array_equal(p.execute(ones), ref)


def test_device_and_host_buffers_agree():
    m = sg.config(2)
    p = spmv.Plan(m.rowptr, m.colind, m.vals)
    y_host = p.execute(m.x)
    xd = torch.from_numpy(m.x).cuda()
    yd = torch.empty(m.n, dtype=torch.float64, device="cuda")
    p.execute(xd, yd)
    assert np.array_equal(yd.cpu().numpy(), y_host)
    # plan-resident buffers (the timed path)
    p2 = spmv.Plan(torch.from_numpy(m.rowptr).cuda(), torch.from_numpy(m.colind).cuda(),
                   torch.from_numpy(m.vals).cuda())
    assert p2.info()["variant"] == p.info()["variant"]
    p2.execute(xd, yd)
    torch.cuda.synchronize()
    assert np.array_equal(yd.cpu().numpy(), y_host)


@pytest.mark.parametrize("lens,vs", [([7] * 5000 + [6, 5] * 700 + [7] * 3, 1), ([3, 4] * 3000 + [5], 1),
                                     ([30, 31, 29] * 900, 4), ([7] * 95 + [6], 1)])
def test_row_count_tiles(lens, vs):
    # regular short rows: tile k = rows [k*Rt, (k+1)*Rt) (Rt = whole warp
    # passes), ragged last tile; structure exported and checked exactly
    g = np.random.default_rng(5)
    lens = np.asarray(lens, np.int64)
    m = sg.from_lengths(lens, lens.size, g, sg.MODE_U11, sg.MODE_U11)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, force_variant="stream", force_vs=vs, seg=0)
    info = p.info()
    Rt = info["rows_per_tile"]
    assert Rt > 0 and Rt % (32 // vs) == 0 and info["tiles_row_aligned"] == 1
    T = -(-m.n // Rt)
    assert np.array_equal(p.export("tile_rows"), np.minimum(np.arange(T + 1) * Rt, m.n))
    assert Rt * int(lens.max()) <= info["tile_nnz"]
    assert_bound(p.execute(m.x, np.full(m.n, np.nan)), m)
    p.destroy()


@pytest.mark.parametrize("extra", [{}, {"no_aligned": 1}, {"d16": 1}, {"force_vs": 4}, {"tile_nnz": 0}])
@pytest.mark.parametrize("name,lens", [("uniform", [7] * 40000), ("mixed", ([3, 0, 9, 27, 1, 64] * 8000)),
                                       ("long_rows", [5] * 20000 + [9000] * 3 + [5] * 20000),
                                       # a row cut into > 2048 tiles: the range fix-ups
                                       ("huge_row", [5] * 20000 + [1_100_000] + [5] * 20000)])
def test_pipelined_host_execute(monkeypatch, name, lens, extra):
    # host x / host y through a STREAM plan: tile blocks overlapped with the
    # x upload and the y download (api.cu host_pipe_*); rows cut at block
    # edges are completed by the next block's fix-up
    monkeypatch.setenv("SPMV_HOST_PIPE_MIN_BYTES", "1")
    monkeypatch.setenv("SPMV_HOST_PIPE_BLOCKS", "7")
    g = np.random.default_rng(11)
    lens = np.asarray(lens, np.int64)
    m = sg.from_lengths(lens, max(lens.size, int(lens.max())), g, sg.MODE_U11, sg.MODE_U11)
    kw = {"tile_nnz": 512, "seg": 0}
    kw.update(extra)  # tile_nnz 0: the plan's own tile rule (row-count tiles on regular rows)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, force_variant="stream", **kw)
    yh = p.execute(m.x, np.full(m.n, np.nan))  # host buffers: pipelined
    assert_bound(yh, m)
    assert np.all(yh[lens == 0] == 0.0)
    xd = torch.from_numpy(m.x).cuda()
    yd = torch.full((m.n,), float("nan"), dtype=torch.float64, device="cuda")
    p.execute(xd, yd)  # device buffers: one launch over all tiles
    yd = yd.cpu().numpy()
    if p.info()["tiles_row_aligned"]:
        assert np.array_equal(yh, yd)  # no carries: identical arithmetic
    else:
        assert_bound(yd, m)
    p.destroy()


@pytest.mark.parametrize("hot", [0, 256])
@pytest.mark.parametrize("name,lens", [("powerlaw", None), ("empty_runs", ([0] * 300 + [700, 3, 0, 5]) * 60),
                                       ("long_rows", [5] * 20000 + [9000] * 3 + [0] * 500 + [5] * 20000),
                                       # rows cut into > 2048 warp tiles, one crossing several pipeline ranges:
                                       # the range fix-ups must not use the plan-wide hierarchical scratch
                                       ("huge_rows", [5] * 20000 + [700_000] + [3] * 3000 + [650_000] + [5] * 20000)])
def test_pipelined_host_execute_nnzsplit(monkeypatch, name, lens, hot):
    # nnz_split ranges with the y download overlapped: range b's carries are
    # added after range b+1 (rows are assigned where they end); every row,
    # empty ones included, must come back complete
    monkeypatch.setenv("SPMV_HOST_PIPE_MIN_BYTES", "1")
    monkeypatch.setenv("SPMV_HOST_PIPE_BLOCKS", "5")
    g = np.random.default_rng(13)
    if lens is None:
        lens = np.minimum((g.pareto(1.2, size=60000) * 3).astype(np.int64), 20000)
    lens = np.asarray(lens, np.int64)
    m = sg.from_lengths(lens, max(lens.size, int(lens.max())), g, sg.MODE_U11, sg.MODE_U11)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, force_variant="nnzsplit", hot_x=hot)
    yh = p.execute(m.x, np.full(m.n, np.nan))
    assert_bound(yh, m)
    assert np.all(yh[lens == 0] == 0.0)
    p.destroy()


def test_deterministic_repeat():
    m = sg.config(3, small=True)
    for v in ALL:
        p = spmv.Plan(m.rowptr, m.colind, m.vals, force_variant=v)
        y0 = p.execute(m.x)
        for _ in range(3):
            assert np.array_equal(p.execute(m.x), y0)


@pytest.mark.parametrize("G", [2, 3, 8])
@pytest.mark.parametrize("variant", ALL)
def test_emulated_shards(G, variant):
    m = sg.config(4, small=True)
    p1 = spmv.Plan(m.rowptr, m.colind, m.vals, force_variant=variant, force_vs=8)
    pg = spmv.Plan(m.rowptr, m.colind, m.vals, ngpus=G, emulate_devices=1, force_variant=variant, force_vs=8)
    assert pg.info()["shard_bounds"] == oracle.shard_bounds(m.rowptr, G).tolist()
    yg = pg.execute(m.x)
    assert_bound(yg, m)
    if variant == "vector":  # fixed per-row order: bit-equal across shard counts
        assert np.array_equal(yg, p1.execute(m.x))


def test_iterated_mode_vs_oracle():
    m = sg.config(5, small=True)
    K = 100
    rc, xr, nur = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, K)
    assert rc == 0
    for G in (1, 3):
        p = spmv.Plan(m.rowptr, m.colind, m.vals, ngpus=G, emulate_devices=1)
        xg, nug = p.iterate(m.x, K)
        # SURVEY 8(c3) #21 end-to-end tolerances
        assert np.max(np.abs(xg - xr)) <= 1e-10 * np.max(np.abs(xr))
        assert abs(nug[-1] - nur[-1]) <= 1e-12 * nur[-1]
        assert np.all(np.abs(nug - nur) <= 1e-12 * nur)
        # stepwise: y_k from the GPU's own x_k obeys the per-row bound
        for k in (1, 49):
            xk, _ = p.iterate(m.x, k)
            yk = p.execute(xk)
            mk = sg.CSR(m.n, m.rowptr, m.colind, m.vals, xk)
            assert_bound(yk, mk)
        assert np.all(np.diff(nug[1:]) >= -1e-13 * nug[1:-1])  # monotone for symmetric A


@pytest.mark.parametrize("scale", [1e40, 1e-40])
def test_iterated_mode_rescale(scale):
    # deferred normalisation (reading 25): the unnormalised iterate
    # grows (or shrinks) by ~1e40 per step, so the exact power-of-two rescale
    # must fire every few iterations; results match the per-step oracle
    m = sg.config(5, small=True)
    vals = m.vals * scale
    K = 40
    rc, xr, nur = oracle.power_iter(m.rowptr, m.colind, vals, m.x, K)
    assert rc == 0
    for G in (1, 2):
        p = spmv.Plan(m.rowptr, m.colind, vals, ngpus=G, emulate_devices=1)
        xg, nug = p.iterate(m.x, K)
        assert np.all(np.isfinite(xg)) and np.all(np.isfinite(nug))
        assert np.max(np.abs(xg - xr)) <= 1e-10 * np.max(np.abs(xr))
        assert np.all(np.abs(nug - nur) <= 1e-12 * nur)


@pytest.mark.parametrize("c,variant", [(2, "stream"), (5, "stream"), (3, "nnzsplit"), (2, "merge")])
def test_execute_norm_fused_partials(c, variant):
    # spmv_execute_norm: y bit-equal to the plain SpMV; the partials (fused
    # per-tile squares for row-aligned STREAM plans, else the separate pass)
    # sum to ||y||^2 up to rounding
    m = sg.config(c, small=True)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, force_variant=variant)
    P = spmv.norm_partial_count()
    xd = torch.from_numpy(m.x).cuda()
    y1 = torch.empty(m.n, dtype=torch.float64, device="cuda")
    y2 = torch.empty(m.n, dtype=torch.float64, device="cuda")
    pa = torch.empty(P, dtype=torch.float64, device="cuda")
    p.execute(xd, y1)
    p.execute_norm(xd, y2, pa)
    torch.cuda.synchronize()
    assert torch.equal(y1, y2)
    ref = float(np.sum(y1.cpu().numpy() ** 2))
    assert abs(float(pa.sum()) - ref) <= 1e-13 * ref
    p.destroy()


def test_iterated_zero_norm():
    rp = np.zeros(11, np.int64)
    p = spmv.Plan(rp, np.zeros(0, np.int32), np.zeros(0))
    with pytest.raises(spmv.SpmvError) as e:
        p.iterate(np.ones(10), 3)
    assert e.value.status == -7


@pytest.mark.slow
def test_c5_full_sampled_rows_and_properties():
    m = sg.config(5)
    p = spmv.Plan(m.rowptr, m.colind, m.vals)
    info = p.info()
    assert info["feat"]["nnz"] == 1520875000 and info["feat"]["maxgap"] == 384 * 384 - 384 - 1
    y = p.execute(m.x)
    g = np.random.default_rng(0)
    rows = np.unique(np.concatenate([g.integers(0, m.n, 200000), np.arange(5000), m.n - 1 - np.arange(5000),
                                     np.arange(0, m.n, 147457)]))
    assert_bound(y, m, rows)
    # A*1 closed form on every row (exact in any order)
    y1 = p.execute(np.ones(m.n))
    assert set(np.unique(y1).tolist()) == {0.0, 9.0, 15.0, 19.0}
    n = 384
    i = np.arange(m.n, dtype=np.int64)
    prod = np.ones(m.n)
    for c in (i % n, (i // n) % n, i // (n * n)):
        prod *= 3 - (c == 0).astype(float) - (c == n - 1)
    assert np.array_equal(y1, 27.0 - prod)


# nnz_split edge cases: rows ending exactly at warp-tile edges, a row spanning
# many tiles, leading / trailing / interleaved empty rows, nnz < one tile,
# nnz an exact multiple of the tile, int64 rowptr
NZ_EDGE = [
    ("tile_aligned_rows", [256] * 8),
    ("row_ends_at_edge", [255, 1, 256, 0, 0, 512]),
    ("one_row_many_tiles", [0, 0, 5000, 0]),
    ("lead_trail_empty", [0] * 7 + [3, 0, 0, 300, 1] + [0] * 9),
    ("tiny", [1, 0, 2]),
    ("len1_mult", [1] * 512),
    ("alternating", [0, 1] * 700 + [0, 257] * 3),
    # runs of > 1024 carries: the hierarchical fix-up (two and three levels)
    ("huge_rows", [3, 600000, 2, 0, 300000, 1]),
    ("huge_adjacent", [270000, 270000, 1, 270000]),
    # long empty runs between sparse non-empty rows: the warp-cooperative gap
    # zeroing (gaps > 8 rows), gaps straddling 32-gap chunks, mixed with short gaps
    ("empty_runs", ([0] * 2300 + [700]) * 40 + [0] * 5000),
    ("empty_runs_mixed", ([0] * 9 + [1] + [0] * 3 + [2] + [0] * 40 + [1]) * 300 + [0] * 77),
    ("empty_runs_dense_ends", ([1] * 40 + [0] * 500) * 20),
]


@pytest.mark.parametrize("rp_dtype", [np.int32, np.int64])
@pytest.mark.parametrize("name,lens", NZ_EDGE, ids=[n for n, _ in NZ_EDGE])
def test_nzsplit_edges(name, lens, rp_dtype):
    g = np.random.default_rng(7)
    lens = np.asarray(lens, np.int64)
    m = sg.from_lengths(lens, max(int(lens.max()), lens.size), g, sg.MODE_U11, sg.MODE_U11)
    rp = m.rowptr.astype(rp_dtype)
    for fv, extra in (("nnzsplit", {}), ("split", {"l_split": 64})):
        p = spmv.Plan(rp, m.colind, m.vals, n_cols=m.x.size, force_variant=fv, **extra)
        y = p.execute(m.x, np.full(m.n, np.nan))
        assert_bound(y, m)
        assert np.all(y[lens == 0] == 0.0)


@pytest.mark.parametrize("K", [2, 1000, 16384])
def test_nzsplit_hot_sizes(K):
    m = sg.config(3, small=True)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, force_variant="nnzsplit", hot_x=K)
    hot, _ = oracle.hot_columns(m.colind, m.n, min(K, 16384))
    assert p.info()["n_hot"] == hot.size
    y = p.execute(m.x)
    assert_bound(y, m)
    for _ in range(2):  # x changes between calls: the hot table is refreshed per SpMV
        x2 = m.x[::-1].copy()
        assert_bound(p.execute(x2), sg.CSR(m.n, m.rowptr, m.colind, m.vals, x2))


# escape-coded D16 (reading 21): large in-row gaps (a 27-point
# stencil with n^2 > 65535, rows of a random matrix with a few big jumps)
@pytest.mark.parametrize("vs", [1, 4])
def test_d16_escapes_parity(vs):
    cases = [sg.stencil(260, 27, rp64=True, x_seed=3, rows=(0, 150000))]
    g = np.random.default_rng(9)
    n = 3000
    lens = g.integers(1, 40, n)
    rp = np.concatenate([[0], np.cumsum(lens)])
    ci = np.empty(rp[-1], np.int32)
    for i in range(n):  # columns spaced by small gaps or one of 5 large jumps
        steps = np.where(g.random(lens[i]) < 0.2, g.choice([70000, 80000, 90001, 123456, 65472], lens[i]),
                         g.integers(1, 50, lens[i]))
        steps[0] = g.integers(0, 100)
        ci[rp[i]:rp[i + 1]] = np.cumsum(steps)
    cases.append(sg.CSR(n, rp, ci, g.uniform(-1, 1, ci.size), g.uniform(-1, 1, int(ci.max()) + 1)))
    for m in cases:
        ncols = m.x.size
        w, mg, dcol, head, esc = oracle.d16_encode_esc(m.rowptr, m.colind)
        assert w == 16 and mg > 65535 and esc.size > 0
        for tile in (512, 1024):
            p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=ncols, force_variant="stream", d16=1, force_vs=vs,
                          tile_nnz=tile)
            info = p.info()
            assert info["sel"]["d16"] == 1 and info["d16_n_esc"] == esc.size
            assert info["feat"]["n_big_gaps"] == esc.size
            assert np.array_equal(p.export("dcol"), dcol)
            assert np.array_equal(p.export("decoded"), m.colind)
            assert_bound(p.execute(m.x), m)



# profile-guided mode: the plan's Fig. 4 classes and Table II
# choice equal the oracle's pure functions of the bounds the plan measured
PROFILE_KEYS = ("p_csr", "p_mb", "p_ml", "p_imb", "p_cmp", "p_peak")


@pytest.mark.parametrize("c,small", [(1, False), (2, True), (3, True), (4, True), (5, True), (2, False), (3, False),
                                     (4, False)])
def test_profile_mode_selection(c, small):
    m = sg.config(c, small=small)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, select_mode=1)
    info = p.info()
    b = {k: info[k] for k in PROFILE_KEYS}
    assert all(v > 0 for v in b.values()) and info["bmax"] > 0
    assert b["p_peak"] > b["p_mb"]                      # S:303-306 invariant
    assert b["p_imb"] >= 0.95 * b["p_csr"]              # median <= max busy time (+ noise)
    assert 0 < info["profile_ms"] <= info["select_ms"]
    f = oracle.features(m.rowptr, m.colind)
    o = oracle.profile_select(f, b, spmv.device_query(0)["access_window_max"], p_stream=info["p_stream"] or None)
    s = info["sel"]
    assert (s["variant"], s["vs"], s["d16"], bool(s["xwin"]), s["classes"]) == \
        (o.variant, o.vs, o.d16, o.xwin, o.classes), (b, info["p_stream"], s)
    assert_bound(p.execute(m.x), m)



@pytest.mark.parametrize("c", [2, 4])
def test_profile_forced_classes_follow_table2(c):
    """force_classes = set: no probes, Table II's mapping of the set (the grid
    search's hook, tools/tune_profile.py) equals the oracle's."""
    m = sg.config(c, small=True)
    f = oracle.features(m.rowptr, m.colind)
    w = spmv.device_query(0)["access_window_max"]
    for mask in range(16):
        p = spmv.Plan(m.rowptr, m.colind, m.vals, select_mode=1, force_classes=mask)
        info = p.info()
        s, o = info["sel"], oracle.profile_select(f, None, w, classes=mask)
        assert (s["variant"], s["vs"], s["d16"], bool(s["xwin"]), s["classes"]) == \
            (o.variant, o.vs, o.d16, o.xwin, o.classes), (mask, s)
        assert info["profile_ms"] == 0.0  # no probes ran
        if mask in (0, 8, 4, 2):
            assert_bound(p.execute(m.x), m)
        p.destroy()


@pytest.mark.parametrize("which", ["C2", "st27_96"])
def test_profile_mode_second_stage_d8(which):
    """Stencils (CMP on the CSR baseline, D8-codable): the second stage times
    the plain stream kernel, which reaches P_MB, so MB and D8 are applied
    (reading 30); the D8 plan's results are within the per-row bound.
    (Tiny stencils such as C5's 20^3 test size are launch-bound: their CTA
    spread calls them IMB, reading 29.)"""
    m = sg.config(2) if which == "C2" else sg.stencil(96, 27, x_seed=5)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, select_mode=1)
    info = p.info()
    assert info["variant"] == "stream" and info["p_stream"] > 0
    b = {k: info[k] for k in PROFILE_KEYS}
    o = oracle.profile_select(oracle.features(m.rowptr, m.colind), b, spmv.device_query(0)["access_window_max"],
                              p_stream=info["p_stream"])
    assert (info["sel"]["d16"], info["sel"]["classes"]) == (o.d16, o.classes)
    if info["p_stream"] >= 0.9 * info["p_mb"]:
        assert info["sel"]["d16"] == 2 and "MB" in info["classes"] and info["d8_n_dict"] + info["d8_patterns"] > 0
    assert_bound(p.execute(m.x), m)
    xg, _ = p.iterate(m.x, 3)
    rc, xr, _ = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, 3)
    assert np.max(np.abs(xg - xr)) <= 1e-10 * np.max(np.abs(xr))
    for d in (0, 1):  # d16 = 0 (off) or 1 (16-bit deltas asked for): no second stage
        q = spmv.Plan(m.rowptr, m.colind, m.vals, select_mode=1, d16=d)
        assert q.info()["p_stream"] == 0.0 and q.info()["sel"]["d16"] != 2


def test_profile_mode_paper_thresholds_option():
    """t_imb / t_ml / approx_tol override the B200 defaults (Fig. 4 with the
    paper's KNC values)."""
    m = sg.config(3, small=True)
    f = oracle.features(m.rowptr, m.colind)
    w = spmv.device_query(0)["access_window_max"]
    for t in ((oracle.T_IMB, oracle.T_ML, oracle.APPROX_TOL), (50.0, 50.0, 0.5)):
        p = spmv.Plan(m.rowptr, m.colind, m.vals, select_mode=1, t_imb=t[0], t_ml=t[1], approx_tol=t[2])
        info = p.info()
        b = {k: info[k] for k in PROFILE_KEYS}
        o = oracle.profile_select(f, b, w, t_imb=t[0], t_ml=t[1], tol=t[2])
        s = info["sel"]
        assert (s["variant"], s["vs"], s["d16"], bool(s["xwin"]), s["classes"]) == \
            (o.variant, o.vs, o.d16, o.xwin, o.classes), (t, b, s)
        assert_bound(p.execute(m.x), m)
        p.destroy()


# full Table I on the device (f4) vs the oracle's definitions
@pytest.mark.parametrize("name,m", SUITE, ids=[n for n, _ in SUITE])
def test_table1_device(name, m):
    p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size)
    t = p.table1()
    o = oracle.table1(m.rowptr, m.colind, n_cols=m.x.size, l2_bytes=spmv.device_query(0)["l2_bytes"])
    for k in ("size_fits_l2", "n_nonempty", "bw_min", "bw_max", "nnz_min", "nnz_max"):
        assert t[k] == o[k], k
    for k in ("density", "nnz_avg", "nnz_sd", "bw_avg", "bw_sd", "scatter_avg", "scatter_sd", "clustering_avg",
              "misses_avg"):
        assert abs(t[k] - o[k]) <= 1e-12 * max(1.0, abs(o[k])), (k, t[k], o[k])


# ---- x-line reuse probe (gather cache mode of the nnz tiles) ----------------
def _splitmix(w):
    M = (1 << 64) - 1
    z = (w + 0x9E3779B97F4A7C15) & M
    z = ((z ^ (z >> 30)) * 0xBF58476D1CE4E5B9) & M
    z = ((z ^ (z >> 27)) * 0x94D049BB133111EB) & M
    return z ^ (z >> 31)


def _reuse_numpy(rp, ci):
    """Sampled fraction of nonzeros of row r (first 256) whose 16-column line
    row r-1 also touches; rows as the plan samples them (all when < 4097)."""
    rp = rp.astype(np.int64)
    n = rp.size - 1
    S = min(n - 1, 4096)
    hits = tot = 0
    for w in range(S):
        r = 1 + w if S == n - 1 else 1 + _splitmix(w) % (n - 1)
        a = ci[rp[r]:rp[r + 1]][:256] >> 4
        b = np.unique(ci[rp[r - 1]:rp[r]] >> 4)
        hits += int(np.isin(a, b).sum())
        tot += a.size
    return hits / tot if tot else 0.0


@pytest.mark.parametrize("kind", ["stencil", "random", "rmat_small"])
def test_x_reuse_probe(kind):
    if kind == "stencil":
        m = sg.stencil(48, 7)
    elif kind == "random":
        m = sg.randrows(300_000, 12, col_seed=5)
    else:
        m = sg.config(3, small=True)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, force_variant="nnzsplit")
    info = p.info()
    want = _reuse_numpy(m.rowptr, m.colind)
    assert info["x_reuse"] == pytest.approx(want, abs=1e-12)
    if kind == "stencil":
        assert want > 0.5 and info["nz_gather_l2"] == 0
    if kind == "random":
        assert want < 0.1 and info["nz_gather_l2"] == 1  # x = 2.4 MB > 1 MB
    y = p.execute(m.x)
    assert_bound(y, m)


# ---- D8: dictionary-coded 8-bit deltas (d8.cu; reading 26) -----------
def _d8_cases():
    g = np.random.default_rng(17)
    out = [("st7_9", sg.stencil(9, 7)), ("st27_11", sg.stencil(11, 27)), ("st27_20_rp64", sg.stencil(20, 27, rp64=True))]
    # banded rows from a small gap alphabet, ragged lengths incl. empty rows
    for name, n, lo, hi in (("banded_ragged", 5003, 0, 30), ("banded_long", 1500, 100, 255), ("tiny", 7, 1, 4)):
        lens = g.integers(lo, hi + 1, n)
        rp = np.zeros(n + 1, np.int64)
        np.cumsum(lens, out=rp[1:])
        ci = np.empty(int(rp[-1]), np.int32)
        for i in range(n):
            if lens[i]:
                steps = g.choice([1, 2, 5, 40], lens[i])
                steps[0] = g.integers(-min(i, 20), 20)
                ci[rp[i]:rp[i + 1]] = i + np.cumsum(steps)
        ncols = int(ci.max()) + 1 if ci.size else n
        out.append((name, sg.CSR(n, rp.astype(np.int32), ci, g.uniform(-1, 1, ci.size), g.uniform(-1, 1, ncols))))
    return out


D8_CASES = _d8_cases()


def _check_d8_structures(p, m, row_shift=0, g=0):
    """The plan's D8 structures equal the oracle's: row patterns (DESIGN.md
    reading 31) when the rows follow <= 256 of them, else dictionary codes;
    the device's own decode gives colind back (round trip). row_shift:
    global row id of the block's first row (emulated shards)."""
    rp = m.rowptr.astype(np.int64)
    pat = oracle.pat_encode(rp, m.colind.astype(np.int64) - row_shift)
    info = p.info()
    assert info["d16_width"] == 8
    if pat is not None and os.environ.get("SPMV_D8_PATTERNS", "1") != "0":
        ids, lens, ofs = pat
        assert info["d8_patterns"] == lens.size and info["d8_n_dict"] == 0
        assert np.array_equal(p.export("pat_ids", g), ids)
        assert np.array_equal(p.export("pat_len", g), lens) and np.array_equal(p.export("pat_ofs", g), ofs)
        assert p.export("d8_codes", g).size == 0
    else:
        d, codes, rlen = oracle.d8_encode(m.rowptr, m.colind)
        assert info["d8_patterns"] == 0 and info["d8_n_dict"] == d.size
        assert np.array_equal(p.export("d8_dict", g), d)
        assert np.array_equal(p.export("d8_codes", g), codes)
        assert np.array_equal(p.export("d8_rlen", g), rlen)
    assert np.array_equal(p.export("decoded", g), m.colind)  # device decode, round trip


@pytest.mark.parametrize("mode", ["patterns", "codes"])
@pytest.mark.parametrize("name,m", D8_CASES, ids=[n for n, _ in D8_CASES])
def test_d8_structures_and_parity(name, m, mode, monkeypatch):
    if mode == "codes":
        monkeypatch.setenv("SPMV_D8_PATTERNS", "0")
    enc = oracle.d8_encode(m.rowptr, m.colind)
    assert enc is not None
    d, codes, rlen = enc
    p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, force_variant="stream", d16=2)
    info = p.info()
    assert info["sel"]["d16"] == 2 and info["feat"]["n_deltas"] == d.size
    _check_d8_structures(p, m)
    Rt = info["rows_per_tile"]
    assert Rt % 16 == 0 and np.array_equal(p.export("tile_rows"), np.minimum(np.arange(info["n_tiles"] + 1) * Rt, m.n))
    y = p.execute(m.x, np.full(m.n, np.nan))
    assert_bound(y, m)
    assert np.all(y[np.diff(m.rowptr.astype(np.int64)) == 0] == 0.0)
    # dyadic inputs: every order exact -> bit-equal (a wrong column shows up)
    g = np.random.default_rng(3)
    xv = g.integers(-1024, 1025, m.x.size) / 1024.0
    vv = g.integers(-1024, 1025, m.vals.size) / 1024.0
    pd = spmv.Plan(m.rowptr, m.colind, vv, n_cols=m.x.size, force_variant="stream", d16=2)
    assert np.array_equal(pd.execute(xv), oracle.spmv(m.rowptr, m.colind, vv, xv))


@pytest.mark.parametrize("un", ["7", "8", "9", "16"])
@pytest.mark.parametrize("pts", [7, 27])
def test_d8_pattern_batch_widths(monkeypatch, un, pts):
    """Row-pattern D8 at every batch width (the plan picks 9 for 27-pt rows,
    7 for 7-pt rows): y within the bound, dyadic inputs bit-exact, and the
    iterated mode vs the oracle."""
    monkeypatch.setenv("SPMV_D8_UN", un)
    m = sg.stencil(20, pts, x_seed=6)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, force_variant="stream", d16=2)
    assert p.info()["d8_patterns"] == 27
    assert_bound(p.execute(m.x), m)
    g = np.random.default_rng(5)
    xv = g.integers(-1024, 1025, m.n) / 1024.0
    assert np.array_equal(p.execute(xv), oracle.spmv(m.rowptr, m.colind, m.vals, xv))
    xg, nug = p.iterate(m.x, 12)
    rc, xr, nur = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, 12)
    assert np.max(np.abs(xg - xr)) <= 1e-10 * np.max(np.abs(xr)) and np.all(np.abs(nug - nur) <= 1e-12 * nur)


@pytest.mark.parametrize("cw", ["4", "6", "8"])
def test_d8_consumer_warp_counts(monkeypatch, cw):
    monkeypatch.setenv("SPMV_D8_CW", cw)
    m = sg.stencil(24, 27, x_seed=5)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, force_variant="stream", d16=2)
    assert p.info()["stream_stages"] == int(cw)
    assert_bound(p.execute(m.x), m)


@pytest.mark.parametrize("mode", ["patterns", "codes"])
@pytest.mark.parametrize("G", [2, 3])
def test_d8_emulated_shards(G, mode, monkeypatch):
    if mode == "codes":
        monkeypatch.setenv("SPMV_D8_PATTERNS", "0")
    m = sg.stencil(16, 27, x_seed=2)
    d, codes, rlen = oracle.d8_encode(m.rowptr, m.colind)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, ngpus=G, emulate_devices=1, force_variant="stream", d16=2)
    b = p.info()["shard_bounds"]
    rp = m.rowptr.astype(np.int64)
    for g in range(G):
        sl = slice(rp[b[g]], rp[b[g + 1]])
        if mode == "codes":  # one global dictionary; shard g's codes are the oracle's slice
            assert np.array_equal(p.export("d8_dict", g), d)
            assert np.array_equal(p.export("d8_codes", g), codes[sl])
        else:  # shard g's patterns: the oracle's on its rows, offsets from the global row id
            ids, lens, ofs = oracle.pat_encode(rp[b[g]:b[g + 1] + 1] - rp[b[g]], m.colind[sl].astype(np.int64) - b[g])
            assert np.array_equal(p.export("pat_ids", g), ids) and np.array_equal(p.export("pat_ofs", g), ofs)
            assert np.array_equal(p.export("pat_len", g), lens)
        assert np.array_equal(p.export("decoded", g), m.colind[sl])
    assert_bound(p.execute(m.x), m)
    # iterated mode through D8 shards (fused per-tile norm partials)
    rc, xr, nur = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, 30)
    xg, nug = p.iterate(m.x, 30)
    assert np.max(np.abs(xg - xr)) <= 1e-10 * np.max(np.abs(xr))
    assert np.all(np.abs(nug - nur) <= 1e-12 * nur)


def test_d8_auto_selected_on_c2_and_host_pipeline(monkeypatch):
    m = sg.config(2)
    p = spmv.Plan(m.rowptr, m.colind, m.vals)
    info = p.info()
    # 27 row patterns (one per boundary class): one byte per row, no per-nonzero index
    assert info["variant"] == "stream" and info["sel"]["d16"] == 2 and info["d8_patterns"] == 27
    assert info["kernel_bytes"] == 8 * m.nnz + m.n + 8 * (info["n_tiles"] + 1) + 16 * m.n
    _check_d8_structures(p, m)
    monkeypatch.setenv("SPMV_D8_PATTERNS", "0")  # the 8-bit codes
    q = spmv.Plan(m.rowptr, m.colind, m.vals)
    iq = q.info()
    monkeypatch.delenv("SPMV_D8_PATTERNS")
    assert iq["d8_n_dict"] == 10 and iq["d8_patterns"] == 0
    assert iq["kernel_bytes"] == 9 * m.nnz + m.n + 8 * (iq["n_tiles"] + 1) + 16 * m.n
    y = p.execute(m.x)
    assert_bound(y, m)
    ones = np.ones(m.n)
    assert np.array_equal(p.execute(ones), oracle.spmv(m.rowptr, m.colind, m.vals, ones))
    monkeypatch.setenv("SPMV_HOST_PIPE_MIN_BYTES", "1")
    monkeypatch.setenv("SPMV_HOST_PIPE_BLOCKS", "7")
    p2 = spmv.Plan(m.rowptr, m.colind, m.vals)
    assert np.array_equal(p2.execute(m.x, np.full(m.n, np.nan)), y)  # pipelined host path, same arithmetic


def test_d16_row_tiles_random_x():
    # forced 16-bit deltas on row-count tiles (no tile_nnz), one lane
    # per row and VS > 1, random x so a wrong decoded column cannot hide
    g = np.random.default_rng(23)
    for lens, vs in (([7] * 20000, 1), ([40] * 3000, 4)):
        lens = np.asarray(lens, np.int64)
        m = sg.from_lengths(lens, 30000, g, sg.MODE_U11, sg.MODE_U11)
        p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, force_variant="stream", d16=1, force_vs=vs)
        info = p.info()
        assert info["sel"]["d16"] == 1 and info["rows_per_tile"] > 0
        if vs == 1:
            assert info["stream_stages"] == 6
        assert_bound(p.execute(m.x), m)
        assert np.array_equal(p.export("decoded"), m.colind)


def test_core_plan_create_signature():
    # the north_star call exactly: spmv_plan_create(n, nnz, int64 rowptr, int32
    # colind, fp64 values, ngpus) -> opaque plan (NULL on failure), spmv_execute,
    # spmv_plan_destroy (include/spmv.h), through ctypes on host arrays
    import ctypes
    lib = spmv.binding.lib
    m = sg.stencil(12, 27, x_seed=4)
    rp = m.rowptr.astype(np.int64)
    h = lib.spmv_plan_create(m.n, m.nnz, rp.ctypes.data, m.colind.ctypes.data, m.vals.ctypes.data, 1)
    assert h
    y = np.full(m.n, np.nan)
    assert lib.spmv_execute(ctypes.c_void_p(h), m.x.ctypes.data, y.ctypes.data) == 0
    assert_bound(y, m)
    lib.spmv_plan_destroy(ctypes.c_void_p(h))
    # failure leaves no plan: invalid CSR -> NULL and a located message
    bad = rp.copy()
    bad[-1] += 1
    assert not lib.spmv_plan_create(m.n, m.nnz, bad.ctypes.data, m.colind.ctypes.data, m.vals.ctypes.data, 1)
    assert lib.spmv_last_status() == -2 and b"rowptr[n] != nnz" in lib.spmv_last_error()
    assert not lib.spmv_plan_create(m.n, m.nnz, rp.ctypes.data, m.colind.ctypes.data, m.vals.ctypes.data, 0)
    assert lib.spmv_last_status() == -1


def test_x_window_limit_reset_on_destroy():
    # ML plans set a persisting-L2 carve-out for the x window; the last plan
    # holding it gives it back on destroy
    m = sg.config(3, small=True)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, force_variant="nnzsplit", xwin=1)
    assert p.info()["sel"]["xwin"] == 1
    assert_bound(p.execute(m.x), m)
    assert _persist_limit() > 0
    p.destroy()
    assert _persist_limit() == 0


def _persist_limit():
    # the device-wide limit through the CUDA runtime (same primary context)
    import ctypes
    import glob
    libs = sorted(glob.glob("/usr/local/cuda/lib64/libcudart.so*"))
    rt = ctypes.CDLL(libs[0])
    v = ctypes.c_size_t(0)
    assert rt.cudaDeviceGetLimit(ctypes.byref(v), 0x06) == 0  # cudaLimitPersistingL2CacheSize
    return v.value


@pytest.mark.parametrize("scale", [1e40, 1e-40, 1.0])
@pytest.mark.parametrize("G,d16", [(1, 2), (1, 0), (2, 2), (3, 0)])
def test_iterated_fused_paths_rescale(scale, G, d16):
    # row-aligned STREAM / D8 plans: one shard runs the lagged one-launch
    # iteration (the norm folded by the next launch's producer lanes, the
    # exact rescale decided one step late, reading 27); several shards the
    # interior-first launches with per-launch partials. ~1e40-scaled values
    # make the rescale fire every few steps.
    m = sg.stencil(16, 27, x_seed=6)
    vals = m.vals * scale
    K = 60
    rc, xr, nur = oracle.power_iter(m.rowptr, m.colind, vals, m.x, K)
    assert rc == 0
    p = spmv.Plan(m.rowptr, m.colind, vals, ngpus=G, emulate_devices=1, force_variant="stream", d16=d16)
    assert p.info()["sel"]["d16"] == d16
    for k in (1, 2, 3, K):
        xg, nug = p.iterate(m.x, k)
        rc, xk, nuk = oracle.power_iter(m.rowptr, m.colind, vals, m.x, k)
        assert np.all(np.isfinite(xg)) and np.all(np.isfinite(nug))
        assert np.max(np.abs(xg - xk)) <= 1e-10 * np.max(np.abs(xk)), k
        assert np.all(np.abs(nug - nuk) <= 1e-12 * nuk), k


@pytest.mark.parametrize("G,d16", [(2, 0), (3, 2), (4, 2), (8, 0)])
def test_iterated_halo_push(G, d16, monkeypatch):
    """Multi-shard iteration with the halo exchange fused into the SpMV
    (each shard's kernel stores the rows its neighbours read into their next
    replicas): banded row blocks take it; the result matches
    the per-step oracle and the halo-copy path (SPMV_NO_PUSH)."""
    m = sg.stencil(12, 27, x_seed=8)  # 1728 rows, band 157: every shard reads only its neighbours at G <= 8
    K = 40
    rc, xr, nur = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, K)
    assert rc == 0
    p = spmv.Plan(m.rowptr, m.colind, m.vals, ngpus=G, emulate_devices=1, force_variant="stream", d16=d16)
    xg, nug = p.iterate(m.x, K)
    assert p.info()["iter_push"] == 1
    assert np.max(np.abs(xg - xr)) <= 1e-10 * np.max(np.abs(xr))
    assert np.all(np.abs(nug - nur) <= 1e-12 * nur)
    for k in (1, 2, 7):  # the exchange of the first steps
        xk, _ = p.iterate(m.x, k)
        rc, xo, _ = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, k)
        assert np.max(np.abs(xk - xo)) <= 1e-10 * np.max(np.abs(xo)), k
    monkeypatch.setenv("SPMV_NO_PUSH", "1")
    q = spmv.Plan(m.rowptr, m.colind, m.vals, ngpus=G, emulate_devices=1, force_variant="stream", d16=d16)
    xc, nuc = q.iterate(m.x, K)
    assert q.info()["iter_push"] == 0
    assert np.max(np.abs(xg - xc)) <= 1e-13 * np.max(np.abs(xc))  # same SpMVs; the norm partials group differently
    assert np.all(np.abs(nug - nuc) <= 1e-13 * nuc)


def test_iterated_push_not_for_scattered_blocks():
    # every shard of a random square matrix reads every block: no prefix /
    # suffix halo, the halo copies run instead (still matching the oracle)
    m = sg.randrows(3000, 6, diag=True, col_seed=11, val_seed=12, x_seed=13, val_mode=sg.MODE_U01)
    K = 20
    rc, xr, nur = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, K)
    assert rc == 0
    p = spmv.Plan(m.rowptr, m.colind, m.vals, ngpus=3, emulate_devices=1, force_variant="stream", seg=0)
    assert p.info()["tiles_row_aligned"] == 1 and p.info()["sel"]["seg"] == 0  # the fused-capable kernel
    xg, nug = p.iterate(m.x, K)
    assert p.info()["iter_push"] == 0
    assert np.max(np.abs(xg - xr)) <= 1e-10 * np.max(np.abs(xr))
    assert np.all(np.abs(nug - nur) <= 1e-12 * nur)


@pytest.mark.parametrize("mode", ["patterns", "codes"])
@pytest.mark.parametrize("rb,re", [(0, 3000), (2000, 5500), (5000, 8000)])
def test_d8_row_block_plan(rb, re, mode, monkeypatch):
    if mode == "codes":
        monkeypatch.setenv("SPMV_D8_PATTERNS", "0")
    # one rank's row block of a 27-pt stencil (the torchrun layout: n_rows <
    # n_cols, rowptr rebased, global column ids): D8 head deltas are taken
    # against the block's local row ids -- the oracle encodes the block the same way
    full = sg.stencil(20, 27, x_seed=9)
    blk = sg.stencil(20, 27, x_seed=9, rows=(rb, re))
    enc = oracle.d8_encode(blk.rowptr, blk.colind)
    assert enc is not None
    p = spmv.Plan(blk.rowptr, blk.colind, blk.vals, n_cols=full.n, force_variant="stream", d16=2)
    assert p.info()["sel"]["d16"] == 2
    _check_d8_structures(p, blk)
    y = p.execute(full.x)
    m = sg.CSR(re - rb, blk.rowptr, blk.colind, blk.vals, full.x)
    assert_bound(y, m)


UPDATE_CASES = [  # (config builder, plan options)
    ("C2 D8", lambda: sg.config(2, small=True), dict()),
    ("C2 D8 packed", lambda: sg.config(2, small=True), dict(force_variant="stream", d16=2)),
    ("C3 nnz_split hot-x", lambda: sg.config(3, small=True), dict(force_variant="nnzsplit", hot_x=512)),
    ("C4 split (bin)", lambda: sg.config(4, small=True), dict(force_variant="split")),
    ("C4 split bins", lambda: sg.config(4, small=True), dict(force_variant="split", split_bins=0)),
    ("C4 split TMA long rows", lambda: sg.config(4, small=True), dict(force_variant="split", long_mode=3)),
    ("C3 merge", lambda: sg.config(3, small=True), dict(force_variant="merge")),
    ("C3 vector", lambda: sg.config(3, small=True), dict(force_variant="vector")),
    ("C5 3 shards", lambda: sg.config(5, small=True), dict(ngpus=3, emulate_devices=1)),
]


@pytest.mark.parametrize("name,mk,opts", UPDATE_CASES, ids=[c[0] for c in UPDATE_CASES])
def test_plan_update_values(name, mk, opts, monkeypatch):
    """spmv_plan_update_values: new values on the same pattern give the
    oracle's result for the new values (every value-derived copy refreshed),
    from host and from device memory; the iterated mode sees them too."""
    if "packed" in name:
        monkeypatch.setenv("SPMV_D8_PACKED", "1")
    m = mk()
    p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, **opts)
    g = np.random.default_rng(17)
    for src in ("host", "device"):
        v2 = g.uniform(-1, 1, m.vals.size)
        if src == "host":
            p.update_values(v2)
        else:
            p.update_values(torch.from_numpy(v2).cuda())
        m2 = sg.CSR(m.n, m.rowptr, m.colind, v2, m.x)
        assert_bound(p.execute(m.x), m2)
    if m.n == m.x.size and "C5" in name:
        v3 = np.abs(v2) + 0.1
        p.update_values(v3)
        xg, _ = p.iterate(m.x, 5)
        rc, xr, _ = oracle.power_iter(m.rowptr, m.colind, v3, m.x, 5)
        assert np.max(np.abs(xg - xr)) <= 1e-10 * np.max(np.abs(xr))
    p.destroy()


def _rows_matrix(rows, n_cols, seed):
    """CSR from explicit per-row column lists (ascending), random values / x."""
    g = np.random.default_rng(seed)
    rp = np.concatenate([[0], np.cumsum([len(r) for r in rows])]).astype(np.int32)
    ci = np.concatenate([np.asarray(r, np.int32) for r in rows]) if rp[-1] else np.zeros(0, np.int32)
    return sg.CSR(len(rows), rp, ci, g.uniform(-1, 1, ci.size), g.uniform(-1, 1, n_cols))


@pytest.mark.parametrize("case", ["256_patterns", "257_patterns", "4096_offsets", "4186_offsets"])
def test_d8_pattern_limits(case):
    """Row-pattern mode at its limits (reading 31): 256 patterns / 4096
    offsets use it, 257 patterns / more offsets fall back to the dictionary
    codes -- the same decision as oracle.pat_encode; structures, bound and
    dyadic bit-exactness either way."""
    if case.endswith("patterns"):
        # row i: the single column i + i (offset i: 256 patterns, 256 deltas), plus (257) one row {i, i+1}
        rows = [[2 * i] for i in range(256)]
        if case == "257_patterns":
            rows.append([len(rows), len(rows) + 1])
    else:
        top = 90 if case == "4096_offsets" else 91  # sum 1..90 = 4095, 1..91 = 4186
        rows = [list(range(i, i + L)) for i, L in enumerate(range(1, top + 1))]
    rows = rows * 3  # repeat: rows reuse their first occurrence
    rows = [[c + i - (i % (len(rows) // 3)) for c in r] for i, r in enumerate(rows)]
    m = _rows_matrix(rows, 3 * len(rows) + 300, 7)
    want = oracle.pat_encode(m.rowptr, m.colind)
    assert (want is not None) == (case in ("256_patterns", "4096_offsets"))
    p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, force_variant="stream", d16=2)
    info = p.info()
    assert info["sel"]["d16"] == 2
    assert (info["d8_patterns"] > 0) == (want is not None)
    _check_d8_structures(p, m)
    assert_bound(p.execute(m.x), m)
    g = np.random.default_rng(2)
    xv = g.integers(-1024, 1025, m.x.size) / 1024.0
    vv = g.integers(-1024, 1025, m.vals.size) / 1024.0
    pd = spmv.Plan(m.rowptr, m.colind, vv, n_cols=m.x.size, force_variant="stream", d16=2)
    assert np.array_equal(pd.execute(xv), oracle.spmv(m.rowptr, m.colind, vv, xv))
