"""CPU-side checks of the C-ABI library (no GPU needed): it loads, exports
every symbol include/spmv.h declares, and its host-only functions (shard
bounds, selection) agree with the oracle."""
import ctypes
import os
import re

import numpy as np
import pytest

import oracle
import synthgen as sg

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def header_functions():
    src = open(os.path.join(ROOT, "include", "spmv.h")).read()
    src = re.sub(r"/\*.*?\*/", "", src, flags=re.S)
    return sorted(set(re.findall(r"\b(spmv_[a-z_0-9]+)\s*\(", src)))


def test_library_exports_every_declared_symbol():
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1711_05487_b200", "libspmv.so"))
    names = header_functions()
    assert len(names) >= 20
    missing = [n for n in names if not hasattr(lib, n)]
    assert not missing, missing


def test_binding_imports_and_has_no_oracle_dependency():
    import paper_1711_05487_b200 as pkg
    import sys
    assert pkg.lib is not None
    for mod in list(sys.modules):
        if mod.startswith("paper_1711_05487_b200"):
            src = getattr(sys.modules[mod], "__file__", None)
            if src and src.endswith(".py"):
                text = open(src).read()
                assert "import oracle" not in text and "from oracle" not in text


def test_no_cpu_fallback_in_product_sources():
    # the product path never imports, includes or loads the oracle
    pkg = os.path.join(ROOT, "paper_1711_05487_b200")
    bad = re.compile(r"import oracle|from oracle|#include\s*\"[^\"]*oracle|liboracle|oracle\.c")
    for dirpath, _, files in os.walk(pkg):
        for f in files:
            if f.endswith((".py", ".cu", ".cuh", ".h", ".cpp")):
                assert not bad.search(open(os.path.join(dirpath, f)).read()), f


def test_shard_bounds_host_function_matches_oracle():
    import paper_1711_05487_b200 as pkg
    g = np.random.default_rng(11)
    for t in range(40):
        n = int(g.integers(1, 500))
        lens = g.choice([0, 1, 3, 40, 0], n) if t % 2 else g.integers(0, 30, n)
        rp = np.zeros(n + 1, np.int64)
        np.cumsum(lens, out=rp[1:])
        for G in (1, 2, 3, 4, 8):
            exp = oracle.shard_bounds(rp, G)
            assert np.array_equal(pkg.shard_bounds(rp, G), exp)
            assert np.array_equal(pkg.shard_bounds(rp.astype(np.int32), G), exp)


def _props(l2=126 * 2 ** 20, win=128 * 2 ** 20):
    return dict(sm_count=148, cc_major=10, cc_minor=0, l2_bytes=l2, persisting_l2_max=l2 * 3 // 4,
                access_window_max=win, global_mem_bytes=180 * 2 ** 30)


@pytest.mark.parametrize("c", [1, 2, 3, 4, 5])
def test_selection_matches_oracle_on_config_features(c):
    import paper_1711_05487_b200 as pkg
    m = sg.config(c, small=True)
    f = oracle.features(m.rowptr, m.colind)
    rpb = m.rowptr.dtype.itemsize
    for l2 in (2 ** 20, 126 * 2 ** 20):
        p = _props(l2)
        s = pkg.select(f, p, rpb)
        o = oracle.select(f, p["l2_bytes"], p["access_window_max"], rpb)
        assert (s["variant"], s["vs"], s["d16"], bool(s["xwin"]), s["classes"]) == \
            (o.variant, o.vs, o.d16, o.xwin, o.classes)


def test_selection_matches_oracle_on_random_features():
    import paper_1711_05487_b200 as pkg
    g = np.random.default_rng(5)
    for _ in range(300):
        n = int(g.integers(1, 10 ** 7))
        avg = float(g.choice([0.5, 3, 7, 15, 27, 40, 200]))
        nnz = int(n * avg)
        f = dict(n=n, nnz=nnz, nnz_min=0, nnz_max=int(g.choice([avg, avg + 1, avg * 2, avg * 500, 10 ** 6])),
                 n_deltas=int(g.choice([1, 15, 256, 257])),
                 n_empty=int(n * g.choice([0, 0.1, 0.3, 0.6])), n_long=int(g.choice([0, 0, 5, 100])),
                 nnz_long=int(g.choice([0, 10 ** 5, 10 ** 7])), n_cols=int(n * g.choice([1, 0.1, 10])),
                 n_big_gaps=int(g.choice([0, 4, 64, 65, 129])),
                 col_min=0, col_max=n - 1,
                 n_short=n, max_short=0, s1=nnz, s2=0, s1_short=0, s2_short=0,
                 maxgap=int(g.choice([3, 300, 70000, 10 ** 6])), misses=int(nnz * g.choice([0.1, 0.6, 0.9])),
                 nnz_avg=nnz / n, nnz_sd=1.0, avg_short=avg, sd_short=avg * float(g.choice([0.1, 0.9, 1.5])))
        p = _props(int(g.choice([2 ** 20, 50 * 2 ** 20, 126 * 2 ** 20])))
        s = pkg.select(f, p, 4)
        o = oracle.select(f, p["l2_bytes"], p["access_window_max"], 4)
        assert (s["variant"], s["vs"], s["d16"], bool(s["xwin"]), s["classes"]) == \
            (o.variant, o.vs, o.d16, o.xwin, o.classes), f


def test_invalid_options_rejected_without_gpu():
    import paper_1711_05487_b200 as pkg
    f = oracle.features(np.array([0, 1]), np.array([0], np.int32))
    with pytest.raises(pkg.SpmvError):
        pkg.select(f, _props(), 4, force_vs=3)
    with pytest.raises(pkg.SpmvError):
        pkg.select(f, _props(), 4, tile_nnz=100)
    # Fig. 4 hyperparameters and the forced class set (profile mode)
    for bad in (dict(t_imb=-1.0), dict(t_ml=float("nan")), dict(approx_tol=1.0), dict(force_classes=16),
                dict(force_classes=-2)):
        with pytest.raises(pkg.SpmvError):
            pkg.select(f, _props(), 4, **bad)
    pkg.select(f, _props(), 4, t_imb=1.24, t_ml=1.25, approx_tol=0.1, force_classes=15)


def test_null_plan_arguments_fail_with_status_not_crash():
    # every plan-taking entry point rejects a NULL plan with SPMV_E_ARG (-1)
    # and a message, without touching a device (include/spmv.h conventions)
    lib = ctypes.CDLL(os.path.join(ROOT, "paper_1711_05487_b200", "libspmv.so"))
    vp = ctypes.c_void_p
    lib.spmv_last_error.restype = ctypes.c_char_p
    buf = (ctypes.c_double * 16)()
    calls = {
        "spmv_execute": (vp(None), buf, buf),
        "spmv_execute_async": (vp(None), buf, buf),
        "spmv_execute_norm": (vp(None), buf, buf, buf),
        "spmv_norm_partials": (vp(None), buf, buf),
        "spmv_norm_step": (vp(None), buf, ctypes.c_int(4), buf, buf),
        "spmv_iter_step": (vp(None), buf, buf, buf, buf, buf),
        "spmv_unit": (vp(None), buf, ctypes.c_int64(4), buf, buf),
        "spmv_plan_update_values": (vp(None), buf),
    }
    for name, args in calls.items():
        rc = getattr(lib, name)(*args)
        assert rc == -1, name
        assert lib.spmv_last_error(), name


def test_binding_struct_layouts_match_the_library():
    """Every ctypes struct of the binding has the size of its C twin
    (spmv_abi_sizes): a field added on one side only would make the library
    write past the binding's buffer (spmv_plan_query) or read garbage."""
    import paper_1711_05487_b200 as pkg
    B = pkg.binding
    out = (ctypes.c_int64 * 6)()
    assert B.lib.spmv_abi_sizes(out, 6) == 6
    mine = [ctypes.sizeof(c) for c in (B.Options, B.Features, B.DeviceProps, B.Selection, B.PlanInfo, B.Table1)]
    assert list(out) == mine, (list(out), mine)
