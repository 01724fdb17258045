"""One small execution of every kernel path, for compute-sanitizer
(memcheck / racecheck / synccheck / initcheck):
  compute-sanitizer --tool memcheck python tools/sanitize_suite.py
Each case checks its result against the oracle (test infrastructure) so a
sanitizer-clean run is also a correct one."""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import oracle
import synthgen as sg
import paper_1711_05487_b200 as spmv

g = np.random.default_rng(3)


def check(name, m, **kw):
    p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, **kw)
    y = p.execute(m.x)
    yr = oracle.spmv(m.rowptr, m.colind, m.vals, m.x)
    s = oracle.absrow(m.rowptr, m.colind, m.vals, m.x)
    ok = bool(np.all(np.abs(y - yr) <= 1e-12 * s))
    print(f"{name:40s} {p.info()['variant']:9s} d16={p.info()['sel']['d16']} ok={ok}", flush=True)
    assert ok
    return p


st = sg.stencil(12, 27, x_seed=1)
st7 = sg.stencil(16, 7, x_seed=2)
pl = sg.config(3, small=True)
c4 = sg.config(4, small=True)
lens = np.asarray([3, 0, 9, 27, 1, 64] * 300, np.int64)
mixed = sg.from_lengths(lens, 3000, g)
huge = sg.from_lengths(np.asarray([5] * 2000 + [3000] + [5] * 2000, np.int64), 4001, g)
check("stream row tiles (27-pt)", st, force_variant="stream", d16=0)
check("stream row tiles CW6 (7-pt)", st7, force_variant="stream", d16=0)
check("stream D8 row patterns (27-pt)", st, force_variant="stream", d16=2)
check("stream D8 row patterns (7-pt)", st7, force_variant="stream", d16=2)
os.environ["SPMV_D8_PATTERNS"] = "0"  # the dictionary codes (row patterns are the default D8 path)
check("stream D8 codes (27-pt)", st, force_variant="stream", d16=2)
check("stream D8 codes (7-pt)", st7, force_variant="stream", d16=2)
del os.environ["SPMV_D8_PATTERNS"]
check("stream D16 row tiles", st7, force_variant="stream", d16=1)
check("stream D16 escapes nnz tiles", st, force_variant="stream", d16=1, tile_nnz=512)
check("stream nnz tiles + fix-up", mixed, force_variant="stream", tile_nnz=512, no_aligned=1)
check("stream seg mode", mixed, force_variant="stream", seg=1, tile_nnz=384)
check("stream VS=8", mixed, force_variant="stream", force_vs=8, tile_nnz=512)
check("nnz_split plain", pl, force_variant="nnzsplit", hot_x=0)
check("nnz_split hot-x", pl, force_variant="nnzsplit", hot_x=512)
check("nnz_split long rows (fix-up)", huge, force_variant="nnzsplit")
check("split fused (tiled long rows)", c4, force_variant="split")
check("split chunks", c4, force_variant="split", long_mode=1)
check("split TMA long rows (long_mode 3)", c4, force_variant="split", long_mode=3)
check("profile mode + second stage (27-pt)", sg.stencil(48, 27, x_seed=4), select_mode=1)
check("merge path", mixed, force_variant="merge")
check("csr_vector VS=4", mixed, force_variant="vector", force_vs=4)
# hierarchical fix-up: a row cut into > 2048 tiles
big = sg.from_lengths(np.asarray([3, 300000, 2], np.int64), 300000, g)
check("merge hierarchical fix-up", big, force_variant="merge")
# iterated mode: fused epilogue (one shard) and emulated shards
# (G > 1: the halo push -- each shard's kernel stores its halo rows into the
# neighbours' replicas -- for both the D8 and the int32 stream kernels; the
# 1e40-scaled values make the exact rescale (and its pushed copies) fire)
for G, d16, scale in ((1, 2, 1.0), (2, 2, 1.0), (3, 2, 1e40), (3, 0, 1e40), (4, 0, 1.0)):
    vals = st.vals * scale
    p = spmv.Plan(st.rowptr, st.colind, vals, ngpus=G, emulate_devices=1, force_variant="stream", d16=d16)
    x, nu = p.iterate(st.x, 8)
    rc, xr, nur = oracle.power_iter(st.rowptr, st.colind, vals, st.x, 8)
    ok = bool(np.max(np.abs(x - xr)) <= 1e-10 * np.max(np.abs(xr)))
    print(f"iterate G={G} d16={d16} scale={scale:g} push={p.info()['iter_push']:<14d} ok={ok}", flush=True)
    assert ok
print("sanitize suite done")
