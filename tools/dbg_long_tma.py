"""Debug (tools only): run each long_mode 3 case of tests/test_gpu_parity.py
LONG_TMA_CASES and the small suite under a per-case timeout."""
import os, subprocess, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
CASES = [(5001, 6, 300, 1500, 64), (20000, 15, 10, 4500, 64), (3000, 4, 3, 2990, 64), (70001, 3, 5, 60000, 4096),
         (9000, 5, 40, 300, 64)]
if len(sys.argv) > 1:
    import numpy as np, time
    import synthgen as sg, oracle
    import paper_1711_05487_b200 as spmv
    which = sys.argv[1]
    if which == "suite":
        for name, m in sg.small_suite(seed=21):
            t = time.time()
            p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.x.size, force_variant="split", force_vs=8, l_split=64,
                          tile_nnz=512, long_mode=3)
            y = p.execute(m.x)
            r = oracle.spmv(m.rowptr, m.colind, m.vals, m.x)
            print(name, p.info()["long_mode"], p.info()["long_rg"], float(np.abs(y - r).max()), f"{time.time()-t:.2f}s",
                  flush=True)
    else:
        n, k, nl, kl, ls = CASES[int(which)]
        m = sg.randrows(n, k, diag=False, long_rows=sg.pick_rows(n, nl, 77 + n), k_long=kl, col_seed=5 + n,
                        val_seed=6, x_seed=7)
        p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=n, force_variant="split", long_mode=3, l_split=ls)
        print("plan", p.info()["long_mode"], p.info()["long_rg"], flush=True)
        y = p.execute(m.x)
        r = oracle.spmv(m.rowptr, m.colind, m.vals, m.x)
        print("case", which, float(np.abs(y - r).max()), flush=True)
    sys.exit(0)
for c in ["suite"] + [str(i) for i in range(len(CASES))]:
    try:
        out = subprocess.run([sys.executable, __file__, c], capture_output=True, text=True, timeout=60)
        print(c, "rc", out.returncode, out.stdout[-2000:], out.stderr[-1500:], flush=True)
    except subprocess.TimeoutExpired as e:
        print(c, "TIMEOUT", (e.stdout or b"")[-2000:], flush=True)
