import sys, os
sys.path.insert(0, os.getcwd())
import numpy as np, oracle, synthgen as sg, paper_1711_05487_b200 as spmv
m = sg.config(5, small=True)
for K2 in (50, 100):
    rc, xr2, nur2 = oracle.power_iter(m.rowptr, m.colind, m.vals, m.x, K2)
    for v in ("stream", "vector"):
        p = spmv.Plan(m.rowptr, m.colind, m.vals, force_variant=v)
        xg, nug = p.iterate(m.x, K2)
        print(os.environ.get("SPMV_PDL"), v, K2, "xerr", np.max(np.abs(xg - xr2)) / np.max(np.abs(xr2)), flush=True)
