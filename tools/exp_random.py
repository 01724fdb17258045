"""Uniform random rows (k distinct columns per row, SURVEY C1/C4 structure) at
several sizes: auto plan vs forced variants (experiment tool for the ML rule).
  python tools/exp_random.py --sizes 100000,1000000,4000000 --k 8,15,30"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1711_05487_b200 as spmv
import synthgen as sg

ap = argparse.ArgumentParser()
ap.add_argument("--sizes", default="100000,1000000,4000000")
ap.add_argument("--k", default="8,15,30")
ap.add_argument("--variants", default="auto,stream,nnzsplit,vector")
ap.add_argument("--reps", type=int, default=50)
a = ap.parse_args()


def timeit(m, **opts):
    p = spmv.Plan(m.rowptr, m.colind, m.vals, n_cols=m.n, **opts)
    xd, yd = p.x_device(), p.y_device()
    p.execute(m.x, np.empty(p.n_rows))
    st = torch.cuda.ExternalStream(p.stream())
    for _ in range(5):
        p.execute_async(xd, yd)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    for _ in range(a.reps):
        p.execute_async(xd, yd)
    e.record(st)
    e.synchronize()
    info = p.info()
    p.destroy()
    return s.elapsed_time(e) / a.reps, info


for n in [int(v) for v in a.sizes.split(",")]:
    for k in [int(v) for v in a.k.split(",")]:
        m = sg.randrows(n, k)
        for var in a.variants.split(","):
            opts = {} if var == "auto" else {"force_variant": var}
            ms, info = timeit(m, **opts)
            print(json.dumps({"n": n, "k": k, "nnz": m.nnz, "req": var, "variant": info["variant"],
                              "seg": info["sel"]["seg"], "classes": info["classes"], "us": round(ms * 1e3, 1)}),
                  flush=True)
