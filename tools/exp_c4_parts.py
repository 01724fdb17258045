"""Experiment (tools only): where C4's time goes. Times the full C4 matrix and
its two halves -- the 1M short rows alone (15 random columns each) and the
100 long rows alone (200,000 columns each, every other row empty) -- under
several forced variants.
  python tools/exp_c4_parts.py"""
import os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synthgen as sg
import paper_1711_05487_b200 as spmv


def time_plan(p, n_rows, x, reps=30):
    xd, yd = p.x_device(), p.y_device()
    p.execute(x, np.empty(n_rows))
    st = torch.cuda.ExternalStream(p.stream())
    for _ in range(5):
        p.execute_async(xd, yd)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    for _ in range(reps):
        p.execute_async(xd, yd)
    e.record(st)
    e.synchronize()
    return s.elapsed_time(e) / reps * 1e3


def run(name, m, variants):
    rp = torch.from_numpy(np.ascontiguousarray(m.rowptr)).cuda()
    ci = torch.from_numpy(m.colind).cuda()
    va = torch.from_numpy(m.vals).cuda()
    for opts in variants:
        p = spmv.Plan(rp, ci, va, n_cols=m.n, **opts)
        inf = p.info()
        us = time_plan(p, inf["n_rows"], m.x)
        print(f"{name:10s} nnz={m.nnz:>9d} {str(opts):60s} -> {inf['variant']:9s} vs={inf['sel']['vs']:2d} "
              f"{us:8.1f} us  {12 * m.nnz / us / 1e3:7.1f} GB/s(12B/nz)", flush=True)
        p.destroy()


def main():
    if len(sys.argv) > 1 and sys.argv[1] == "--tma":  # long_mode 2 vs 3 only
        s = sg.seeds(4)
        lr = sg.pick_rows(1000000, 100, s["pick"])
        longm = sg.randrows(1000000, 0, diag=False, long_rows=lr, k_long=200000, col_seed=s["matrix"],
                            val_seed=s["value"], x_seed=s["x"])
        run("long", longm, [dict(force_variant="split", long_mode=2), dict(force_variant="split", long_mode=3)])
        run("full", sg.config(4), [dict(force_variant="split", long_mode=2), dict(force_variant="split", long_mode=3)])
        return
    s = sg.seeds(4)
    n, nl, kl = 1000000, 100, 200000
    lr = sg.pick_rows(n, nl, s["pick"])
    full = sg.config(4)
    short = sg.randrows(n, 15, diag=False, col_seed=s["matrix"], val_seed=s["value"], x_seed=s["x"])
    longm = sg.randrows(n, 0, diag=False, long_rows=lr, k_long=kl, col_seed=s["matrix"], val_seed=s["value"],
                        x_seed=s["x"])
    run("full", full, [{}, dict(force_variant="split", long_mode=3), dict(force_variant="nnzsplit"),
                       dict(force_variant="split", split_bins=0)])
    run("short", short, [{}, dict(force_variant="nnzsplit"), dict(force_variant="nnzsplit", hot_x=0),
                         dict(force_variant="stream"), dict(force_variant="stream", seg=1),
                         dict(force_variant="vector", force_vs=16), dict(force_variant="merge")])
    run("long", longm, [{}, dict(force_variant="split", long_mode=2), dict(force_variant="split", long_mode=3),
                        dict(force_variant="split", long_mode=1),
                        dict(force_variant="nnzsplit")])


if __name__ == "__main__":
    main()
