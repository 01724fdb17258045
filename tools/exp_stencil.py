"""Experiment: time cta_stream on a pts-point stencil n^3 with forced options
(e.g. D16 on a 27-pt grid small enough for 16-bit deltas).
  python tools/exp_stencil.py --n 180 --pts 27 --opts '[{"d16":0},{"d16":1}]'"""
import argparse, json, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import paper_1711_05487_b200 as spmv
import synthgen as sg
import bench

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=180)
ap.add_argument("--pts", type=int, default=27)
ap.add_argument("--rp64", type=int, default=1)
ap.add_argument("--opts", default='[{}]')
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
m = sg.stencil(a.n, a.pts, rp64=bool(a.rp64), x_seed=5)
N, nnz = m.n, int(m.rowptr[-1])
byts = bench.algo_bytes(N, N, nnz, 8 if a.rp64 else 4)
for o in json.loads(a.opts):
    p = spmv.Plan(m.rowptr, m.colind, m.vals, **o)
    info = p.info()
    xd, yd = p.x_device(), p.y_device()
    p.execute(m.x, np.empty(N))
    st = torch.cuda.ExternalStream(p.stream())
    for _ in range(3):
        p.execute_async(xd, yd)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    for _ in range(a.reps):
        p.execute_async(xd, yd)
    e.record(st)
    e.synchronize()
    ms = s.elapsed_time(e) / a.reps
    print(json.dumps({"n": a.n, "pts": a.pts, "opts": o, "variant": info["variant"], "d16": info["sel"]["d16"],
                      "tile": info["tile_nnz"], "ms": ms, "pct_8tbs": 100 * byts / (ms * 1e-3) / 8e12}), flush=True)
    p.destroy()
