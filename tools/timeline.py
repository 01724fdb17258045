"""Kernel timeline of a few SpMVs via torch.profiler (CUPTI): start/end of
every kernel (ours included) on every stream -- the concurrency check nsys
would give. python tools/timeline.py --config 4 [--opts '{...}'] [--stage 0]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1711_05487_b200 as spmv

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--opts", default="{}")
ap.add_argument("--stage", type=int, default=0)
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
blk = bench.build_block(a.config, 0, 1, spmv)
p = spmv.Plan(blk["rowptr"], blk["colind"], blk["vals"], n_cols=blk["N"], **json.loads(a.opts))
xd, yd = p.x_device(), p.y_device()
p.execute(blk["x"], np.empty(p.n_rows))
for _ in range(5):
    p.execute_stage(xd, yd, a.stage)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    for _ in range(a.reps):
        p.execute_stage(xd, yd, a.stage)
    torch.cuda.synchronize()
evs = [e for e in prof.events() if e.device_type == torch.autograd.DeviceType.CUDA]
rows = []
for e in evs:
    rows.append((e.time_range.start, e.time_range.end, e.name))
rows.sort()
t0 = rows[0][0] if rows else 0
for s, e, n in rows:
    print(f"{s - t0:10.1f} {e - t0:10.1f} {e - s:8.1f}  {n[:80]}")
