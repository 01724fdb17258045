"""CUPTI timeline of one end-to-end SpMV through the host pipeline (pinned
host x in, host y out; api.cu host_pipe_*): H2D chunks, tile-range kernels,
D2H blocks.  python tools/timeline_e2e.py [--config 5]"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1711_05487_b200 as spmv

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
a = ap.parse_args()
blk = bench.build_block(a.config, 0, 1, spmv)
p = spmv.Plan(blk["rowptr"], blk["colind"], blk["vals"], n_cols=blk["N"])
xh = torch.from_numpy(blk["x"]).pin_memory()
yh = torch.empty(p.n_rows, dtype=torch.float64).pin_memory()
for _ in range(3):
    p.execute(xh, yh)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    p.execute(xh, yh)
    torch.cuda.synchronize()
evs = sorted((e.time_range.start, e.time_range.end, e.name[:50]) for e in prof.events()
             if e.device_type == torch.autograd.DeviceType.CUDA)
t0 = evs[0][0]
for s, t, n in evs:
    print(f"{s - t0:9.1f} {t - t0:9.1f} {t - s:8.1f}  {n}")
print("total_us", evs[-1][1] - t0)
