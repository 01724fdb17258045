"""Build one plan with the given options and run a few SpMVs (for ncu)."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1711_05487_b200 as spmv

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=3)
ap.add_argument("--opts", default="{}")
ap.add_argument("--reps", type=int, default=3)
a = ap.parse_args()
blk = bench.build_block(a.config, 0, 1, spmv)
p = spmv.Plan(blk["rowptr"], blk["colind"], blk["vals"], n_cols=blk["N"], **json.loads(a.opts))
# device buffers: every launch is a whole SpMV (a host x/y would take the
# pipelined tile-range path and ncu would capture one block)
xd = torch.from_numpy(blk["x"]).cuda()
yd = torch.empty(p.n_rows, dtype=torch.float64, device="cuda")
for _ in range(a.reps):
    p.execute(xd, yd)
print(json.dumps({k: v for k, v in p.info().items() if k in ("variant", "sel", "tile_nnz", "n_tiles")}))
