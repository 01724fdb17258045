"""Build C4's long rows alone (100 rows x 200,000 columns) with given plan
options and run a few SpMVs (for ncu)."""
import json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synthgen as sg
import paper_1711_05487_b200 as spmv
opts = json.loads(sys.argv[1]) if len(sys.argv) > 1 else {}
s = sg.seeds(4)
m = sg.randrows(1000000, 0, diag=False, long_rows=sg.pick_rows(1000000, 100, s["pick"]), k_long=200000,
                col_seed=s["matrix"], val_seed=s["value"], x_seed=s["x"])
p = spmv.Plan(torch.from_numpy(m.rowptr).cuda(), torch.from_numpy(m.colind).cuda(), torch.from_numpy(m.vals).cuda(),
              n_cols=m.n, **opts)
xd = torch.from_numpy(m.x).cuda()
yd = torch.empty(m.n, dtype=torch.float64, device="cuda")
for _ in range(3):
    p.execute(xd, yd)
torch.cuda.synchronize()
print(p.info()["long_mode"], p.info()["long_rg"])
