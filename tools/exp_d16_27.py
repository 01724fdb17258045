"""D16 vs plain stream on a 27-point 180^3 stencil (16-bit gaps: D16-eligible;
DESIGN.md reading 9). Experiment tool: python tools/exp_d16_27.py"""
import sys, os, json
sys.path.insert(0, "/root/repo")
import numpy as np, torch
import paper_1711_05487_b200 as spmv, synthgen as sg
m = sg.stencil(180, 27, x_seed=5)
for opts in ({}, {"d16": 0}):
    p = spmv.Plan(m.rowptr, m.colind, m.vals, **opts)
    xd, yd = p.x_device(), p.y_device()
    p.execute(m.x, np.empty(m.n))
    st = torch.cuda.ExternalStream(p.stream())
    for _ in range(5): p.execute_async(xd, yd)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    for _ in range(50): p.execute_async(xd, yd)
    e.record(st); e.synchronize()
    i = p.info()
    print(json.dumps({"opts": opts, "us": s.elapsed_time(e) / 50 * 1e3, "d16": i["sel"]["d16"], "rows_per_tile": i["rows_per_tile"], "tile": i["tile_nnz"], "row_tiles_env": os.environ.get("SPMV_ROW_TILES")}))
    p.destroy()
