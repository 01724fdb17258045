"""Where does the cold-L2 penalty of a small STREAM / D8 SpMV come from?

Times one SpMV after each of: nothing (back-to-back, warm), a 252-MB clean
read flush (cold, as bench.py), the flush followed by a read of x (x back in
L2, streams cold), and the flush followed by a read of x and y."""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1711_05487_b200 as spmv

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--opts", default="{}")
ap.add_argument("--reps", type=int, default=20)
a = ap.parse_args()
blk = bench.build_block(a.config, 0, 1, spmv)
p = spmv.Plan(blk["rowptr"], blk["colind"], blk["vals"], n_cols=blk["N"], **json.loads(a.opts))
st = torch.cuda.ExternalStream(p.stream())
xd = torch.from_numpy(blk["x"]).cuda()
yd = torch.empty(p.n_rows, dtype=torch.float64, device="cuda")
flush = torch.ones(2 * 126 * 2 ** 20 // 4, dtype=torch.float32, device="cuda")
sink = torch.empty((), dtype=torch.float32, device="cuda")
sx = torch.empty((), dtype=torch.float64, device="cuda")
torch.cuda.synchronize()


def run(pre):
    ts = []
    for _ in range(a.reps):
        with torch.cuda.stream(st):
            pre()
        s0, e0 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        s0.record(st)
        p.execute_async(xd, yd)
        e0.record(st)
        e0.synchronize()
        ts.append(s0.elapsed_time(e0) * 1e3)
    return float(np.median(ts))


def nothing():
    pass


def fl():
    torch.sum(flush, dim=0, out=sink)


def fl_x():
    fl()
    torch.sum(xd, dim=0, out=sx)


def fl_xy():
    fl_x()
    torch.sum(yd, dim=0, out=sx)


def sl_fl():
    torch.cuda._sleep(200_000)
    fl()


def sl():
    torch.cuda._sleep(200_000)


def fl_small():
    torch.sum(flush[: 64 * 2 ** 20 // 4], dim=0, out=sink)


for _ in range(3):
    p.execute_async(xd, yd)
res = {"info": {k: v for k, v in p.info().items() if k in ("variant", "sel", "tile_nnz", "n_tiles")}}
for name, f in (("warm", nothing), ("cold", fl), ("cold_x_in_l2", fl_x), ("cold_xy_in_l2", fl_xy),
                ("flush64MB", fl_small), ("sleep_warm", sl), ("sleep_cold", sl_fl), ("warm2", nothing)):
    res[name + "_us"] = run(f)
print(json.dumps(res))
