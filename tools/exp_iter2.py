"""C2/C5 iterated-mode overhead (experiment tool): device time per iteration of
spmv_iterate (the library's own loop) vs back-to-back ping-pong SpMVs, over
many iterations in one call.  python tools/exp_iter2.py --config 2 --iters 1000"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1711_05487_b200 as spmv

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=2)
ap.add_argument("--iters", type=int, default=1000)
a = ap.parse_args()
blk = bench.build_block(a.config, 0, 1, spmv)
p = spmv.Plan(blk["rowptr"], blk["colind"], blk["vals"], n_cols=blk["N"])
st = torch.cuda.ExternalStream(p.stream())
xa = torch.from_numpy(blk["x"]).cuda()
xb = xa.clone()
x0 = xa.clone()
bufs = (xa, xb)


def t_ev(f):
    f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    f()
    e.record(st)
    e.synchronize()
    return s.elapsed_time(e) * 1e3


def pingpong():
    xa.copy_(x0)
    for k in range(a.iters):
        p.execute_async(bufs[k & 1], bufs[(k + 1) & 1])


x0 = xa.clone()


def native():
    xa.copy_(x0)  # (the ping-pong run left overflowed values behind)
    try:
        p.iterate(xa, a.iters, x_out=xb)
    except spmv.SpmvError as e:  # timing-experiment builds may not produce nu
        print("note:", e)


with torch.cuda.stream(st):
    tp = t_ev(pingpong) / a.iters
    tn = t_ev(native) / a.iters
print({"config": a.config, "env": {k: v for k, v in os.environ.items() if k.startswith("SPMV_")},
       "pingpong_us": round(tp, 2), "iterate_us": round(tn, 2), "overhead_pct": round(100 * (tn / tp - 1), 2)})
