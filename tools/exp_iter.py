"""Where the iterated mode's time goes (experiment tool): per-iteration device
time of (a) the plain SpMV on the plan buffers, (b) the SpMV ping-ponging two
replicas, (c) the iteration step + a separate norm-step kernel, (d) the fused step
(norm step in the SpMV epilogue), (e) the full
parallel.iterate (world 1).  python tools/exp_iter.py --config 5 --iters 50"""
import argparse, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import torch
import bench
import paper_1711_05487_b200 as spmv
from paper_1711_05487_b200 import parallel

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=5)
ap.add_argument("--iters", type=int, default=50)
a = ap.parse_args()
blk = bench.build_block(a.config, 0, 1, spmv)
p = spmv.Plan(blk["rowptr"], blk["colind"], blk["vals"], n_cols=blk["N"])
n = blk["N"]
st = torch.cuda.ExternalStream(p.stream())
P = spmv.norm_partial_count()
with torch.cuda.stream(st):
    xa = torch.from_numpy(blk["x"]).cuda()
    xb = xa.clone()
    pl = torch.empty(P, dtype=torch.float64, device="cuda")
    nn = torch.zeros(2, dtype=torch.float64, device="cuda")
    nu = torch.empty(a.iters + 2, dtype=torch.float64, device="cuda")
torch.cuda.synchronize()
xd, yd = p.x_device(), p.y_device()
p.execute(blk["x"], torch.empty(n, dtype=torch.float64).numpy())


def timed(f):
    for _ in range(2):
        f(0)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    for k in range(a.iters):
        f(k)
    e.record(st)
    e.synchronize()
    return s.elapsed_time(e) / a.iters * 1e3


bufs = (xa, xb)
x0 = xa.clone()


def reset():
    xa.copy_(x0)
    xb.copy_(x0)
    nn.zero_()
    torch.cuda.synchronize()


res = {"a_plain": timed(lambda k: p.execute_async(xd, yd))}
reset()
res["b_pingpong"] = timed(lambda k: p.execute_async(bufs[k & 1], bufs[(k + 1) & 1]))
reset()
res["c_step_then_norm"] = timed(lambda k: (p.iter_step(bufs[k & 1], bufs[(k + 1) & 1], pl, nn),
                                           p.norm_step(pl, P, nn, nu[k:k + 1])))
reset()
res["d_fused_step"] = timed(lambda k: p.iter_step(bufs[k & 1], bufs[(k + 1) & 1], pl, nn, nu[k:k + 1]))
reset()
res["f_step_no_norm"] = timed(lambda k: p.iter_step(bufs[k & 1], bufs[(k + 1) & 1], pl, nn))
reset()
res["g_execute_norm"] = timed(lambda k: p.execute_norm(bufs[k & 1], bufs[(k + 1) & 1], pl))
reset()
steps = parallel.native_steps(p)
pa = pl
b = [0, n]
with torch.cuda.stream(st):
    parallel.iterate(parallel.NoDist, steps, b, 0, 1, xa, xb, pl, pa, nu, nn, 2)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    parallel.iterate(parallel.NoDist, steps, b, 0, 1, xa, xb, pl, pa, nu, nn, a.iters)
    e.record(st)
    e.synchronize()
    res["e_parallel_iterate"] = s.elapsed_time(e) / a.iters * 1e3
print({k: round(v, 1) for k, v in res.items()}, "us per iteration")
