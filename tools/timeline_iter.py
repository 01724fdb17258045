"""Timeline of the multi-shard iterated mode (emulated shards on one GPU), via
torch.profiler (CUPTI) -- SURVEY 8(f) f2: by default the halo push (one
kernel per shard and iteration, storing its halo rows into the neighbours'
replicas); with --no-push the interior-tile kernels, halo copies and
boundary-tile kernels per stream.
  python tools/timeline_iter.py [--n 160] [--G 4] [--iters 3] [--no-push]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import synthgen as sg
import paper_1711_05487_b200 as spmv

ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=160)
ap.add_argument("--G", type=int, default=4)
ap.add_argument("--iters", type=int, default=3)
ap.add_argument("--out", default="")
ap.add_argument("--no-push", action="store_true", help="halo copies + interior-first tiles instead of the halo push")
a = ap.parse_args()
if a.no_push:
    os.environ["SPMV_NO_PUSH"] = "1"  # read when the plan first iterates
m = sg.stencil(a.n, 27, x_seed=3)
p = spmv.Plan(m.rowptr, m.colind, m.vals, ngpus=a.G, emulate_devices=1)
p.iterate(m.x, 2)  # warm-up (plans the interior ranges)
torch.cuda.synchronize()
from torch.profiler import profile, ProfilerActivity
with profile(activities=[ProfilerActivity.CUDA]) as prof:
    p.iterate(m.x, a.iters)
    torch.cuda.synchronize()
evs = []
for e in prof.events():
    if e.device_type != torch.autograd.DeviceType.CUDA:
        continue
    name = e.name
    kind = "copy" if "Memcpy" in name or "memcpy" in name else ("set" if "Memset" in name else "kernel")
    evs.append((e.time_range.start, e.time_range.end, kind, name[:60]))
evs.sort()
t0 = evs[0][0] if evs else 0
rows = [{"start_us": round(s - t0, 1), "end_us": round(t - t0, 1), "kind": k, "name": n} for s, t, k, n in evs]
for r in rows:
    print(f"{r['start_us']:10.1f} {r['end_us']:10.1f}  {r['kind']:6s} {r['name']}")
# overlap: copy time covered by a concurrently running kernel
cov = tot = 0.0
ks = [(r["start_us"], r["end_us"]) for r in rows if r["kind"] == "kernel"]
for r in rows:
    if r["kind"] != "copy":
        continue
    tot += r["end_us"] - r["start_us"]
    for s, t in ks:
        cov += max(0.0, min(t, r["end_us"]) - max(s, r["start_us"]))
print(json.dumps({"n": a.n, "G": a.G, "iters": a.iters, "copy_us": round(tot, 1),
                  "copy_us_overlapped_by_kernels": round(cov, 1)}))
if a.out:
    json.dump(rows, open(a.out, "w"))
