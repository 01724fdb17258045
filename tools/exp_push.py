"""Experiment log (tools only): the multi-shard iterated mode with the halo
exchange fused into the SpMV kernels (halo push) vs the halo copies
(SPMV_NO_PUSH=1), emulated shards on ONE GPU: the shards' kernels serialise
on the one device, so this shows the launches and copies the push removes
from every iteration, not NVLink overlap.
  python tools/exp_push.py [--n 256] [--iters 40]"""
import argparse, os, subprocess, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))

if len(sys.argv) > 1 and sys.argv[1] == "--one":
    import numpy as np
    import torch
    import synthgen as sg
    import paper_1711_05487_b200 as spmv
    n, G, iters, d16 = (int(v) for v in sys.argv[2:6])
    m = sg.stencil(n, 27, x_seed=3)
    p = spmv.Plan(m.rowptr, m.colind, m.vals, ngpus=G, emulate_devices=1, force_variant="stream", d16=d16)
    p.iterate(m.x, 3)
    best = 1e30
    for _ in range(3):
        torch.cuda.synchronize()
        t = time.perf_counter()
        x, nu = p.iterate(m.x, iters)
        torch.cuda.synchronize()
        best = min(best, time.perf_counter() - t)
    inf = p.info()
    print(f"27-pt {n}^3 G={G} d16={d16} push={inf['iter_push']}: {best / iters * 1e3:.3f} ms/iteration "
          f"(host wall, best of 3 x {iters}; includes x0 upload and the final unit)", flush=True)
    sys.exit(0)
ap = argparse.ArgumentParser()
ap.add_argument("--n", type=int, default=256)
ap.add_argument("--iters", type=int, default=40)
a = ap.parse_args()
for G in (2, 4, 8):
    for d16 in (2, 0):
        for env in ({}, {"SPMV_NO_PUSH": "1"}):
            subprocess.run([sys.executable, __file__, "--one", str(a.n), str(G), str(a.iters), str(d16)],
                           env={**os.environ, **env}, check=True)
