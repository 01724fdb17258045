#!/usr/bin/env python
"""Forced-variant sweep on one config: time every variant / VS / tile / D16 /
D8 choice, report GB/s and the selection regret (feature-guided pick vs the
exhaustive best, the paper's "oracle" optimizer P:805-807 and the trivial
optimizer cost P:921-926) and N_iters,min.

  python tools/sweep.py --config 2 [--reps 50]
"""
import argparse
import itertools
import json
import os
import sys
import time

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", type=int, default=2)
    ap.add_argument("--reps", type=int, default=30)
    ap.add_argument("--quick", action="store_true")
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    import torch
    import paper_1711_05487_b200 as spmv
    import synthgen as sg
    import bench

    blk = bench.build_block(a.config, 0, 1, spmv)
    rp = torch.from_numpy(blk["rowptr"]).cuda()
    ci = torch.from_numpy(blk["colind"]).cuda()
    va = torch.from_numpy(blk["vals"]).cuda()
    N, nnz = blk["N"], blk["nnz"]
    byts = bench.algo_bytes(N, N, nnz, blk["rp_bytes"])

    def run(**opts):
        t0 = time.time()
        p = spmv.Plan(rp, ci, va, n_cols=N, **opts)
        t_plan = time.time() - t0
        info = p.info()
        xd, yd = p.x_device(), p.y_device()
        p.execute(blk["x"], np.empty(info["n_rows"]))
        st = torch.cuda.ExternalStream(p.stream())
        for _ in range(3):
            p.execute_async(xd, yd)
        torch.cuda.synchronize()
        rates = []
        for _ in range(3):  # paper methodology: runs of back-to-back SpMVs, harmonic mean
            s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            s.record(st)
            for _ in range(a.reps):
                p.execute_async(xd, yd)
            e.record(st)
            e.synchronize()
            rates.append(a.reps / (s.elapsed_time(e) * 1e-3))
        hm = len(rates) / sum(1 / r for r in rates)
        ms = 1e3 / hm
        r = {"opts": opts, "variant": info["variant"], "vs": info["sel"]["vs"], "d16": info["sel"]["d16"],
             "tile": info["tile_nnz"], "ms": ms, "gbs": byts / (ms * 1e-3) / 1e9, "gflops": 2 * nnz / (ms * 1e-3) / 1e9,
             "plan_ms": {k: info[k] for k in ("upload_ms", "inspect_ms", "select_ms", "encode_ms")},
             "plan_wall_ms": t_plan * 1e3}
        p.destroy()
        return r

    res = [run()]
    auto = res[0]
    print(json.dumps({"auto": auto}), flush=True)
    grid = []
    vss = (1, 2, 4, 8, 16, 32) if not a.quick else (4, 8, 32)  # VS=32 = warp-per-row baseline
    for vs in vss:
        grid.append(dict(force_variant="vector", force_vs=vs))
    svs = (1, 2, 4) if not a.quick else (1, 4)
    tiles = (256, 384, 512, 640, 768, 1024) if not a.quick else (512, 640, 768)
    stages = (4, 8) if not a.quick else (4,)
    d16s = (0, 1) if a.config in (1, 2) else (0,)
    # the plan's own tile rule (row-count tiles on regular rows, 4/6 consumer warps)
    grid.append(dict(force_variant="stream", force_vs=1, d16=0))
    grid.append(dict(force_variant="stream", force_vs=1, d16=1))
    # dictionary-coded 8-bit deltas (D8; the kernel picks 4/6/8 consumer warps)
    grid.append(dict(force_variant="stream", d16=2))
    for vs, t, sg_, d in itertools.product(svs, tiles, stages, d16s):
        grid.append(dict(force_variant="stream", force_vs=vs, tile_nnz=t, stages=sg_, d16=d))
    for t in tiles:
        grid.append(dict(force_variant="stream", seg=1, tile_nnz=t))
    grid.append(dict(force_variant="merge"))
    grid.append(dict(force_variant="nnzsplit"))
    grid.append(dict(force_variant="nnzsplit", hot_x=0))
    grid.append(dict(force_variant="nnzsplit", hot_x=16384))
    for sg_ in (0, 1):
        for t in tiles:
            grid.append(dict(force_variant="split", seg=sg_, tile_nnz=t))
    for g in grid:
        try:
            r = run(**g)
        except Exception as ex:  # a forced choice may not fit (e.g. smem)
            r = {"opts": g, "error": str(ex)}
        res.append(r)
        print(json.dumps(r), flush=True)
    ok = [r for r in res[1:] if "ms" in r]
    best = min(ok, key=lambda r: r["ms"])
    base = [r for r in ok if r["variant"] == "vector" and r["vs"] == 32][0]
    t_pre = (auto["plan_ms"]["inspect_ms"] + auto["plan_ms"]["select_ms"] + auto["plan_ms"]["encode_ms"]) * 1e-3
    d = base["ms"] - auto["ms"]
    summary = {"config": a.config, "auto": {k: auto[k] for k in ("variant", "vs", "d16", "tile", "ms", "gbs")},
               "best": {k: best[k] for k in ("opts", "ms", "gbs")}, "regret": auto["ms"] / best["ms"] - 1,
               "baseline_warp_per_row_ms": base["ms"],
               "n_iters_min": (t_pre / (d * 1e-3)) if d > 0 else None,
               "trivial_optimizer_s": sum(r.get("plan_wall_ms", 0) for r in ok) * 1e-3}
    print(json.dumps({"summary": summary}), flush=True)
    if a.out:
        json.dump({"results": res, "summary": summary}, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
