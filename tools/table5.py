"""Table V analogue: per config, the feature-guided and the
profile-guided optimizer vs the CSR baseline (csr_vector): the chosen variant,
its SpMV time, the optimizer overhead t_pre (inspector + selection incl. the
profile micro-benchmarks + format conversion; upload excluded as the
baseline needs it too) and N_iters,min = t_pre / (t_base - t_opt)
(P:932-950).
  python tools/table5.py [--configs 2,3,4,5] [--out profiles/r01_table5.json]"""
import argparse, json, math, os, sys, time
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1711_05487_b200 as spmv


def time_plan(p, n_rows, x, reps):
    xd, yd = p.x_device(), p.y_device()
    p.execute(x, np.empty(n_rows))
    st = torch.cuda.ExternalStream(p.stream())
    for _ in range(3):
        p.execute_async(xd, yd)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    for _ in range(reps):
        p.execute_async(xd, yd)
    e.record(st)
    e.synchronize()
    return s.elapsed_time(e) / reps * 1e-3


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--configs", default="1,2,3,4,5")
    ap.add_argument("--reps", type=int, default=20)
    ap.add_argument("--out", default=None)
    a = ap.parse_args()
    rows = []
    for c in [int(v) for v in a.configs.split(",")]:
        blk = bench.build_block(c, 0, 1, spmv)
        rp = torch.from_numpy(blk["rowptr"]).cuda()
        ci = torch.from_numpy(blk["colind"]).cuda()
        va = torch.from_numpy(blk["vals"]).cuda()
        N = blk["N"]
        res = {"config": c}
        for name, opts in (("baseline", dict(force_variant="vector")), ("feature", {}), ("profile", dict(select_mode=1))):
            # a first plan of the same kind loads its kernels (lazy module
            # loading is a per-process cost, not the optimizer's t_pre)
            spmv.Plan(rp, ci, va, n_cols=N, **opts).destroy()
            t0 = time.time()
            p = spmv.Plan(rp, ci, va, n_cols=N, **opts)
            wall = time.time() - t0
            info = p.info()
            t = time_plan(p, info["n_rows"], blk["x"], a.reps)
            r = {"variant": info["variant"], "classes": info["classes"], "ms": t * 1e3,
                 "t_pre_ms": info["inspect_ms"] + info["select_ms"] + info["encode_ms"],
                 "select_ms": info["select_ms"], "plan_wall_ms": wall * 1e3}
            if name == "profile":
                r["bounds_gflops"] = {k: info[k] / 1e9 for k in ("p_csr", "p_mb", "p_ml", "p_imb", "p_cmp", "p_peak")}
                r["bmax_gbs"] = info["bmax"] / 1e9
                r["profile_ms"] = info["profile_ms"]
            res[name] = r
            p.destroy()
        tb = res["baseline"]["ms"]
        for name in ("feature", "profile"):
            d = (tb - res[name]["ms"]) * 1e-3
            res[name]["speedup_vs_baseline"] = tb / res[name]["ms"]
            res[name]["n_iters_min"] = (res[name]["t_pre_ms"] * 1e-3 / d) if d > 0 else math.inf
        rows.append(res)
        print(json.dumps(res), flush=True)
    if a.out:
        json.dump(rows, open(a.out, "w"), indent=1)


if __name__ == "__main__":
    main()
