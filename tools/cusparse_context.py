"""Vendor-library context (optional; the paper compares against
MKL CSR): cuSPARSE fp64 CSR SpMV through torch.sparse_csr_tensor
@ x on the same synthetic matrices, next to this library's auto plan. Context
only, not a target or a baseline of the bench.
  python tools/cusparse_context.py [--configs 2,3,4,5] [--out profiles/r01_cusparse.json]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1711_05487_b200 as spmv


def t_events(f, reps, stream=None):
    for _ in range(3):
        f()
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(stream)
    for _ in range(reps):
        f()
    e.record(stream)
    e.synchronize()
    return s.elapsed_time(e) / reps


ap = argparse.ArgumentParser()
ap.add_argument("--configs", default="2,3,4,5")
ap.add_argument("--reps", type=int, default=20)
ap.add_argument("--out", default=None)
a = ap.parse_args()
rows = []
for c in [int(v) for v in a.configs.split(",")]:
    blk = bench.build_block(c, 0, 1, spmv)
    n, nnz = blk["N"], blk["nnz"]
    r = {"config": c, "nnz": nnz}
    # this library
    p = spmv.Plan(blk["rowptr"], blk["colind"], blk["vals"], n_cols=n)
    xd, yd = p.x_device(), p.y_device()
    p.execute(blk["x"], np.empty(p.n_rows))
    st = torch.cuda.ExternalStream(p.stream())
    ms = t_events(lambda: p.execute_async(xd, yd), a.reps, st)
    r["ours"] = {"variant": p.info()["variant"], "ms": ms, "gflops": 2 * nnz / ms / 1e6}
    p.destroy()
    # cuSPARSE via torch: fp64 values, int32 indices where they fit (the
    # same index bytes as this library), else int64
    for idt, name in ((np.int32, "cusparse_i32"), (np.int64, "cusparse_i64")):
        try:
            rp = blk["rowptr"].astype(np.int64)
            if idt == np.int32 and rp[-1] >= 2 ** 31:
                continue
            A = torch.sparse_csr_tensor(torch.from_numpy(rp.astype(idt)).cuda(),
                                        torch.from_numpy(blk["colind"].astype(idt)).cuda(),
                                        torch.from_numpy(blk["vals"]).cuda(), size=(n, n))
            x = torch.from_numpy(blk["x"]).cuda()
            ms2 = t_events(lambda: A @ x, a.reps)
            r[name] = {"ms": ms2, "gflops": 2 * nnz / ms2 / 1e6, "speedup_of_ours": ms2 / ms}
            del A, x
        except Exception as ex:  # noqa: BLE001
            r[name] = {"error": str(ex)[:200]}
        torch.cuda.empty_cache()
    torch.cuda.empty_cache()
    rows.append(r)
    print(json.dumps(r), flush=True)
if a.out:
    json.dump(rows, open(a.out, "w"), indent=1)
