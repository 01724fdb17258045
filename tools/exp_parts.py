"""Time the parts of a config separately: the whole matrix, its short rows
alone (long rows emptied) and its long rows alone (short rows emptied), each
with the auto plan and the given forced variants (experiment tool).
  python tools/exp_parts.py --config 4 [--lsplit 4096] [--variants split,nnzsplit]"""
import argparse, json, os, sys
sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np
import torch
import bench
import paper_1711_05487_b200 as spmv

ap = argparse.ArgumentParser()
ap.add_argument("--config", type=int, default=4)
ap.add_argument("--lsplit", type=int, default=4096)
ap.add_argument("--variants", default="auto,nnzsplit")
ap.add_argument("--reps", type=int, default=50)
ap.add_argument("--parts", default="all,short,long")
a = ap.parse_args()
blk = bench.build_block(a.config, 0, 1, spmv)
rp = blk["rowptr"].astype(np.int64)
ln = np.diff(rp)


def sub(keep):
    """CSR with only the rows in `keep` (others empty)."""
    kl = np.where(keep, ln, 0)
    nrp = np.zeros(rp.size, np.int64)
    nrp[1:] = np.cumsum(kl)
    sel = np.repeat(keep, ln)
    return nrp.astype(blk["rowptr"].dtype), blk["colind"][sel], blk["vals"][sel]


def timeit(rpx, col, val, **opts):
    p = spmv.Plan(rpx, col, val, n_cols=blk["N"], **opts)
    xd, yd = p.x_device(), p.y_device()
    p.execute(blk["x"], np.empty(p.n_rows))
    st = torch.cuda.ExternalStream(p.stream())
    for _ in range(5):
        p.execute_async(xd, yd)
    torch.cuda.synchronize()
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(st)
    for _ in range(a.reps):
        p.execute_async(xd, yd)
    e.record(st)
    e.synchronize()
    ms = s.elapsed_time(e) / a.reps
    v = p.info()["variant"]
    p.destroy()
    return ms, v


parts = {"all": (blk["rowptr"], blk["colind"], blk["vals"]),
         "short": sub(ln <= a.lsplit), "long": sub(ln > a.lsplit)}
for name, (r, c, v) in parts.items():
    if name not in a.parts.split(","):
        continue
    nnz = int(np.asarray(r, np.int64)[-1])
    for var in a.variants.split(","):
        opts = {} if var == "auto" else {"force_variant": var}
        try:
            ms, vv = timeit(r, c, v, **opts)
            print(json.dumps({"part": name, "nnz": nnz, "req": var, "variant": vv, "us": round(ms * 1e3, 1),
                              "gbs": round((12 * nnz + 4 * rp.size + 16 * blk["N"]) / ms / 1e6, 1)}), flush=True)
        except Exception as ex:  # noqa: BLE001
            print(json.dumps({"part": name, "req": var, "error": str(ex)[:200]}), flush=True)
