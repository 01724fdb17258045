import sys, os; sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np, bench, paper_1711_05487_b200 as spmv
for c in (2, 3, 4):
    blk = bench.build_block(c, 0, 1, spmv)
    print({k: (type(v).__name__, getattr(v, "dtype", None), getattr(v, "device", None)) for k, v in blk.items() if k in ("rowptr", "colind", "vals", "x")})
    for v in (None, "nnzsplit"):
        kw = {} if v is None else {"force_variant": v}
        try:
            p = spmv.Plan(blk["rowptr"], blk["colind"], blk["vals"], n_cols=blk["N"], **kw)
        except TypeError as e:
            print("kw", e); continue
        i = p.info(); print(c, v, i["variant"], round(i["x_reuse"], 3), i["nz_gather_l2"], flush=True)
        del p
