"""bench.py's per-rank row blocks (one process per GPU): every
rank generates only its nnz-balanced block; the blocks concatenate to the
whole config matrix (CPU, no GPU needed)."""
import numpy as np
import pytest

import bench
import oracle
import synthgen as sg

spmv = pytest.importorskip("paper_1711_05487_b200")


@pytest.mark.parametrize("cfg,world", [(2, 2), (2, 3), (4, 3)])
def test_rank_blocks_concatenate_to_the_config(cfg, world):
    m = sg.config(cfg)
    rp = m.rowptr.astype(np.int64)
    assert np.array_equal(bench.build_block(cfg, 0, world, spmv)["bounds"], oracle.shard_bounds(rp, world))
    cols, vals, lens = [], [], []
    for r in range(world):
        b = bench.build_block(cfg, r, world, spmv)
        brp = b["rowptr"].astype(np.int64)
        assert brp[0] == 0 and brp[-1] == b["colind"].size == b["vals"].size
        assert b["nnz"] == m.nnz and b["N"] == m.n
        assert np.array_equal(b["x"], m.x)
        cols.append(b["colind"])
        vals.append(b["vals"])
        lens.append(np.diff(brp))
    assert np.array_equal(np.concatenate(lens), np.diff(rp))
    assert np.array_equal(np.concatenate(cols), m.colind)
    assert np.array_equal(np.concatenate(vals), m.vals)
