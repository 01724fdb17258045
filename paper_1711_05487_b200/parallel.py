"""Row-sharded multi-GPU driver, one process per GPU.

Rank g owns rows [b_g, b_{g+1}) of A (the nnz-balanced lower_bound rule,
P:708-711, computed by ``spmv_shard_bounds``) and a full replica of x.

* single SpMV: no collective; every rank writes its y block.
* iterated mode (BJ.configs[5]): per iteration
    1. y_g = A_g x                      (libspmv kernel, plan stream)
    2. partials_g = fixed-chunk sums of y_g^2   (libspmv kernel)
    3. all-gather of the partials (rank order)    -- NCCL
    4. nu = sqrt(sum of all partials in rank order) on every rank (identical),
       x[b_g:b_{g+1}] = y_g / nu                  (libspmv kernel)
    5. the x exchange  -- NCCL
       * all-gather(v): one broadcast per rank into its slice of every
         replica (blocks differ in size), or
       * halo exchange: rank g's rows only read x columns
         [col_min_g, col_max_g] (the plan's features), so rank h sends rank
         g just the part of its block inside that range (point-to-point);
         for banded matrices a few planes instead of the whole vector
         (27-pt 384^3 at G = 8: ~2.4 MB per rank per iteration vs 396 MB).

This module only orchestrates (argument marshalling, process-group calls);
every arithmetic step runs in the native library. The step functions are
injectable so the orchestration is tested with the ``gloo`` backend on CPU.
"""
from __future__ import annotations

from dataclasses import dataclass
from typing import Callable, Sequence


@dataclass
class ShardSteps:
    """Per-rank local steps. Tensors are 1-D float64 on the rank's device."""
    spmv: Callable[[object, object], None]            # (x_full, y_local)
    partials: Callable[[object, object], None]        # (y_local, partials_local[P])
    normalize: Callable[[object, object, int, object, object], None]  # (y, partials_all, count, x_block, nu[1])


def halo_plan(bounds: Sequence[int], needs: Sequence[Sequence[int]], rank: int):
    """Point-to-point x exchange of rank `rank` (pure function).

    bounds: b_0..b_G (rows owned); needs[g] = (lo, hi): rank g reads x[lo:hi)
    (hi = col_max + 1; (0, 0) when it reads nothing). Returns (sends, recvs):
    lists of (peer, lo, hi) -- rank h sends rank g x[max(lo_g, b_h) :
    min(hi_g, b_{h+1})) when non-empty; a rank never sends to itself."""
    G = len(bounds) - 1
    b0, b1 = int(bounds[rank]), int(bounds[rank + 1])
    sends, recvs = [], []
    for g in range(G):
        if g == rank:
            continue
        lo, hi = int(needs[g][0]), int(needs[g][1])
        s_lo, s_hi = max(lo, b0), min(hi, b1)  # my block inside g's range
        if s_lo < s_hi:
            sends.append((g, s_lo, s_hi))
        mlo, mhi = int(needs[rank][0]), int(needs[rank][1])
        r_lo, r_hi = max(mlo, int(bounds[g])), min(mhi, int(bounds[g + 1]))  # g's block inside my range
        if r_lo < r_hi:
            recvs.append((g, r_lo, r_hi))
    return sends, recvs


def halo_bytes(bounds: Sequence[int], needs: Sequence[Sequence[int]], rank: int) -> int:
    """fp64 bytes rank `rank` receives per iteration in the halo exchange."""
    return 8 * sum(hi - lo for _, lo, hi in halo_plan(bounds, needs, rank)[1])


def exchange_x(dist, bounds, rank, world, x_full, halo=None, group=None):
    """One x exchange: the halo plan (sends, recvs) when given, else the
    all-gather(v) of the blocks."""
    if world == 1:
        return
    if halo is not None:
        sends, recvs = halo
        ops = [dist.isend(x_full[lo:hi], dst=g, group=group) for g, lo, hi in sends]
        ops += [dist.irecv(x_full[lo:hi], src=g, group=group) for g, lo, hi in recvs]
        for w in ops:
            w.wait()
        return
    works = [dist.broadcast(x_full[int(bounds[g]):int(bounds[g + 1])], src=g, group=group, async_op=True)
             for g in range(world) if bounds[g + 1] > bounds[g]]
    for w in works:
        w.wait()


def iterate(dist, steps: ShardSteps, bounds: Sequence[int], rank: int, world: int, x_full, y_local,
            partials_local, partials_all, nu_hist, iters: int, group=None, halo=None):
    """Run `iters` power iterations in place on x_full (the replica).

    partials_all: tensor of world * P; nu_hist: tensor of >= iters (nu_k);
    halo: this rank's halo_plan(...) to exchange only the x ranges the ranks
    read (else the full all-gather). Returns nothing; x_full holds x_iters on
    every rank (with a halo plan: at least the range this rank reads).
    """
    P = partials_local.numel()
    b0, b1 = int(bounds[rank]), int(bounds[rank + 1])
    for k in range(iters):
        steps.spmv(x_full, y_local)
        steps.partials(y_local, partials_local)
        dist.all_gather_into_tensor(partials_all, partials_local, group=group)
        steps.normalize(y_local, partials_all, world * P, x_full[b0:b1], nu_hist[k:k + 1])
        exchange_x(dist, bounds, rank, world, x_full, halo, group)


def exchange_only(dist, bounds: Sequence[int], rank: int, world: int, x_full, partials_local, partials_all,
                  group=None, halo=None):
    """The two collectives of one iteration alone (for the exchange-time report)."""
    dist.all_gather_into_tensor(partials_all, partials_local, group=group)
    exchange_x(dist, bounds, rank, world, x_full, halo, group)


class NoDist:
    """World-size-1 stand-in for torch.distributed (no process group needed):
    the all-gather of one rank's partials is a copy into the output buffer."""

    @staticmethod
    def all_gather_into_tensor(out, inp, group=None):
        out.copy_(inp)


def native_steps(plan) -> ShardSteps:
    """ShardSteps backed by a libspmv plan (device pointers, plan stream)."""
    return ShardSteps(
        spmv=lambda x, y: plan.execute_async(x, y),
        partials=lambda y, p: plan.norm_partials(y, p),
        normalize=lambda y, pa, cnt, xb, nu: plan.normalize(y, pa, cnt, xb, nu),
    )
