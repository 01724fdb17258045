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
    5. all-gather(v) of the x blocks into every replica: one broadcast per
       rank into its slice of x (blocks differ in size)  -- NCCL

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


def iterate(dist, steps: ShardSteps, bounds: Sequence[int], rank: int, world: int, x_full, y_local,
            partials_local, partials_all, nu_hist, iters: int, group=None):
    """Run `iters` power iterations in place on x_full (the replica).

    partials_all: tensor of world * P; nu_hist: tensor of >= iters (nu_k).
    Returns nothing; x_full holds x_iters on every rank.
    """
    P = partials_local.numel()
    b0, b1 = int(bounds[rank]), int(bounds[rank + 1])
    for k in range(iters):
        steps.spmv(x_full, y_local)
        steps.partials(y_local, partials_local)
        dist.all_gather_into_tensor(partials_all, partials_local, group=group)
        steps.normalize(y_local, partials_all, world * P, x_full[b0:b1], nu_hist[k:k + 1])
        if world > 1:
            works = [dist.broadcast(x_full[int(bounds[g]):int(bounds[g + 1])], src=g, group=group, async_op=True)
                     for g in range(world) if bounds[g + 1] > bounds[g]]
            for w in works:
                w.wait()


def exchange_only(dist, bounds: Sequence[int], rank: int, world: int, x_full, partials_local, partials_all,
                  group=None):
    """The two collectives of one iteration alone (for the exchange-time report)."""
    dist.all_gather_into_tensor(partials_all, partials_local, group=group)
    if world > 1:
        works = [dist.broadcast(x_full[int(bounds[g]):int(bounds[g + 1])], src=g, group=group, async_op=True)
                 for g in range(world) if bounds[g + 1] > bounds[g]]
        for w in works:
            w.wait()


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
