"""Row-sharded multi-GPU driver, one process per GPU.

Rank g owns rows [b_g, b_{g+1}) of A (the nnz-balanced lower_bound rule,
P:708-711, computed by ``spmv_shard_bounds``) and a full replica of x.

* single SpMV: no collective; every rank writes its y block.
* iterated mode (BJ.configs[5]), deferred normalisation (DESIGN.md reading
  25): two x replicas A, B; iteration k reads `cur` (x_0, then yh_{k-1}) and
    1. yh_k block = s * A_g cur, s = the pending exact power-of-two rescale
       of the previous step (nn[1]); partials_g = fixed-chunk sums of
       yh_k^2 -- one libspmv call (spmv_iter_step), written straight into
       the rank's block of `nxt` on the plan stream
    2. all-gather of the partials (rank order)        -- NCCL
    3. norm step on every rank (identical): nu_k = ||yh_k|| / ||yh_{k-1}||,
       a pending rescale factor when the magnitude drifts (never in place)
    4. the exchange of `nxt` blocks                   -- NCCL, or none:
       * halo push (the exchange fused into step 1): for
         banded row blocks the kernel of step 1 also stores the rows each
         neighbour reads straight into that neighbour's `nxt` replica (CUDA
         IPC mapping, NVLink peer stores); the all-gather of step 2 is what
         orders those stores with the neighbour's reads and its previous
         reads of that replica (push_plan, open_push)
       * all-gather(v): one broadcast per rank into its slice of every
         replica (blocks differ in size), or
       * halo exchange: rank g's rows only read x columns
         [col_min_g, col_max_g] (the plan's features), so rank h sends rank
         g just the part of its block inside that range (point-to-point);
         for banded matrices a few planes instead of the whole vector
         (27-pt 384^3 at G = 8: ~2.4 MB per rank per iteration vs 396 MB).
  and swaps the replicas; no x = y / nu pass per iteration. With one rank,
  the library runs the whole loop (spmv_iterate): for row-aligned STREAM /
  D8 plans one launch per iteration, each folding the previous launch's
  per-CTA sums into the norm at its start. At the end x_iters =
  yh_{iters-1} * nn[1] / ||yh_{iters-1}|| over the replica.

This module only orchestrates (argument marshalling, process-group calls);
every arithmetic step runs in the native library. The step functions are
injectable so the orchestration is tested with the ``gloo`` backend on CPU.
"""
from __future__ import annotations

from contextlib import nullcontext
from dataclasses import dataclass
from typing import Callable, Optional, Sequence


@dataclass
class ShardSteps:
    """Per-rank local steps. Tensors are 1-D float64 on the rank's device."""
    # (x_full, y_block, partials_local[P], nn[2], nu[1] or None): y_block = nn[1] * A_g x_full (nn[1] = 0: 1),
    # the partials of y_block^2, and the norm step on them when nu is given (one rank)
    iter_step: Callable[[object, object, object, object, Optional[object]], None]
    norm_step: Callable[[object, int, object, object], None]  # (partials_all, count, nn[2], nu[1])
    unit: Callable[[object, object, object], None]    # (y, nn[2], x_out): x_out = y * nn[1] / nn[0]
    # optional whole single-rank run (x_full, iters, nu_hist): the library's own
    # loop (spmv_iterate), which needs nothing between two SpMVs
    iterate_all: Optional[Callable[[object, int, object], None]] = None
    # optional halo-push form of iter_step (x_full, y_block, partials_local, nn,
    # push_lo, push_lo_end, push_hi, push_hi_begin): also stores local rows
    # [0, push_lo_end) at push_lo and [push_hi_begin, m) at push_hi (device
    # pointers of the neighbours' replicas + this block's first row, or None)
    iter_step_push: Optional[Callable[..., None]] = None
    # optional context-manager factory making the steps' stream the current
    # one, so the collectives (issued on the current stream) are ordered with
    # the native steps (issued on the plan's stream)
    stream: Optional[Callable[[], object]] = None


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


def push_plan(bounds: Sequence[int], needs: Sequence[Sequence[int]], world: int):
    """Halo-push layout of every rank (pure function; the rule
    of the in-process shards, api.cu prepare_push).

    None unless, for every rank g, the rows the other ranks read from g's
    block form a prefix read by one lower rank and/or a suffix read by one
    upper rank (banded row blocks). Else, per rank g, (lo_peer, lo_end,
    hi_peer, hi_begin): g's kernel stores its local rows [0, lo_end) into rank
    lo_peer's replica and [hi_begin, m_g) into hi_peer's (-1, 0 and -1, m_g
    when there is no such peer) -- the same rows halo_plan sends."""
    out = []
    for g in range(world):
        b0, b1 = int(bounds[g]), int(bounds[g + 1])
        lo_peer, lo_end, hi_peer, hi_begin = -1, 0, -1, b1 - b0
        for h in range(world):
            if h == g:
                continue
            lo, hi = int(needs[h][0]), int(needs[h][1])
            a, b = max(lo, b0), min(hi, b1)  # h reads x[a:b) of g's block
            if a >= b:
                continue
            if h < g:
                if lo_peer >= 0 or a != b0:
                    return None
                lo_peer, lo_end = h, b - b0
            else:
                if hi_peer >= 0 or b != b1:
                    return None
                hi_peer, hi_begin = h, a - b0
        out.append((lo_peer, lo_end, hi_peer, hi_begin))
    return out


def open_push(dist, plan, layout, rank: int, world: int, group=None):
    """Collective (every rank calls it): exchange the CUDA IPC handles of the
    plan replicas (spmv_plan_replicas / spmv_ipc_export) and map this rank's
    push peers' (spmv_ipc_open). Returns this rank's `push` argument of
    iterate: ((lo_A, lo_B) or None, lo_end, (hi_A, hi_B) or None, hi_begin),
    the peers' replica base pointers in replica order. iterate() must then run
    on the plan replicas (x_full = replica A, x_alt = replica B) on every
    rank."""
    a, b = plan.replicas()
    handles = [None] * world
    dist.all_gather_object(handles, plan.ipc_export(a) + plan.ipc_export(b), group=group)
    lo_peer, lo_end, hi_peer, hi_begin = layout[rank]
    n = len(handles[rank]) // 2

    def peer(h):
        return (plan.ipc_open(handles[h][:n]), plan.ipc_open(handles[h][n:])) if h >= 0 else None
    return peer(lo_peer), lo_end, peer(hi_peer), hi_begin


def exchange_x(dist, bounds, rank, world, x_full, halo=None, group=None):
    """One x exchange: the halo plan (sends, recvs) when given, else the
    all-gather(v) of the blocks."""
    if world == 1:
        return
    if halo is not None:
        # one coalesced batch (NCCL group): every rank sends and receives at
        # once, so no send waits on a peer's later receive whatever the sizes
        sends, recvs = halo
        ops = [dist.P2POp(dist.isend, x_full[lo:hi], g, group) for g, lo, hi in sends]
        ops += [dist.P2POp(dist.irecv, x_full[lo:hi], g, group) for g, lo, hi in recvs]
        if ops:
            for w in dist.batch_isend_irecv(ops):
                w.wait()
        return
    works = [dist.broadcast(x_full[int(bounds[g]):int(bounds[g + 1])], src=g, group=group, async_op=True)
             for g in range(world) if bounds[g + 1] > bounds[g]]
    for w in works:
        w.wait()


def iterate(dist, steps: ShardSteps, bounds: Sequence[int], rank: int, world: int, x_full, x_alt,
            partials_local, partials_all, nu_hist, nn, iters: int, group=None, halo=None, push=None):
    """Run `iters` power iterations (deferred normalisation) on x_full.

    x_alt: a second replica (len n); partials_all: tensor of world * P;
    nu_hist: tensor of >= iters (nu_k); nn: 2 doubles of state (zeroed here);
    halo: this rank's halo_plan(...) to exchange only the x ranges the ranks
    read (else the full all-gather); push: this rank's open_push(...) result
    (every rank passes one, or none does): the halo rows are stored by the
    SpMV kernels into the neighbours' replicas and no exchange runs. On return
    x_full holds x_iters on every rank (with a halo plan or push: at least the
    range this rank reads and its own block); x_alt is scratch.
    """
    P = partials_local.numel()
    b0, b1 = int(bounds[rank]), int(bounds[rank + 1])
    if world == 1 and steps.iterate_all is not None:
        steps.iterate_all(x_full, iters, nu_hist)
        return
    with steps.stream() if steps.stream is not None else nullcontext():
        nn.zero_()
        cur, nxt = x_full, x_alt
        if push is not None and world > 1:
            # the first pushes write the peers' x_alt: wait until every peer
            # is done with it (its unit() of a previous call reads it)
            dist.all_gather_into_tensor(partials_all, partials_local, group=group)
        for k in range(iters):
            if world == 1:  # the rank's partials are all of them: norm step fused into the step
                steps.iter_step(cur, nxt[b0:b1], partials_local, nn, nu_hist[k:k + 1])
            elif push is not None:
                # nxt is replica (k + 1) % 2 on every rank; the kernel stores the
                # neighbours' halo rows into their replica of that parity
                lo, lo_end, hi, hi_begin = push
                par = (k + 1) & 1
                steps.iter_step_push(cur, nxt[b0:b1], partials_local, nn,
                                     lo[par] + 8 * b0 if lo else None, lo_end,
                                     hi[par] + 8 * b0 if hi else None, hi_begin)
                # orders every peer's pushes into nxt before the next SpMV here
                # reads it, and this rank's reads of cur before peers write it
                dist.all_gather_into_tensor(partials_all, partials_local, group=group)
                steps.norm_step(partials_all, world * P, nn, nu_hist[k:k + 1])
            else:
                steps.iter_step(cur, nxt[b0:b1], partials_local, nn, None)
                dist.all_gather_into_tensor(partials_all, partials_local, group=group)
                steps.norm_step(partials_all, world * P, nn, nu_hist[k:k + 1])
                exchange_x(dist, bounds, rank, world, nxt, halo, group)
            cur, nxt = nxt, cur
        steps.unit(cur, nn, x_full)


def exchange_only(dist, bounds: Sequence[int], rank: int, world: int, x_full, partials_local, partials_all,
                  group=None, halo=None, x_exchange=True):
    """The collectives of one iteration alone (for the exchange-time report;
    x_exchange=False: the halo push, whose x transfer runs inside the SpMV)."""
    dist.all_gather_into_tensor(partials_all, partials_local, group=group)
    if x_exchange:
        exchange_x(dist, bounds, rank, world, x_full, halo, group)


class NoDist:
    """World-size-1 stand-in for torch.distributed (no process group needed):
    the all-gather of one rank's partials is a copy into the output buffer."""

    @staticmethod
    def all_gather_into_tensor(out, inp, group=None):
        if out.data_ptr() != inp.data_ptr():  # (callers may pass one buffer for both: no copy kernel)
            out.copy_(inp)


def native_steps(plan) -> ShardSteps:
    """ShardSteps backed by a libspmv plan (device pointers, plan stream).
    iterate() runs under torch.cuda.stream(<the plan stream>), so NCCL
    collectives and torch ops are enqueued in order with the native steps."""
    import torch

    def stream():
        return torch.cuda.stream(torch.cuda.ExternalStream(plan.stream(), device=torch.cuda.current_device()))

    def iterate_all(x, iters, nu):
        with stream():
            _, nu_h = plan.iterate(x, iters, x_out=x)
            nu[:iters].copy_(torch.from_numpy(nu_h), non_blocking=False)

    return ShardSteps(
        stream=stream,
        iterate_all=iterate_all,
        iter_step=lambda x, y, p, nn, nu: plan.iter_step(x, y, p, nn, nu),
        iter_step_push=lambda x, y, p, nn, lo, le, hi, hb: plan.iter_step_push(x, y, p, nn, lo, le, hi, hb),
        norm_step=lambda pa, cnt, nn, nu: plan.norm_step(pa, cnt, nn, nu),
        unit=lambda y, nn, x: plan.unit(y, nn, x),
    )


def device_view(ptr: int, n: int, device):
    """A float64 torch tensor over n doubles at device pointer ptr (no copy;
    the memory stays owned by whoever allocated it, e.g. the plan's replicas)."""
    import torch

    class _View:
        __cuda_array_interface__ = {"shape": (int(n),), "typestr": "<f8", "data": (int(ptr), False),
                                    "version": 3, "strides": None}
    return torch.as_tensor(_View(), device=device)
