"""Multi-GPU query partitioner: one process per GPU, torch.distributed for the
plumbing (NCCL on GPUs, gloo for the CPU tests).

Queries are independent through the whole Picard/horizon loop (reading R5), so the
only data movement is after the solve: each rank owns a contiguous range of GLOBAL query ids,
solves it with qid_base = its first id (the Philox counter carries the global id, so results
are bit-identical for any number of ranks or split), and the per-slice results are gathered
once. The Picard residuals ε_j(k) need one all-reduce of 2·K·Kp partial sums.
"""
from __future__ import annotations

from typing import Callable

import numpy as np

# history outputs are [K][Kp][M](...): their query axis is 2; every other output leads with M
_HIST = ("vhist", "chist", "dvhist")


def partition(M: int, world: int, rank: int) -> tuple[int, int]:
    """Contiguous balanced split of M global query ids: (first id, count) of `rank`."""
    if world < 1 or not (0 <= rank < world) or M < 0:
        raise ValueError("bad partition arguments")
    base, rem = divmod(M, world)
    count = base + (1 if rank < rem else 0)
    start = rank * base + min(rank, rem)
    return start, count


def _gather_axis(t, counts, axis, group=None):
    """all_gather of a tensor whose `axis` has per-rank sizes `counts` (padded to the max)."""
    import torch
    import torch.distributed as dist

    world = len(counts)
    cmax = max(counts)
    t = t.movedim(axis, 0).contiguous()
    pad = torch.zeros((cmax,) + tuple(t.shape[1:]), dtype=t.dtype, device=t.device)
    pad[: t.shape[0]] = t
    parts = [torch.empty_like(pad) for _ in range(world)]
    dist.all_gather(parts, pad, group=group)
    full = torch.cat([p[:c] for p, c in zip(parts, counts)], dim=0)
    return full.movedim(0, axis)


def gather_results(local: dict, M: int, group=None) -> dict:
    """Gather every rank's result dict (tensors) into full-slice tensors on every rank."""
    import torch.distributed as dist

    world = dist.get_world_size(group)
    counts = [partition(M, world, r)[1] for r in range(world)]
    out = {}
    for k, t in local.items():
        if t is None:
            continue
        axis = 2 if k in _HIST else 0
        out[k] = _gather_axis(t, counts, axis, group)
    return out


def solve_sharded(solve_fn: Callable, x: np.ndarray, group=None, gather: bool = True):
    """Run `solve_fn(x_local, qid_base)` on this rank's query range, optionally gather.

    solve_fn is e.g. `lambda xl, base: solver.solve_slice(xl, qid_base=base)`.
    Returns (result dict, (start, count))."""
    import torch.distributed as dist

    world, rank = dist.get_world_size(group), dist.get_rank(group)
    start, count = partition(x.shape[0], world, rank)
    local = solve_fn(x[start:start + count], start)
    if not gather:
        return local, (start, count)
    return gather_results(local, x.shape[0], group), (start, count)


def residuals_sharded(vhist_local: np.ndarray, g0_local: np.ndarray, device=None, group=None):
    """ε_j(k) = ‖v^(k+1) − v^(k)‖₂ / ‖v^(k)‖₂ over the whole sharded slice (R11): host
    partial sums from hjmc_residual_partials, one all-reduce (SUM) of the K·Kp·2 doubles, then
    hjmc_residual_eps. The all-reduce runs on the backend's device (CUDA for NCCL)."""
    import torch
    import torch.distributed as dist

    from .solver import residual_eps, residual_partials

    part = residual_partials(vhist_local, g0_local)          # [K][Kp][2]
    if dist.is_initialized():
        if device is None:
            device = (torch.device("cuda", torch.cuda.current_device())
                      if dist.get_backend(group) == "nccl" else torch.device("cpu"))
        t = torch.from_numpy(part).to(device)
        dist.all_reduce(t, op=dist.ReduceOp.SUM, group=group)
        part = t.cpu().numpy()
    return residual_eps(part)
