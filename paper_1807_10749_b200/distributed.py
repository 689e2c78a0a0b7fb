"""Path partitioning across GPUs (one process per GPU) and the final reduce.

The reference shards one job per retained prefix over forked CPU workers
(``orchestrator.shard``, ``orchestrator.py:80-85``; round-robin assignment
``:251-270``) and folds the complex128 shard vectors in ascending prefix order
(``_merge_verified``, ``:340-342``).  Here each rank owns one contiguous
range of the sorted retained prefixes (all their branches), so the prefix
sharing of the path tree stays inside one GPU, accumulates its complex128
partial in HBM, and a single ``all_reduce``/``reduce`` (NCCL over
NVLink/NVSwitch) joins them.  There is no other exchange.
"""
from __future__ import annotations

import numpy as np


def partition_prefixes(prefixes, world_size: int, rank: int) -> np.ndarray:
    """Contiguous slice of the sorted prefixes for ``rank``; sizes differ by at most one.

    Every prefix carries the same number of branches, so equal prefix counts
    are equal path counts.
    """
    if not 0 <= rank < world_size:
        raise ValueError(f"rank {rank} outside world of {world_size}")
    pre = np.sort(np.asarray(prefixes, dtype=np.int64))
    n = pre.size
    lo = (n * rank) // world_size
    hi = (n * (rank + 1)) // world_size
    return pre[lo:hi]


def sharded_sum(partial_fn, prefixes, group=None, dst: int | None = None):
    """Run ``partial_fn(my_prefixes) -> torch float64 tensor (2*n_req)`` and sum over ranks.

    ``dst=None`` all-reduces (every rank gets the total), otherwise reduces
    to rank ``dst``.  Works with any torch.distributed backend: NCCL on
    device tensors for the product path, gloo on CPU tensors in the tests.
    """
    import torch.distributed as dist

    world = dist.get_world_size(group)
    rank = dist.get_rank(group)
    mine = partition_prefixes(prefixes, world, rank)
    part = partial_fn(mine)
    if world > 1:
        if dst is None:
            dist.all_reduce(part, op=dist.ReduceOp.SUM, group=group)
        else:
            dist.reduce(part, dst=dst, op=dist.ReduceOp.SUM, group=group)
    return part


REPRO_SLICES = 8  # fixed reduction slices: results bit-identical at 1, 2, 4 and 8 ranks


def reproducible_sum(partial_fn, prefixes, group=None, n_slices: int = REPRO_SLICES):
    """Bit-reproducible form of :func:`sharded_sum` (optional).

    The sorted prefixes are cut into ``n_slices`` fixed contiguous slices that
    do not depend on the world size; each rank evaluates the slices it owns
    (``partial_fn(slice)`` per slice), one ``all_gather`` collects every
    slice's partial, and every rank sums them in slice order.  The sum order
    is then the same at any world size dividing ``n_slices`` -- NCCL's
    reduction order is not -- so the totals are bitwise equal at 1, 2, 4 and 8
    GPUs.  Costs ``n_slices`` partials of traffic instead of one.
    """
    import torch
    import torch.distributed as dist

    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if n_slices % world:
        raise ValueError(f"world size {world} does not divide the {n_slices} reduction slices")
    per = n_slices // world
    mine = [partial_fn(partition_prefixes(prefixes, n_slices, s)) for s in range(rank * per, (rank + 1) * per)]
    local = torch.stack(mine)
    if world > 1:
        gathered = [torch.empty_like(local) for _ in range(world)]
        dist.all_gather(gathered, local, group=group)
        parts = torch.cat(gathered)
    else:
        parts = local
    total = parts[0].clone()
    for s in range(1, n_slices):
        total += parts[s]
    return total


def run_batched_sharded(circuit, plan, requests, prefixes=None, group=None, dst: int | None = 0,
                        device: int | None = None, dtype="c64", reproducible: bool = False):
    """Multi-GPU ``run_batched``: this rank's prefix range on its GPU, then an NCCL reduce.

    Returns the :class:`AmplitudeBatch` on rank ``dst`` (every rank when
    ``dst`` is None) and ``None`` elsewhere.  ``reproducible=True`` sums fixed
    prefix slices in a fixed order (:func:`reproducible_sum`): bitwise the same
    amplitudes at 1, 2, 4 and 8 GPUs.
    """
    import torch
    import torch.distributed as dist

    from .amplitudes import AmplitudeBatch
    from .pathsum import _engine_for

    if device is None:
        device = torch.cuda.current_device()
    from .engine import ENGINES

    eng = ENGINES.get(device, dtype)
    with eng.lock:
        eng, idx = _engine_for(circuit, plan, requests, device, dtype)
        pre = plan.retained if prefixes is None else np.asarray(prefixes, dtype=np.int64)
        # run on torch's stream: the partial's allocation, the engine's writes and the
        # collective that reads them are then ordered by construction
        eng.set_stream(torch.cuda.current_stream(device).cuda_stream)
        try:
            def partial(mine):
                if not mine.size:
                    return torch.zeros(2 * idx.size, dtype=torch.float64, device=f"cuda:{device}")
                out = torch.empty(2 * idx.size, dtype=torch.float64, device=f"cuda:{device}")
                # accumulate=False: the engine writes every entry of ``out``
                eng.run(plan.x_p, mine, 0, plan.branch_space, out_device_ptr=out.data_ptr(),
                        want_host=False)
                return out

            if reproducible:
                total = reproducible_sum(partial, pre, group=group)
            else:
                total = sharded_sum(partial, pre, group=group, dst=dst)
        finally:
            eng.set_stream(None)
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    if dst is not None and rank != dst:
        return None
    host = total.cpu().numpy().view(np.complex128)
    return AmplitudeBatch(idx, host)
