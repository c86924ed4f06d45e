"""Multi-GPU CALS: model batches sharded over GPUs, tensor replicated.

SURVEY.md section 8(e): models never interact (each output column block
depends only on its own factors), so a sweep over K models partitions into
per-GPU batches with no collective on the data path.  One process per GPU
(``torchrun``); each rank runs the device-resident engine on its share and
the results are gathered once at the end.

The partition is a rank-balanced snake: models sorted by rank (descending,
stable), dealt 0,1,..,P-1,P-1,..,0,... so every GPU carries about W/P columns
(the MTTKRP cost is proportional to the fused width).
"""

from __future__ import annotations

from typing import Callable, Sequence


def snake_partition(ranks: Sequence[int], world: int) -> list[list[int]]:
    """Indices of ``ranks`` per shard, balanced on sum of ranks; each shard
    keeps the input (FIFO) order of its models."""
    if world < 1:
        raise ValueError("world must be >= 1")
    order = sorted(range(len(ranks)), key=lambda i: (-int(ranks[i]), i))
    shards: list[list[int]] = [[] for _ in range(world)]
    for pos, idx in enumerate(order):
        lap, off = divmod(pos, world)
        shards[off if lap % 2 == 0 else world - 1 - off].append(idx)
    return [sorted(s) for s in shards]


def row_ranges(extent: int, world: int) -> list[tuple[int, int]]:
    """Contiguous mode-0 row blocks, as even as possible (config 5: 2000/8 = 250)."""
    base, extra = divmod(int(extent), world)
    out, at = [], 0
    for r in range(world):
        n = base + (1 if r < extra else 0)
        out.append((at, at + n))
        at += n
    return out


def drive_mode0_sharded(engines, tol: float, max_iterations: int, sqnorm: float,
                        allreduce: Callable) -> int:
    """Lock-step driver of the mode-0-sharded CALS loop (SURVEY.md 8(e),
    config 5).  Every rank holds rows [r0, r1) of mode 0 of the tensor and
    of every A0; A1.. are replicated.  Per driver iteration:

      mode 0:  local MTTKRP -> local A0 update -> all-reduce of the mode-0
               Gramians (A0^T A0 summed over row blocks);
      mode n>0: partial MTTKRP over the local rows -> all-reduce -> the same
               (replicated) update on every rank.

    All-reduced inputs are bitwise identical on every rank, so every rank
    takes identical convergence / retirement / admission decisions.
    ``engines`` are the engines this process drives (one per rank in a real
    run, several when ranks are simulated on one GPU); ``allreduce(list)``
    must leave the elementwise sum over all ranks in every tensor of the list.
    Returns the number of driver iterations."""
    import torch

    order = engines[0].order
    for e in engines:
        e.begin(tol, max_iterations, sqnorm)
    bufs = [e.buffers() for e in engines]
    dims = engines[0].dims
    iters = 0
    while True:
        torch.cuda.current_stream().synchronize()
        if all(e.done() for e in engines):
            return iters
        for n in range(order):
            for e in engines:
                e.enqueue_mttkrp(n)
            if n > 0:
                allreduce([b["mttkrp"][:dims[n]] for b in bufs])
            for e in engines:
                e.enqueue_update(n)
            if n == 0:
                allreduce([b["grams"][0] for b in bufs])
        for e in engines:
            e.enqueue_plan()
        iters += 1


def run_mode0_sharded(t_local, rows: tuple[int, int], models: Sequence, cfg, *,
                      r_star: int, sqnorm: float, group=None) -> list:
    """Config-5 entry point for one rank (one process per GPU, NCCL).

    ``t_local`` is this rank's slab of the tensor (rows ``rows`` of mode 0,
    a DenseTensor of dims (r1-r0, I1, ..)); ``models`` carry the full
    starting factors; ``sqnorm`` is ||T||^2 of the whole tensor.  Returns
    the fitted models (full factors, gathered) in retirement order."""
    import numpy as np
    import torch.distributed as dist

    from .engine import CalsEngine
    from .model import STATUS_FROM_CODE, Model, ModelStatus

    r0, r1 = rows
    eng = CalsEngine(t_local.device(), r_star, [m.rank for m in models])
    try:
        eng.load_pool(eng.pack([[m.factors[0][r0:r1]] + list(m.factors[1:]) for m in models]))

        def allreduce(ts):
            for x in ts:
                dist.all_reduce(x, group=group)

        drive_mode0_sharded([eng], cfg.tol, cfg.max_iterations, sqnorm, allreduce)
        res = eng.results()
    finally:
        eng.close()
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    local_a0 = [eng.unpack(res.pool, k)[0] for k in range(len(models))]
    blocks = [local_a0]
    if world > 1:
        blocks = [None] * world
        dist.all_gather_object(blocks, local_a0, group=group)
    out = []
    for k in np.argsort(res.retire_seq, kind="stable"):
        facs = eng.unpack(res.pool, k)
        facs[0] = np.asfortranarray(np.vstack([b[k] for b in blocks]))
        src = models[k]
        src.status = ModelStatus.ACTIVE
        out.append(Model(id=src.id, rank=src.rank, factors=facs, error=float(res.error[k]),
                         fit=float(res.fit[k]), iterations_done=int(res.iterations[k]),
                         status=STATUS_FROM_CODE[int(res.status[k])],
                         seconds_active=float(res.seconds_active[k]), meta=dict(src.meta)))
    return out


def shard_widths(ranks: Sequence[int], world: int) -> list[int]:
    return [sum(int(ranks[i]) for i in s) for s in snake_partition(ranks, world)]


def run_sharded(t, models: Sequence, cfg, *, r_star: int | None = None, group=None,
                runner: Callable | None = None, **kwargs) -> list:
    """Run this rank's share of ``models`` and gather every result on every
    rank.  Output: the shards' outputs concatenated in rank order, each in
    its own retirement order.  ``r_star`` defaults to each shard's width."""
    import torch.distributed as dist

    if runner is None:
        from .driver import run as runner
    world = dist.get_world_size(group) if dist.is_initialized() else 1
    rank = dist.get_rank(group) if dist.is_initialized() else 0
    parts = snake_partition([m.rank for m in models], world)
    mine = [models[i] for i in parts[rank]]
    cap = r_star if r_star is not None else max(1, sum(m.rank for m in mine))
    local = runner(t, mine, cfg, r_star=cap, **kwargs) if mine else []
    if world == 1:
        return list(local)
    gathered: list = [None] * world
    dist.all_gather_object(gathered, list(local), group=group)
    return [m for shard in gathered for m in shard]
