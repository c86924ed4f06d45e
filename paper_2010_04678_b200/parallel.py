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

import math
from typing import Callable, Sequence

import numpy as np


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
    # tol <= 0: every admitted model runs exactly max_iterations, so the number
    # of driver iterations is known from the FIFO admission alone and they are
    # enqueued back to back (stream-ordered NCCL all-reduces, no per-iteration
    # host round trip); failures only retire models earlier, which leaves the
    # remaining iterations no-ops on the device
    known = fixed_iteration_count(engines[0].ranks, engines[0].r_star,
                                  max_iterations) if tol <= 0 else 0
    iters = 0
    while True:
        if known <= 0 or iters >= known:
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


def fixed_iteration_count(ranks: Sequence[int], capacity: int, max_iterations: int) -> int:
    """Driver iterations of a run in which every model takes exactly
    ``max_iterations`` (tol <= 0): the FIFO admission with head-of-line
    blocking of driver.py:199-208 replayed on the host (as the engine's
    fixed_iteration_count in csrc/engine.cu).  0 if the queue can block
    forever (a rank above the capacity)."""
    active: list[list[int]] = []  # [rank, iterations left]
    head, width, count = 0, 0, 0
    ranks = [int(r) for r in ranks]

    def admit():
        nonlocal head, width
        while head < len(ranks) and width + ranks[head] <= capacity:
            active.append([ranks[head], max_iterations])
            width += ranks[head]
            head += 1

    admit()
    while active:
        count += 1
        keep = []
        for a in active:
            a[1] -= 1
            if a[1] > 0:
                keep.append(a)
            else:
                width -= a[0]
        active[:] = keep
        admit()
        if not active and head < len(ranks):
            return 0
    return count


def _allreduce_sum(tensors, group=None) -> None:
    """In-place elementwise sum over the group.  NCCL reduces CUDA tensors
    directly; gloo (CPU tests, several processes sharing one GPU) goes
    through host copies.  Either way every rank ends with identical bits
    (ring reduction order fixed by the collective)."""
    import torch.distributed as dist

    if not dist.is_initialized() or dist.get_world_size(group) == 1:
        return
    gloo = dist.get_backend(group) == "gloo"
    for x in tensors:
        if gloo and x.is_cuda:
            h = x.cpu()
            dist.all_reduce(h, group=group)
            x.copy_(h)
        else:
            dist.all_reduce(x, group=group)


def synthetic_slab(dims, rows: tuple[int, int], true_rank: int, noise_level: float = 0.1,
                   seed: int = 0, *, block_rows: int = 50, device=None, group=None):
    """This rank's mode-0 row slab of a config-5-style synthetic tensor,
    generated where it lives -- the whole tensor (32 GB at c5) never exists
    on one host or device.

    Signal: the factors ``generate_synthetic`` draws (io.py:114-136: one
    ``rng.random((I_n, true_rank))`` per mode from ``default_rng(seed)``),
    drawn identically on every rank (a few MB), contracted on ``device`` for
    rows ``[r0, r1)`` only.  Noise: standard normal per fixed block of
    ``block_rows`` mode-0 rows from a generator seeded by (seed, block), so
    the tensor does not depend on the world size; its scale
    ``noise_level * ||signal|| / ||G||`` uses the global norms (one
    all-reduce of two scalars, setup only).  The noise stream is not the
    reference's (its generator draws the full tensor at once).

    Returns ``(slab, sqnorm)``: a CUDA/CPU float64 tensor holding the slab
    linearised mode-0 fastest (flat index ``i + (r1 - r0) * (j + I1 * k)``)
    and ||T||^2 of the whole tensor."""
    import torch

    dims = tuple(int(d) for d in dims)
    r0, r1 = int(rows[0]), int(rows[1])
    if len(dims) != 3:
        raise ValueError("synthetic_slab builds 3-way tensors")
    if r0 % block_rows or (r1 % block_rows and r1 != dims[0]):
        raise ValueError(f"slab rows {rows} must lie on {block_rows}-row noise blocks")
    dev = torch.device(device) if device is not None else torch.device("cuda")
    rng = np.random.default_rng(seed)
    fac = [rng.random((d, true_rank)) for d in dims]  # generate_synthetic's draw order
    b = torch.from_numpy(fac[1]).to(dev)
    c = torch.from_numpy(fac[2]).to(dev)
    n_blocks = (dims[0] + block_rows - 1) // block_rows
    blocks = range(r0 // block_rows, (r1 + block_rows - 1) // block_rows)

    # Everything is formed per fixed row block (signal, noise, partial norms)
    # and the norms are summed in block order, so every world size produces
    # the same tensor bit for bit.
    def block_rows_of(blk):
        return blk * block_rows, min(dims[0], (blk + 1) * block_rows)

    def signal(blk):
        lo, hi = block_rows_of(blk)
        a = torch.from_numpy(fac[0][lo:hi]).to(dev)
        return torch.einsum("kr,jr,ir->kji", c, b, a)  # (I2, I1, rows): mode-0 fastest

    def noise(blk):
        lo, hi = block_rows_of(blk)
        g = torch.Generator(device=dev)
        g.manual_seed(int(seed) * 1_000_003 + blk)
        return torch.randn((dims[2], dims[1], hi - lo), generator=g, device=dev,
                           dtype=torch.float64)

    def ordered_total(per_block):
        _allreduce_sum([per_block], group)  # each block's value comes from one rank
        return float(sum(float(v) for v in per_block.cpu().tolist()))

    slab = torch.empty((dims[2], dims[1], r1 - r0), dtype=torch.float64, device=dev)
    sig_sq = torch.zeros(n_blocks, dtype=torch.float64, device=dev)
    g_sq = torch.zeros(n_blocks, dtype=torch.float64, device=dev)
    for blk in blocks:
        lo, hi = block_rows_of(blk)
        sb = signal(blk)
        slab[:, :, lo - r0:hi - r0] = sb
        sig_sq[blk] = torch.sum(sb * sb)
        if noise_level > 0.0:
            g = noise(blk)
            g_sq[blk] = torch.sum(g * g)
    if noise_level > 0.0:
        scale = noise_level * math.sqrt(ordered_total(sig_sq)) / math.sqrt(ordered_total(g_sq))
        for blk in blocks:
            lo, hi = block_rows_of(blk)
            slab[:, :, lo - r0:hi - r0].add_(noise(blk), alpha=scale)
    sq = torch.zeros(n_blocks, dtype=torch.float64, device=dev)
    for blk in blocks:
        lo, hi = block_rows_of(blk)
        part = slab[:, :, lo - r0:hi - r0]
        sq[blk] = torch.sum(part * part)
    return slab.reshape(-1), ordered_total(sq)


class Mode0Shard:
    """One rank of the config-5 run: the engine over this rank's slab (rows
    ``rows`` of mode 0 of the tensor and of every A0), the model pool on the
    device, and the lock-step sweep (``drive_mode0_sharded`` with a
    torch.distributed all-reduce).  ``t_local`` is a DenseTensor of the slab,
    a DeviceTensor, or a CUDA float64 tensor holding the slab (mode-0
    fastest, as ``synthetic_slab`` returns it)."""

    def __init__(self, t_local, rows: tuple[int, int], dims, models: Sequence, *, r_star: int,
                 group=None):
        import torch

        from .engine import CalsEngine
        from .tensor import DeviceTensor

        self.rows = (int(rows[0]), int(rows[1]))
        self.dims = tuple(int(d) for d in dims)
        self.group = group
        self.models = list(models)
        local_dims = (self.rows[1] - self.rows[0],) + self.dims[1:]
        if isinstance(t_local, torch.Tensor):
            self._slab = t_local  # keep the borrowed device buffer alive
            dev_t = DeviceTensor.from_device(local_dims, t_local.data_ptr())
        elif hasattr(t_local, "handle"):
            dev_t = t_local
        else:
            dev_t = t_local.device()
        self.dev_t = dev_t
        self.engine = CalsEngine(dev_t, r_star, [m.rank for m in self.models])
        r0, r1 = self.rows
        host = self.engine.pack([[m.factors[0][r0:r1]] + list(m.factors[1:])
                                 for m in self.models])
        self.pool = torch.from_numpy(host).cuda()

    def sweep(self, tol: float, max_iterations: int, sqnorm: float) -> int:
        """One full sweep from the starting pool; returns driver iterations."""
        self.engine.load_pool(self.pool)
        return drive_mode0_sharded([self.engine], tol, max_iterations, sqnorm,
                                   lambda ts: _allreduce_sum(ts, self.group))

    def results(self) -> list:
        """The fitted models (full A0 gathered from every rank) in retirement
        order, as ``run`` returns them."""
        import torch.distributed as dist

        from .model import STATUS_FROM_CODE, Model, ModelStatus

        eng = self.engine
        res = eng.results()
        world = dist.get_world_size(self.group) if dist.is_initialized() else 1
        local_a0 = [eng.unpack(res.pool, k)[0] for k in range(len(self.models))]
        blocks = [local_a0]
        if world > 1:
            blocks = [None] * world
            dist.all_gather_object(blocks, local_a0, group=self.group)
        out = []
        for k in np.argsort(res.retire_seq, kind="stable"):
            facs = eng.unpack(res.pool, k)
            facs[0] = np.asfortranarray(np.vstack([b[k] for b in blocks]))
            src = self.models[k]
            src.status = ModelStatus.ACTIVE
            out.append(Model(id=src.id, rank=src.rank, factors=facs,
                             error=float(res.error[k]), fit=float(res.fit[k]),
                             iterations_done=int(res.iterations[k]),
                             status=STATUS_FROM_CODE[int(res.status[k])],
                             seconds_active=float(res.seconds_active[k]), meta=dict(src.meta)))
        return out

    def close(self) -> None:
        self.engine.close()


def run_mode0_sharded(t_local, rows: tuple[int, int], models: Sequence, cfg, *,
                      r_star: int, sqnorm: float, dims=None, group=None) -> list:
    """Config-5 entry point for one rank (one process per GPU; NCCL, or gloo
    for processes sharing a device).  ``t_local`` is this rank's slab
    (see Mode0Shard); ``models`` carry the full starting factors; ``sqnorm``
    is ||T||^2 of the whole tensor; ``dims`` the full tensor's extents
    (default: the slab's with I0 from the models).  Returns the fitted
    models (full factors, gathered on every rank) in retirement order."""
    if dims is None:
        dims = tuple(int(f.shape[0]) for f in models[0].factors)
    shard = Mode0Shard(t_local, rows, dims, models, r_star=r_star, group=group)
    try:
        shard.sweep(cfg.tol, cfg.max_iterations, sqnorm)
        return shard.results()
    finally:
        shard.close()


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
