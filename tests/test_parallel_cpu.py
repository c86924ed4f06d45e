"""Multi-GPU host logic on CPU: snake partition and the world_size-2 gather
path over the gloo backend (the GPU runner is replaced by a stub that fits
nothing -- only the sharding / collective plumbing is under test here)."""
import os
import socket

import numpy as np
import pytest
import torch.distributed as dist
import torch.multiprocessing as mp

from paper_2010_04678_b200.parallel import run_sharded, shard_widths, snake_partition


def test_snake_partition_balanced_and_complete():
    ranks = [r for r in range(1, 21) for _ in range(25)]  # config 4: 500 models, W = 5250
    for world in (1, 2, 4, 8):
        parts = snake_partition(ranks, world)
        assert sorted(i for p in parts for i in p) == list(range(len(ranks)))
        w = shard_widths(ranks, world)
        assert sum(w) == 5250
        assert max(w) - min(w) <= 20  # within one model of the largest rank
        for p in parts:
            assert p == sorted(p)  # FIFO order kept inside a shard


def test_snake_partition_edge_cases():
    assert snake_partition([], 3) == [[], [], []]
    assert snake_partition([5], 2) == [[0], []]
    with pytest.raises(ValueError):
        snake_partition([1], 0)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2010_04678_b200.model import Model, ModelStatus

    models = [Model.random((4, 3, 2), r, np.random.default_rng(i), id=f"m{i}")
              for i, r in enumerate([1, 2, 3, 4, 5, 6, 7])]

    def stub_runner(t, ms, cfg, r_star):
        assert sum(m.rank for m in ms) <= r_star
        return [Model(id=m.id, rank=m.rank, factors=m.copy_factors(), iterations_done=rank,
                      status=ModelStatus.ITERATION_CAP) for m in ms]

    out = run_sharded(None, models, None, runner=stub_runner)
    q.put((rank, [(m.id, m.iterations_done) for m in out]))
    dist.destroy_process_group()


def test_world_size_two_gloo_gather():
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, 2, port, q)) for r in range(2)]
    for p in procs:
        p.start()
    res = dict(q.get(timeout=120) for _ in procs)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    assert res[0] == res[1]  # every rank sees the full, identical result list
    ids = [i for i, _ in res[0]]
    assert sorted(ids) == sorted(f"m{i}" for i in range(7))
    parts = snake_partition([1, 2, 3, 4, 5, 6, 7], 2)
    assert ids == [f"m{i}" for i in parts[0]] + [f"m{i}" for i in parts[1]]
    assert [it for _, it in res[0]] == [0] * len(parts[0]) + [1] * len(parts[1])


def _slab_worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    from paper_2010_04678_b200.parallel import row_ranges, synthetic_slab

    dims = (40, 6, 5)
    r0, r1 = row_ranges(dims[0], world)[rank]
    slab, sq = synthetic_slab(dims, (r0, r1), 3, 0.1, seed=7, block_rows=10, device="cpu")
    parts = [None] * world
    dist.all_gather_object(parts, (r0, r1, slab.numpy()))
    if rank == 0:
        full = np.empty(dims, order="F")
        for a, b, d in parts:
            full[a:b] = d.reshape((b - a,) + dims[1:], order="F")
        q.put((sq, full))
    dist.destroy_process_group()


def _slab(world):
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_slab_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    out = q.get(timeout=120)
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    return out


def test_config5_slab_generator_gloo():
    """The per-rank slab generator (config 5) builds one tensor whatever the
    world size: signal from generate_synthetic's factors (io.py:114-136),
    noise per fixed row block, norms all-reduced over gloo."""
    sq1, t1 = _slab(1)
    sq4, t4 = _slab(4)
    assert np.array_equal(t1, t4)
    assert abs(sq1 - sq4) <= 1e-12 * sq1
    rng = np.random.default_rng(7)
    fac = [rng.random((d, 3)) for d in (40, 6, 5)]
    signal = np.einsum("ir,jr,kr->ijk", *fac)
    noise = t1 - signal
    assert abs(np.linalg.norm(noise) / np.linalg.norm(signal) - 0.1) < 1e-9


def test_fixed_iteration_count_replays_fifo():
    """The host replay of the FIFO admission (driver.py:199-208) that lets the
    sharded driver enqueue tol <= 0 sweeps without per-iteration syncs."""
    from paper_2010_04678_b200.parallel import fixed_iteration_count as f

    assert f([1, 2, 3], 100, 5) == 5              # all admitted at once
    assert f([4] * 12, 8, 3) == 18                # waves of two (test_driver.py:77-90 shape)
    assert f([3, 3, 4], 7, 2) == 4                # head-of-line blocking: 3+3, then 4
    assert f(list(range(1, 21)) * 5, 1050, 5) == 5
    assert f([5], 4, 3) == 0                      # never admissible
