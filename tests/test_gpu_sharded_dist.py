"""Config 5 through torch.distributed: two processes (gloo; both on cuda:0,
this box has one GPU), each holding a mode-0 row slab of a down-scaled
240 x 200 x 100 tensor and running parallel.run_mode0_sharded -- the partial
MTTKRPs of modes 1, 2 and the mode-0 Gramians all-reduced every driver
iteration.  Rank 0 checks the gathered models against the
oracle on the full tensor (reference driver.py:185-285 + 213-235), at the
north_star bars: factors 1e-9 after 5 fixed iterations; equal statuses,
retirement order and iteration counts for the converging refill run.

Also: the per-rank slab generator builds the same tensor for every world
size (noise blocks are world-independent), here 1 vs 2 ranks."""
import os
import socket

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = (240, 200, 100)


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    port = s.getsockname()[1]
    s.close()
    return port


def _worker(rank, world, port, case, q):
    import sys

    sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    import torch
    import torch.distributed as dist

    torch.cuda.set_device(0)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import paper_2010_04678_b200 as cals
        from oracle import cals_oracle as O
        from paper_2010_04678_b200.parallel import row_ranges, run_mode0_sharded, synthetic_slab

        if case == "slab":
            r0, r1 = row_ranges(DIMS[0], world)[rank]
            slab, sq = synthetic_slab(DIMS, (r0, r1), 4, 0.1, seed=3, block_rows=40)
            parts = [None] * world
            dist.all_gather_object(parts, (r0, r1, slab.cpu().numpy()))
            if rank == 0:
                full = np.empty(DIMS, order="F")
                for a, b, d in parts:
                    full[a:b] = d.reshape((b - a,) + DIMS[1:], order="F")
                q.put(("slab", world, sq, full.ravel(order="F")))
            return
        tol, iters, r_star = case
        dims, data = O.generate_synthetic(DIMS, 4, 0.1, seed=0)
        arr = data.reshape(dims, order="F")
        r0, r1 = row_ranges(dims[0], world)[rank]
        t_local = cals.DenseTensor.from_array(arr[r0:r1])
        models = [cals.Model(id=i, rank=r, factors=f)
                  for i, r, f in O.build_models(dims, [1, 2, 3, 4], 2, seed=1)]
        out = run_mode0_sharded(t_local, (r0, r1), models,
                                cals.ConvergenceConfig(tol=tol, max_iterations=iters),
                                r_star=r_star, sqnorm=float(data @ data), dims=dims)
        if rank == 0:
            q.put(("run", [(m.id, m.status.value, m.iterations_done, m.fit,
                            [np.asarray(f) for f in m.factors]) for m in out]))
    finally:
        dist.destroy_process_group()


def _spawn(world, case):
    import torch.multiprocessing as mp

    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, case, q)) for r in range(world)]
    for p in procs:
        p.start()
    try:
        res = q.get(timeout=300)
    finally:
        for p in procs:
            p.join(timeout=120)
    for p in procs:
        assert p.exitcode == 0
    return res


@pytest.mark.parametrize("tol,iters,r_star", [(0.0, 5, 20), (1e-6, 60, 6)])
def test_mode0_sharded_two_processes_match_oracle(tol, iters, r_star):
    from oracle import cals_oracle as O

    kind, got = _spawn(2, (tol, iters, r_star))
    dims, data = O.generate_synthetic(DIMS, 4, 0.1, seed=0)
    ref = O.run_cals(data, dims, O.build_models(dims, [1, 2, 3, 4], 2, seed=1), tol, iters,
                     r_star)
    assert [g[0] for g in got] == [r.id for r in ref]
    for (mid, status, its, fit, facs), want in zip(got, ref):
        assert status == want.status and its == want.iterations, mid
        assert abs(fit - want.fit) <= 1e-9, mid
        for a, b in zip(facs, want.factors):
            assert np.linalg.norm(a - b) / max(np.linalg.norm(b), 1.0) <= 1e-9, mid


def test_slab_generator_world_independent():
    _, w1, sq1, t1 = _spawn(1, "slab")
    _, w2, sq2, t2 = _spawn(2, "slab")
    assert np.array_equal(t1, t2)
    assert abs(sq1 - sq2) <= 1e-12 * sq1
    assert abs(sq1 - float(t1 @ t1)) <= 1e-10 * sq1
