"""Config-5 decomposition (mode-0 tensor sharding + all-reduce of the partial
MTTKRPs and mode-0 Gramians) on ONE GPU: every "rank" is its own engine over
its row slab, driven in lock step by parallel.drive_mode0_sharded with an
in-process all-reduce (sum).  The multi-process NCCL run uses the same driver
with torch.distributed.all_reduce.  Checked against the oracle on the full
tensor."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


def _sum_allreduce(ts):
    s = ts[0].clone()
    for x in ts[1:]:
        s += x
    for x in ts:
        x.copy_(s)


@pytest.mark.parametrize("world,r_star,tol,iters", [(2, 20, 0.0, 5), (3, 20, 0.0, 5),
                                                    (2, 6, 1e-6, 60)])
def test_mode0_sharded_matches_oracle(world, r_star, tol, iters):
    import paper_2010_04678_b200 as cals
    from oracle import cals_oracle as O
    from paper_2010_04678_b200.engine import CalsEngine
    from paper_2010_04678_b200.parallel import drive_mode0_sharded, row_ranges

    dims, data = O.generate_synthetic((25, 20, 16), 4, 0.1, seed=0)
    models = O.build_models(dims, [1, 2, 3, 4], 2, seed=1)
    ref = O.run_cals(data, dims, models, tol, iters, r_star)
    arr = data.reshape(dims, order="F")
    sq = float(data @ data)
    engines, ranges = [], row_ranges(dims[0], world)
    for r0, r1 in ranges:
        tl = cals.DenseTensor.from_array(arr[r0:r1])
        e = CalsEngine(tl.device(), r_star, [r for _, r, _ in models])
        e._keep = tl
        e.load_pool(e.pack([[f[0][r0:r1]] + f[1:] for _, _, f in models]))
        engines.append(e)
    drive_mode0_sharded(engines, tol, iters, sq, _sum_allreduce)
    res = [e.results() for e in engines]
    # replicated state is identical on every rank
    for r in res[1:]:
        assert np.array_equal(r.status, res[0].status)
        assert np.array_equal(r.iterations, res[0].iterations)
        assert np.array_equal(r.retire_seq, res[0].retire_seq)
        assert np.array_equal(r.fit, res[0].fit)
    order = np.argsort(res[0].retire_seq, kind="stable")
    assert [models[k][0] for k in order] == [x.id for x in ref]
    for k, want in zip(order, ref):
        assert res[0].iterations[k] == want.iterations
        assert abs(res[0].fit[k] - want.fit) <= 1e-9
        facs = engines[0].unpack(res[0].pool, k)
        facs[0] = np.vstack([engines[w].unpack(res[w].pool, k)[0] for w in range(world)])
        for a, b in zip(facs, want.factors):
            assert np.linalg.norm(a - b) / max(np.linalg.norm(b), 1.0) <= 1e-9
    for e in engines:
        e.close()
