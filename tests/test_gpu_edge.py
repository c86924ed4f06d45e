"""Edge cases of the GPU driver against the numpy oracle: odd / tiny extents,
high order, ranks above the register fast path, heavy refill churn, empty
input, degenerate tensors."""
import numpy as np
import pytest

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cals():
    import paper_2010_04678_b200 as c

    c._native.load()
    return c


def _vs_oracle(cals, dims, ranks, per_rank, tol, iters, r_star, fac_tol=1e-9, seed=0):
    from oracle import cals_oracle as O

    dims, data = O.generate_synthetic(dims, max(2, max(ranks)), 0.1, seed=seed)
    models = O.build_models(dims, ranks, per_rank, seed=seed + 1)
    ref = O.run_cals(data, dims, models, tol, iters, r_star)
    t = cals.DenseTensor(dims, data)
    ms = [cals.Model(id=i, rank=r, factors=[f.copy() for f in fac]) for i, r, fac in models]
    out = cals.run(t, ms, cals.ConvergenceConfig(tol=tol, max_iterations=iters), r_star=r_star)
    assert [m.id for m in out] == [r.id for r in ref]
    for m, r in zip(out, ref):
        assert m.status.value == r.status and m.iterations_done == r.iterations
        assert abs(m.fit - r.fit) <= 1e-6
        for a, b in zip(m.factors, r.factors):
            assert np.linalg.norm(a - b) / max(np.linalg.norm(b), 1.0) <= fac_tol, m.id
    return out


def test_odd_and_tiny_extents(cals):
    _vs_oracle(cals, (13, 9, 7), [1, 2, 3], 2, 0.0, 5, 12)
    _vs_oracle(cals, (3, 2, 5), [1, 2], 2, 0.0, 5, 6)
    _vs_oracle(cals, (1, 6, 5), [1], 2, 0.0, 3, 2)


def test_high_order(cals):
    _vs_oracle(cals, (4, 3, 5, 2, 3), [1, 2, 3], 1, 0.0, 5, 6)


def test_generic_update_path_ranks_above_32(cals):
    """R > 32 runs the generic (non-register) update instantiation."""
    _vs_oracle(cals, (40, 36, 34), [33, 40], 1, 0.0, 4, 80, fac_tol=1e-8)


def test_generic_update_path_ranks_above_128(cals):
    """R > 128: the generic update keeps its R x R matrix in global scratch
    (csrc/update.cuh kSmemRankMax); the reference has no rank limit."""
    _vs_oracle(cals, (170, 165, 160), [130, 150], 1, 0.0, 3, 280, fac_tol=1e-8)


def test_update_factor_rank_200(cals):
    """The operator API (als.py:74-96) at rank 200 against scipy's cho_solve."""
    from scipy.linalg import cho_factor, cho_solve

    rng = np.random.default_rng(11)
    a = rng.random((260, 200))
    h = a.T @ a + np.eye(200)
    m = rng.standard_normal((90, 200))
    want = cho_solve(cho_factor(h, lower=False), m.T).T
    got = cals.update_factor(m, h)
    assert np.linalg.norm(got - want) / np.linalg.norm(want) <= 1e-10
    with pytest.raises(ValueError):
        cals.update_factor(np.ones((2, 513)), np.eye(513))


@pytest.mark.parametrize("ranks", [[1, 8], [9, 16], [17, 24], [25, 32]])
def test_update_rank_buckets(cals, ranks):
    """The update kernel is instantiated per rank bucket (largest rank of the
    batch: <= 8 / 16 / 24 / 32); each bucket at both of its ends."""
    _vs_oracle(cals, (34, 33, 35), ranks, 1, 0.0, 4, sum(ranks), fac_tol=1e-8)


def test_refill_churn(cals):
    _vs_oracle(cals, (10, 9, 8), [1, 2, 3], 12, 1e-5, 60, 5, fac_tol=1e-6, seed=7)


def test_empty_and_degenerate(cals):
    t = cals.DenseTensor((3, 3, 3), np.ones(27))
    assert cals.run(t, [], cals.ConvergenceConfig()) == []
    z = cals.DenseTensor((3, 3, 3), np.zeros(27))
    with pytest.raises(ValueError):
        cals.run(z, [cals.Model.random((3, 3, 3), 1, 0, id="a")], cals.ConvergenceConfig())
    with pytest.raises(ValueError):
        cals.run(t, [cals.Model.random((3, 3, 4), 1, 0, id="a")], cals.ConvergenceConfig())


def test_sequential_and_parallel_modes_match_fused(cals):
    rng = np.random.default_rng(3)
    t = cals.DenseTensor.from_array(rng.standard_normal((9, 8, 7)))
    starts = [cals.Model.random(t.dims, r, rng, id=f"r{r}") for r in (1, 2, 4)]
    cfg = cals.ConvergenceConfig(tol=0.0, max_iterations=6)
    outs = {mode: {m.id: m for m in cals.run(t, starts, cfg, mode=mode, r_star=7)}
            for mode in cals.ExecutionMode}
    trace = []
    cals.run(t, starts, cfg, mode=cals.ExecutionMode.SEQUENTIAL, trace=trace)
    assert [s.label for s in trace] == [f"als:r{r}" for r in (1, 2, 4)]
    for mode in (cals.ExecutionMode.SEQUENTIAL, cals.ExecutionMode.PARALLEL):
        for k, m in outs[mode].items():
            for a, b in zip(m.factors, outs[cals.ExecutionMode.CALS][k].factors):
                assert np.array_equal(a, b)
