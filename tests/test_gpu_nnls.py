"""Non-negative updates on the GPU (warp-per-row Lawson-Hanson, csrc/nnls.cuh)
against golden vectors of the reference (als.py:185-278, driver.py:226-227)."""
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def cals():
    import paper_2010_04678_b200 as c

    c._native.load()
    return c


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1.0)


def test_nnls_rows_match_reference(cals):
    g = np.load(os.path.join(GOLDEN, "nnls_rows.npz"))
    for i in range(int(g["n_cases"])):
        x, act, conv = cals.als.nnls_solve_row(g[f"p{i}_h"], g[f"p{i}_f"], g[f"p{i}_act"])
        assert conv == bool(g[f"p{i}_conv"])
        assert np.array_equal(act, g[f"p{i}_newact"]), i
        assert np.all(x >= 0.0)
        assert rel(x, g[f"p{i}_x"]) <= 1e-10, (i, rel(x, g[f"p{i}_x"]))


def test_nnls_update_block_and_state(cals):
    rng = np.random.default_rng(5)
    a = rng.standard_normal((12, 6))
    h = a.T @ a
    m = rng.standard_normal((40, 6))
    st = cals.NnlsState((40, 3), 6)
    x = cals.nnls_update(m, h, st, 0)
    assert x.shape == (40, 6) and np.all(x >= 0)
    assert np.array_equal(st.active[0], x == 0.0)
    # KKT: gradient f - h x <= tol on the pinned variables, == 0 on the free ones
    w = m - x @ h
    assert np.all(w[st.active[0]] <= 1e-9 * np.abs(m).max())
    assert np.allclose(w[~st.active[0]], 0.0, atol=1e-9 * np.abs(m).max())


def _compare(cals, name, t, models, tol, iters, r_star, ls=False, fac_tol=1e-9):
    g = np.load(os.path.join(GOLDEN, f"run_{name}.npz"))
    trace = []
    out = cals.run(t, models, cals.ConvergenceConfig(tol=tol, max_iterations=iters), r_star=r_star,
                   trace=trace, nonneg=True, ls=cals.LineSearchConfig(enabled=ls))
    assert [m.id for m in out] == [str(s) for s in g["order"]]
    assert [m.status.value for m in out] == [str(s) for s in g["status"]]
    assert [m.iterations_done for m in out] == g["iterations"].tolist()
    assert [s.meta["width"] for s in trace] == g["widths"].tolist()
    for m, f in zip(out, g["fit"]):
        assert abs(m.fit - f) <= 1e-6
        for n in range(t.order):
            assert np.all(m.factors[n] >= 0.0)
            assert rel(m.factors[n], g[f"{m.id}_f{n}"]) <= fac_tol, (m.id, n)
    return out


def test_nonneg_cals_matches_reference(cals):
    t = cals.generate_synthetic((12, 10, 8), 3, 0.1, seed=0)
    _compare(cals, "nn_fixed", t, cals.build_models(t.dims, [1, 2, 3, 4], 2, seed=1), 0.0, 8, 20)
    _compare(cals, "nn_tol", t, cals.build_models(t.dims, [2, 3], 2, seed=2), 1e-6, 300, 6,
             fac_tol=1e-6)


def test_nonneg_with_line_search(cals):
    """test_driver.py:138-151: both per-instance options in the fused driver."""
    g = np.load(os.path.join(GOLDEN, "nn_ls_inputs.npz"))
    t = cals.DenseTensor((6, 5, 4), g["data"])
    models = [cals.Model(id=f"m{i}", rank=2, factors=[g[f"m{i}_f{n}"] for n in range(3)])
              for i in range(3)]
    out = cals.run(t, models, cals.ConvergenceConfig(tol=1e-7, max_iterations=300), r_star=6,
                   ls=cals.LineSearchConfig(enabled=True), nonneg=True)
    ref = np.load(os.path.join(GOLDEN, "run_nn_ls.npz"))
    for m in out:
        assert m.status is cals.ModelStatus.CONVERGED
        assert m.fit > 0.99
        assert all(f.min() >= 0.0 for f in m.factors)
    assert sorted(m.id for m in out) == sorted(str(s) for s in ref["order"])
