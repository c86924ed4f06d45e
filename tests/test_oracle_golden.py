"""Pin the numpy oracle against golden vectors produced by the real reference.

CPU only.  The fixtures come from oracle/make_golden.py (reference imported
from /root/reference in the build container).
"""
import json
import os

import numpy as np
import pytest

from oracle import cals_oracle as O

from conftest import GOLDEN


def load(name):
    return np.load(os.path.join(GOLDEN, name), allow_pickle=False)


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def test_known_answers():
    k = load("kat.npz")
    ones = np.ones((2, 1))
    got = O.mttkrp(np.arange(1.0, 9.0), (2, 2, 2), [ones, ones, ones], 0).ravel()
    assert got.tolist() == k["mttkrp_2x2x2_mode0"].tolist() == [16.0, 20.0]
    assert O.khatri_rao(np.array([[1.0], [2.0]]), np.array([[3.0], [4.0], [5.0]])).ravel().tolist() \
        == k["krp_12_345"].tolist() == [3, 4, 5, 6, 8, 10]
    assert O.update_factor(np.array([[16.0], [20.0]]), np.array([[4.0]])).ravel().tolist() \
        == k["update_16_20_over_4"].tolist() == [4.0, 5.0]
    assert O.mttkrp_flops((300, 300, 300), 1) == 54_000_000


def test_mttkrp_matches_reference_all_orders():
    g = load("mttkrp.npz")
    for ci in range(int(g["n_cases"])):
        dims = tuple(int(d) for d in g[f"c{ci}_dims"])
        fac = [g[f"c{ci}_f{n}"] for n in range(len(dims))]
        for n in range(len(dims)):
            want = g[f"c{ci}_m{n}"]
            assert rel(O.mttkrp(g[f"c{ci}_data"], dims, fac, n), want) <= 1e-12, (ci, n)


def test_update_and_error_match_reference():
    g = load("update.npz")
    for i in range(int(g["n_cases"])):
        got = O.update_factor(g[f"u{i}_m"], g[f"u{i}_h"])
        assert rel(got, g[f"u{i}_a"]) <= 1e-10, i
    dims = (5, 4, 3)
    fac = [g[f"fe_f{n}"] for n in range(3)]
    ml = O.mttkrp(g["fe_data"], dims, fac, 2)
    e = O.fast_error(float(g["fe_data"] @ g["fe_data"]), fac[2], ml, [O.gramian(f) for f in fac])
    assert e == pytest.approx(float(g["fe_error"]), rel=1e-12)
    assert O.fit_from_error(e, float(g["fe_data"] @ g["fe_data"])) == pytest.approx(float(g["fe_fit"]), abs=1e-13)


def test_builders_bitwise():
    g = load("builders.npz")
    _, data = O.generate_synthetic((7, 6, 5), 3, 0.1, seed=0)
    assert np.array_equal(data, g["synth_7x6x5"])
    for k, (mid, _, fac) in enumerate(O.build_models((7, 6, 5), [1, 2, 3], 2, seed=1)):
        assert mid == str(g[f"model{k}_id"])
        for n, f in enumerate(fac):
            assert np.array_equal(f, g[f"model{k}_f{n}"])


def _check_run(name, dims, data, models, tol, iters, r_star, fac_tol=1e-9):
    g = load(f"run_{name}.npz")
    trace = []
    with np.errstate(invalid="ignore"):
        out = O.run_cals(data, dims, models, tol, iters, r_star, trace=trace)
    assert [r.id for r in out] == [str(s) for s in g["order"]]
    assert [r.status for r in out] == [str(s) for s in g["status"]]
    assert [r.iterations for r in out] == g["iterations"].tolist()
    assert [t["width"] for t in trace] == g["widths"].tolist()
    for r, f in zip(out, g["fit"]):
        if np.isfinite(f):
            assert abs(r.fit - f) <= 1e-10
    for r in out:
        key = f"{r.id}_f0"
        if key in g.files and r.status != "failed":
            for n in range(len(dims)):
                assert rel(r.factors[n], g[f"{r.id}_f{n}"]) <= fac_tol, (r.id, n)


def test_run_small_fixed_and_refill():
    dims, data = O.generate_synthetic((12, 10, 8), 3, 0.1, seed=0)
    models = O.build_models(dims, [1, 2, 3, 4], 2, seed=1)
    _check_run("small_fixed5", dims, data, models, 0.0, 5, sum(m[1] for m in models))
    _check_run("small_refill", dims, data, O.build_models(dims, [1, 2, 3, 4], 2, seed=1), 1e-6, 200, 6,
               fac_tol=1e-6)


def test_run_c1():
    dims, data = O.generate_synthetic((50, 50, 50), 5, 0.1, seed=0)
    meta = json.load(open(os.path.join(GOLDEN, "meta.json")))
    import hashlib
    assert hashlib.sha256(np.ascontiguousarray(data, "<f8").tobytes()).hexdigest() == meta["c1_tensor_sha256"]
    _check_run("c1_fixed5", dims, data, O.build_models(dims, [1, 2, 3, 4, 5], 4, seed=1), 0.0, 5, 60)
    _check_run("c1_tol", dims, data, O.build_models(dims, [1, 2, 3, 4, 5], 4, seed=1), 1e-6, 1000, 60)


def test_run_line_search():
    dims, data = O.generate_synthetic((12, 10, 8), 3, 0.1, seed=0)
    for name, ranks, seed, r_star, alpha in [("ls_cube_root", [1, 2, 3, 4], 1, 20, None),
                                             ("ls_const", [2, 3], 7, 6, 1.5)]:
        g = load(f"run_{name}.npz")
        out = O.run_cals(data, dims, O.build_models(dims, ranks, 2, seed=seed), 0.0, 8, r_star,
                         ls=True, ls_alpha=alpha)
        assert [r.id for r in out] == [str(s) for s in g["order"]]
        for r in out:
            for n in range(3):
                assert rel(r.factors[n], g[f"{r.id}_f{n}"]) <= 1e-9


def test_run_other_orders_and_failure():
    dims, data = O.generate_synthetic((9, 7), 2, 0.05, seed=3)
    _check_run("order2", dims, data, O.build_models(dims, [1, 2, 3], 2, seed=4), 0.0, 6, 12)
    dims, data = O.generate_synthetic((5, 4, 6, 3), 2, 0.05, seed=5)
    _check_run("order4", dims, data, O.build_models(dims, [1, 2, 3], 2, seed=6), 0.0, 6, 12)
    f = load("fail_inputs.npz")
    models = [("bad", 2, [f[f"bad_f{n}"] for n in range(3)]), ("good", 2, [f[f"good_f{n}"] for n in range(3)])]
    _check_run("fail", (4, 4, 3), f["data"], models, 0.0, 3, 4)


def test_oracle_c2_benchmark_config_matches_reference():
    """configs[1] as the bench times it (200^3, 200 models, 5 iterations,
    r_star 2100): the oracle against the reference's own run
    (run_c2_fixed5.npz, oracle/make_golden_configs.py) -- so the GPU test that
    compares all 200 models with the oracle is anchored to the reference."""
    g = load("run_c2_fixed5.npz")
    dims, data = O.generate_synthetic((200, 200, 200), 20, 0.1, seed=0)
    models = O.build_models(dims, list(range(1, 21)), 10, seed=1)
    out = O.run_cals(data, dims, models, 0.0, 5, 2100)
    assert [r.id for r in out] == [str(s) for s in g["order"]]
    assert [r.iterations for r in out] == g["iterations"].tolist()
    for r, f in zip(out, g["fit"]):
        assert abs(r.fit - f) <= 1e-12
        if f"{r.id}_f0" in g.files:
            for n in range(3):
                assert rel(r.factors[n], g[f"{r.id}_f{n}"]) <= 1e-11, (r.id, n)
