"""Generate the golden fixtures in tests/golden/ from the REAL reference.

Run in the build container only (it imports /root/reference/pkg/src, which
does not exist on the GPU box):

    python oracle/make_golden.py

The fixtures pin both the numpy oracle (oracle/cals_oracle.py) and the CUDA
path.  Everything is seeded; re-running reproduces the files bit for bit on
the same numpy/scipy build.  TEST INFRASTRUCTURE ONLY.
"""

from __future__ import annotations

import hashlib
import json
import os
import sys

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def _ref():
    sys.path.insert(0, REF)
    import cals  # noqa: F401  (the unmodified reference package)
    return cals


def sha(a: np.ndarray) -> str:
    return hashlib.sha256(np.ascontiguousarray(a, dtype="<f8").tobytes()).hexdigest()


def main() -> None:
    cals = _ref()
    from cals.driver import ExecutionMode, SegmentTrace, run
    from cals.io import build_models, generate_synthetic
    from cals.model import Model
    from cals.mttkrp import MttkrpWorkspace, mttkrp
    from cals.als import ConvergenceConfig, update_factor, fast_error, fit_from_error
    from cals.tensor import DenseTensor, gramian, khatri_rao

    os.makedirs(OUT, exist_ok=True)
    meta: dict = {"reference": "arxiv/paper_2010_04678 pkg/src/cals",
                  "numpy": np.__version__, "cases": {}}

    # ---- 1. known-answer tests (test_mttkrp.py:43-47, test_tensor.py:87-90, test_als.py:28-30)
    kat = {}
    t = DenseTensor((2, 2, 2), np.arange(1.0, 9.0))
    ones = np.ones((2, 1), order="F")
    kat["mttkrp_2x2x2_mode0"] = np.array(mttkrp(t, [ones, ones, ones], 0)).ravel()
    kat["krp_12_345"] = khatri_rao(np.array([[1.0], [2.0]]), np.array([[3.0], [4.0], [5.0]])).ravel()
    kat["update_16_20_over_4"] = update_factor(np.array([[16.0], [20.0]]), np.array([[4.0]])).ravel()
    np.savez(os.path.join(OUT, "kat.npz"), **kat)

    # ---- 2. MTTKRP per mode, orders 2..5 (default variant table)
    mt = {}
    shapes = [((4, 3, 2), 3), ((7, 9, 5), 5), ((6, 5, 4), 8), ((13, 11, 9), 7),
              ((16, 2), 3), ((3, 4, 5, 2), 2), ((2, 3, 2, 2, 2), 4), ((21, 10, 3), 33)]
    rng = np.random.default_rng(2024)
    for ci, (dims, w) in enumerate(shapes):
        arr = rng.standard_normal(dims)
        tt = DenseTensor.from_array(arr)
        fac = [np.asfortranarray(rng.standard_normal((d, w))) for d in dims]
        ws = MttkrpWorkspace(dims, w)
        mt[f"c{ci}_dims"] = np.array(dims)
        mt[f"c{ci}_data"] = tt.data.copy()
        for n, f in enumerate(fac):
            mt[f"c{ci}_f{n}"] = f
            mt[f"c{ci}_m{n}"] = np.array(mttkrp(tt, fac, n, ws=ws))
    mt["n_cases"] = np.array(len(shapes))
    np.savez(os.path.join(OUT, "mttkrp.npz"), **mt)

    # ---- 3. factor updates incl. the singular / pinv branch
    up = {}
    rng = np.random.default_rng(77)
    cases = []
    for r, rows in [(1, 5), (3, 7), (5, 11), (8, 4), (20, 30)]:
        a = rng.standard_normal((rows + r, r))
        h = gramian(a)
        m = rng.standard_normal((rows, r))
        cases.append((m, h))
    cases.append((np.array([[2.0, 2.0]]), np.array([[1.0, 1.0], [1.0, 1.0]])))  # singular
    v = rng.standard_normal((4, 2))
    cases.append((rng.standard_normal((6, 4)), v @ v.T))  # rank-deficient 4x4
    for i, (m, h) in enumerate(cases):
        up[f"u{i}_m"], up[f"u{i}_h"] = m, h
        up[f"u{i}_a"] = update_factor(m, h)
    up["n_cases"] = np.array(len(cases))
    # fast error / fit known values
    rng = np.random.default_rng(78)
    dims = (5, 4, 3)
    arr = rng.standard_normal(dims)
    tt = DenseTensor.from_array(arr)
    fac = [np.asfortranarray(rng.standard_normal((d, 2))) for d in dims]
    ml = np.array(mttkrp(tt, fac, 2))
    grams = [gramian(f) for f in fac]
    up["fe_data"] = tt.data.copy()
    for n, f in enumerate(fac):
        up[f"fe_f{n}"] = f
    up["fe_error"] = np.array(fast_error(tt.sqnorm, fac, ml, grams))
    up["fe_fit"] = np.array(fit_from_error(float(up["fe_error"]), tt.sqnorm))
    np.savez(os.path.join(OUT, "update.npz"), **up)

    # ---- 4. input builders are reproduced bit for bit
    gb = {}
    t0 = generate_synthetic((7, 6, 5), 3, 0.1, seed=0)
    gb["synth_7x6x5"] = t0.data.copy()
    for k, m in enumerate(build_models((7, 6, 5), [1, 2, 3], per_rank=2, seed=1)):
        gb[f"model{k}_id"] = np.array(m.id)
        for n, f in enumerate(m.factors):
            gb[f"model{k}_f{n}"] = f
    np.savez(os.path.join(OUT, "builders.npz"), **gb)
    c1 = generate_synthetic((50, 50, 50), 5, 0.1, seed=0)
    meta["c1_tensor_sha256"] = sha(c1.data)
    eem = generate_synthetic((250, 251, 21), 10, 0.1, seed=0)
    meta["c3_tensor_sha256"] = sha(eem.data)
    c2 = generate_synthetic((200, 200, 200), 20, 0.1, seed=0)
    meta["c2_tensor_sha256"] = sha(c2.data)
    meta["c2_models_sha256"] = sha(np.concatenate(
        [f.ravel(order="F") for m in build_models(c2.dims, list(range(1, 21)), 10, seed=1)
         for f in m.factors]))

    # ---- 5. full CALS runs through the reference driver
    def run_case(name, tensor, models, tol, iters, r_star, keep_factors=True):
        trace: list = []
        out = run(tensor, models, ConvergenceConfig(tol=tol, max_iterations=iters),
                  mode=ExecutionMode.CALS, r_star=r_star, trace=trace)
        d = {"order": np.array([m.id for m in out]),
             "status": np.array([m.status.value for m in out]),
             "iterations": np.array([m.iterations_done for m in out]),
             "fit": np.array([m.fit for m in out]),
             "error": np.array([m.error for m in out]),
             "widths": np.array([s.meta["width"] for s in trace]),
             "n_active": np.array([s.meta["n_active"] for s in trace])}
        if keep_factors:
            for m in out:
                for n, f in enumerate(m.factors):
                    d[f"{m.id}_f{n}"] = f
        np.savez(os.path.join(OUT, f"run_{name}.npz"), **d)
        meta["cases"][name] = {"dims": list(tensor.dims), "tol": tol, "max_iterations": iters,
                               "r_star": r_star, "n_models": len(models)}

    small = generate_synthetic((12, 10, 8), 3, 0.1, seed=0)
    ms = build_models(small.dims, [1, 2, 3, 4], per_rank=2, seed=1)
    run_case("small_fixed5", small, ms, 0.0, 5, sum(m.rank for m in ms))
    run_case("small_refill", small, build_models(small.dims, [1, 2, 3, 4], per_rank=2, seed=1),
             1e-6, 200, 6)
    c1m = build_models(c1.dims, [1, 2, 3, 4, 5], per_rank=4, seed=1)
    run_case("c1_fixed5", c1, c1m, 0.0, 5, 60)
    run_case("c1_tol", c1, build_models(c1.dims, [1, 2, 3, 4, 5], per_rank=4, seed=1),
             1e-6, 1000, 60, keep_factors=False)
    o2 = generate_synthetic((9, 7), 2, 0.05, seed=3)
    run_case("order2", o2, build_models(o2.dims, [1, 2, 3], per_rank=2, seed=4), 0.0, 6, 12)
    o4 = generate_synthetic((5, 4, 6, 3), 2, 0.05, seed=5)
    run_case("order4", o4, build_models(o4.dims, [1, 2, 3], per_rank=2, seed=6), 0.0, 6, 12)
    # line search in the fused driver (driver.py:250-259, 272-273)
    from cals.als import LineSearchConfig

    def run_ls_case(name, tensor, models, tol, iters, r_star, alpha):
        trace: list = []
        out = run(tensor, models, ConvergenceConfig(tol=tol, max_iterations=iters),
                  mode=ExecutionMode.CALS, r_star=r_star, trace=trace,
                  ls=LineSearchConfig(enabled=True, alpha=alpha))
        d = {"order": np.array([m.id for m in out]),
             "status": np.array([m.status.value for m in out]),
             "iterations": np.array([m.iterations_done for m in out]),
             "fit": np.array([m.fit for m in out]), "error": np.array([m.error for m in out]),
             "widths": np.array([s.meta["width"] for s in trace]),
             "n_active": np.array([s.meta["n_active"] for s in trace])}
        for m in out:
            for n, f in enumerate(m.factors):
                d[f"{m.id}_f{n}"] = f
        np.savez(os.path.join(OUT, f"run_{name}.npz"), **d)
        meta["cases"][name] = {"dims": list(tensor.dims), "tol": tol, "max_iterations": iters,
                               "r_star": r_star, "ls_alpha": alpha}

    run_ls_case("ls_cube_root", small, build_models(small.dims, [1, 2, 3, 4], 2, seed=1),
                0.0, 8, 20, None)
    run_ls_case("ls_const", small, build_models(small.dims, [2, 3], 2, seed=7), 0.0, 8, 6, 1.5)
    run_ls_case("ls_c1_tol", c1, build_models(c1.dims, [1, 2, 3, 4, 5], 4, seed=1),
                1e-6, 1000, 60, None)

    # non-negative updates (driver.py:226-227, als.py:185-278)
    from cals.als import nnls_solve_row

    def run_nn_case(name, tensor, models, tol, iters, r_star, ls_on=False):
        trace: list = []
        out = run(tensor, models, ConvergenceConfig(tol=tol, max_iterations=iters),
                  mode=ExecutionMode.CALS, r_star=r_star, trace=trace, nonneg=True,
                  ls=LineSearchConfig(enabled=ls_on))
        d = {"order": np.array([m.id for m in out]),
             "status": np.array([m.status.value for m in out]),
             "iterations": np.array([m.iterations_done for m in out]),
             "fit": np.array([m.fit for m in out]), "error": np.array([m.error for m in out]),
             "widths": np.array([s.meta["width"] for s in trace]),
             "n_active": np.array([s.meta["n_active"] for s in trace])}
        for m in out:
            for n, f in enumerate(m.factors):
                d[f"{m.id}_f{n}"] = f
        np.savez(os.path.join(OUT, f"run_{name}.npz"), **d)
        meta["cases"][name] = {"dims": list(tensor.dims), "tol": tol, "max_iterations": iters,
                               "r_star": r_star, "nonneg": True, "ls": ls_on}

    run_nn_case("nn_fixed", small, build_models(small.dims, [1, 2, 3, 4], 2, seed=1), 0.0, 8, 20)
    run_nn_case("nn_tol", small, build_models(small.dims, [2, 3], 2, seed=2), 1e-6, 300, 6)
    rng = np.random.default_rng(67)
    ldims = (6, 5, 4)
    truth = [rng.random((d, 2)) for d in ldims]
    lt = DenseTensor.from_array(np.einsum("ir,jr,kr->ijk", *truth))
    lmodels = [Model.random(ldims, 2, rng, id=f"m{i}") for i in range(3)]
    nn_in = {"data": lt.data.copy()}
    for i, m in enumerate(lmodels):
        for n in range(3):
            nn_in[f"m{i}_f{n}"] = m.factors[n].copy()
    np.savez(os.path.join(OUT, "nn_ls_inputs.npz"), **nn_in)
    run_nn_case("nn_ls", lt, lmodels, 1e-7, 300, 6, ls_on=True)
    rows = {}
    rng = np.random.default_rng(99)
    cnt = 0
    for r in (1, 3, 8, 20):
        for _ in range(12):
            a = rng.standard_normal((r + 5, r))
            h = a.T @ a
            f = rng.standard_normal(r) * 2.0
            act = rng.random(r) < 0.3
            x, newact, conv = nnls_solve_row(h, f, act)
            rows.update({f"p{cnt}_h": h, f"p{cnt}_f": f, f"p{cnt}_act": act, f"p{cnt}_x": x,
                         f"p{cnt}_newact": newact, f"p{cnt}_conv": np.array(conv)})
            cnt += 1
    rows["n_cases"] = np.array(cnt)
    np.savez(os.path.join(OUT, "nnls_rows.npz"), **rows)

    # failure isolation (test_driver.py:117-135)
    rng = np.random.default_rng(66)
    fd = (4, 4, 3)
    ft = DenseTensor.from_array(rng.standard_normal(fd))
    bad = Model.random(fd, 2, rng, id="bad")
    bad.factors[-1][0, 0] = np.nan
    good = Model.random(fd, 2, rng, id="good")
    fail_in = {"data": ft.data.copy()}
    for n in range(3):
        fail_in[f"bad_f{n}"] = bad.factors[n].copy()
        fail_in[f"good_f{n}"] = good.factors[n].copy()
    np.savez(os.path.join(OUT, "fail_inputs.npz"), **fail_in)
    with np.errstate(invalid="ignore"):
        run_case("fail", ft, [bad, good], 0.0, 3, 4)

    with open(os.path.join(OUT, "meta.json"), "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)
    print("wrote", sorted(os.listdir(OUT)))


if __name__ == "__main__":
    main()
