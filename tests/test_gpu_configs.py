"""End-to-end parity at the configurations the bench times (BASELINE.json
configs[1..3]), on the kernels the bench uses (INT8 Ozaki MTTKRP, default
dimension tree, bucketed update kernel), through the public ``run()``.

north_star bar: factors within 1e-9 relative Frobenius after a fixed 5
iterations; final fit within 1e-6 with equal converged iteration counts.
References: the real reference package's outputs on the same inputs
(``tests/golden/run_c2_fixed5.npz`` / ``run_c3_full.npz``, written by
``oracle/make_golden_configs.py``) and, for every c2 model, the numpy oracle
run on the box.  Match: reference driver.py:185-285 (loop), :266-271
(stopping rule).
"""
import ctypes as C
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
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def kernel_kinds(cals, t, width):
    out = []
    for n in range(t.order):
        k, ops = C.c_int32(), C.c_double()
        cals._native.call("cals_mttkrp_kernel_info", t.device().handle, n, width, C.byref(k),
                          C.byref(ops))
        out.append(int(k.value))
    return out


def _check_structure(out, g, trace=None):
    assert [m.id for m in out] == [str(s) for s in g["order"]]
    assert [m.status.value for m in out] == [str(s) for s in g["status"]]
    assert [m.iterations_done for m in out] == g["iterations"].tolist()
    if trace is not None:
        assert [s.meta["width"] for s in trace] == g["widths"].tolist()
        assert [s.meta["n_active"] for s in trace] == g["n_active"].tolist()


@pytest.mark.slow
def test_c2_full_sweep(cals):
    """configs[1] exactly as bench.py times it: 200^3, 200 models (ranks
    1..20 x 10), tol 0, 5 iterations, r_star 2100, INT8 MTTKRP for every mode."""
    from oracle import cals_oracle as O

    g = np.load(os.path.join(GOLDEN, "run_c2_fixed5.npz"))
    t = cals.generate_synthetic((200, 200, 200), 20, 0.1, seed=0)
    assert kernel_kinds(cals, t, 2100) == [1, 1, 1]  # the bench's kernels
    ms = cals.build_models(t.dims, list(range(1, 21)), 10, seed=1)
    trace = []
    out = cals.run(t, ms, cals.ConvergenceConfig(tol=0.0, max_iterations=5), r_star=2100,
                   trace=trace)
    _check_structure(out, g, trace)
    worst_ref = 0.0
    for m, f in zip(out, g["fit"]):
        assert abs(m.fit - f) <= 1e-9, (m.id, m.fit, f)
        if f"{m.id}_f0" in g.files:  # the 20 models the fixture keeps factors for
            for n in range(3):
                worst_ref = max(worst_ref, rel(m.factors[n], g[f"{m.id}_f{n}"]))
    assert worst_ref <= 1e-9, worst_ref
    # every model against the numpy oracle on the same inputs
    om = [(m.id, m.rank, m.factors) for m in cals.build_models(t.dims, list(range(1, 21)), 10,
                                                              seed=1)]
    ref = O.run_cals(t.data, t.dims, om, 0.0, 5, 2100)
    assert [r.id for r in ref] == [m.id for m in out]
    worst = 0.0
    for m, r in zip(out, ref):
        assert m.iterations_done == r.iterations == 5
        assert abs(m.fit - r.fit) <= 1e-9
        for n in range(3):
            worst = max(worst, rel(m.factors[n], r.factors[n]))
    assert worst <= 1e-9, worst


@pytest.mark.slow
def test_c3_full_sweep(cals):
    """configs[2] exactly as ``bench.py --config c3`` times it: 250x251x21,
    180 models (ranks 2..10 x 20), tol 1e-6, cap 1000, r_star 300
    (converged-slot refill): identical statuses, retirement order, iteration
    counts and per-iteration widths / active counts; |dfit| <= 1e-6."""
    g = np.load(os.path.join(GOLDEN, "run_c3_full.npz"))
    t = cals.generate_synthetic((250, 251, 21), 10, 0.1, seed=0)
    ms = cals.build_models(t.dims, list(range(2, 11)), 20, seed=1)
    trace = []
    out = cals.run(t, ms, cals.ConvergenceConfig(tol=1e-6, max_iterations=1000), r_star=300,
                   trace=trace)
    _check_structure(out, g, trace)
    dfit = max(abs(m.fit - f) for m, f in zip(out, g["fit"]))
    assert dfit <= 1e-6, dfit


@pytest.mark.slow
def test_c4_shape_contraction(cals):
    """configs[3] shape: 500^3 at the full width W = 5250 (INT8, Kp = 512).
    Column-separable, so 64 columns spread over the width are checked
    against an FP64 numpy contraction (reference tolerance 1e-12)."""
    import torch

    dims, W = (500, 500, 500), 5250
    rng = np.random.default_rng(4)
    data = rng.random(int(np.prod(dims)))
    t = cals.DenseTensor(dims, data)
    assert kernel_kinds(cals, t, W) == [1, 1, 1]
    fac = [np.asfortranarray(rng.random((d, W))) for d in dims]
    ws = cals.MttkrpWorkspace(dims, W)
    cols = np.sort(np.random.default_rng(1).choice(W, 64, replace=False))
    x = data.reshape(dims, order="F")
    sub = [f[:, cols] for f in fac]
    want = [np.einsum("ijk,jr,kr->ir", x, sub[1], sub[2], optimize=True),
            np.einsum("ijk,ir,kr->jr", x, sub[0], sub[2], optimize=True),
            np.einsum("ijk,ir,jr->kr", x, sub[0], sub[1], optimize=True)]
    for n in range(3):
        got = np.array(cals.mttkrp(t, fac, n, ws=ws))[:, cols]
        assert rel(got, want[n]) <= 1e-12, (n, rel(got, want[n]))
    del ws
    t.release_device()
    torch.cuda.empty_cache()


@pytest.mark.parametrize("dims,modes", [((2048, 136, 40), (1, 2)), ((136, 2040, 40), (0,)),
                                        ((2000, 130, 48), (1, 2))])
def test_int8_long_contraction_edge(cals, dims, modes):
    """The INT8 kernel's contraction-length limit (Kp <= 2048: 7 products of
    8-bit slices per group accumulate exactly in int32).  Random data and the
    worst case for the accumulators -- every entry just below a power of two,
    so every slice is at its maximum -- against the oracle at 1e-12."""
    from oracle import cals_oracle as O

    rng = np.random.default_rng(sum(dims))
    W = 40
    for kind in ("random", "saturated"):
        if kind == "random":
            arr = rng.standard_normal(dims)
            fac = [np.asfortranarray(rng.standard_normal((d, W))) for d in dims]
        else:
            v = 1.0 - 2.0 ** -45
            arr = np.full(dims, v)
            fac = [np.asfortranarray(np.full((d, W), v)) for d in dims]
        t = cals.DenseTensor.from_array(arr)
        kinds = kernel_kinds(cals, t, W)
        for n in modes:
            assert kinds[n] == 1, (dims, n, kinds)  # the INT8 path is what is tested
            got = np.array(cals.mttkrp(t, fac, n, ws=cals.MttkrpWorkspace(dims, W)))
            want = O.mttkrp(t.data, dims, fac, n)
            assert rel(got, want) <= 1e-12, (kind, dims, n, rel(got, want))
        t.release_device()
