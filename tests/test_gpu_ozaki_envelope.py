"""Accuracy envelope of the INT8 (Ozaki-sliced) tensor-core MTTKRP on data
with within-row dynamic range, and the guard that sends a tensor view to
the FP64 (DMMA) kernel when its rows would lose too many bits.

The INT8 path scales every tensor row (and factor column) by its maximum
and keeps 55 bits below it, so an entry 2^-d below its row maximum keeps
55 - d bits.  Data sets: 1 % of entries spiking by 1e6, log-uniform
magnitudes over 1e-12..1 with random signs, an EEM-like tensor (zero region
below the emission = excitation diagonal, a Rayleigh-scatter ridge 1e4 above
the fluorescence), spiky factor columns.  Bars: the reference's MTTKRP
tolerance (1e-12 relative Frobenius, test_mttkrp.py:64-78) and the
north_star sweep bar (factors 1e-9 after 5 iterations).  The shape
160x150x144 takes the INT8 kernel for every mode on ordinary data.
"""
import ctypes as C
import os

import numpy as np
import pytest

pytestmark = pytest.mark.gpu

DIMS = (160, 150, 144)
# run with CALS_OZ_RANGE_GUARD=0 (test_gpu_forced_ozaki.py) every view takes
# the INT8 kernel, so the bars below then pin the raw INT8 envelope
RAW_INT8 = os.environ.get("CALS_OZ_RANGE_GUARD") == "0"


@pytest.fixture(scope="module")
def cals():
    import paper_2010_04678_b200 as c

    c._native.load()
    return c


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def kinds(cals, t, width):
    out = []
    for n in range(t.order):
        k, ops = C.c_int32(), C.c_double()
        cals._native.call("cals_mttkrp_kernel_info", t.device().handle, n, width, C.byref(k),
                          C.byref(ops))
        out.append(int(k.value))
    return out


def spiky(rng, dims, frac=0.01, factor=1e6):
    x = rng.random(dims)
    mask = rng.random(dims) < frac
    x[mask] *= factor
    return x


def log_uniform(rng, dims):
    return np.exp(rng.uniform(np.log(1e-12), 0.0, dims)) * rng.choice([-1.0, 1.0], dims)


def eem_like(rng, dims):
    """emission x excitation x sample: zero below the diagonal, scatter ridge."""
    em = np.arange(dims[0])[:, None] * (dims[1] / dims[0])
    ex = np.arange(dims[1])[None, :]
    fl = np.einsum("ir,jr,kr->ijk", rng.random((dims[0], 3)), rng.random((dims[1], 3)),
                   rng.random((dims[2], 3)))
    fl[(em < ex - 2)] = 0.0
    ridge = np.abs(em - ex) < 1.5
    fl[ridge] += 1e4 * rng.random((int(ridge.sum()), dims[2]))
    return fl


DATA = {"spiky_1e6": spiky, "log_uniform_1e-12": log_uniform, "eem_like": eem_like}


@pytest.mark.parametrize("name", sorted(DATA))
def test_mttkrp_envelope(cals, name):
    from oracle import cals_oracle as O

    rng = np.random.default_rng(11)
    arr = DATA[name](rng, DIMS)
    t = cals.DenseTensor.from_array(arr)
    W = 48
    facs = {"uniform": [np.asfortranarray(rng.random((d, W))) for d in DIMS],
            "spiky": [np.asfortranarray(spiky(rng, (d, W), 0.02, 1e6)) for d in DIMS]}
    used = kinds(cals, t, W)
    if RAW_INT8:
        assert used == [1, 1, 1]
    for fname, fac in facs.items():
        ws = cals.MttkrpWorkspace(DIMS, W)
        for n in range(3):
            got = np.array(cals.mttkrp(t, fac, n, ws=ws))
            want = O.mttkrp(t.data, DIMS, fac, n)
            assert rel(got, want) <= 1e-12, (name, fname, n, used, rel(got, want))
    t.release_device()


@pytest.mark.parametrize("name", ["spiky_1e6", "eem_like"])
def test_sweep_envelope(cals, name):
    """5 fixed CALS iterations on the hard data against the oracle."""
    from oracle import cals_oracle as O

    rng = np.random.default_rng(12)
    arr = DATA[name](rng, DIMS)
    t = cals.DenseTensor.from_array(arr)
    used = kinds(cals, t, 20)
    if RAW_INT8 or name == "eem_like":
        assert used == [1, 1, 1], used
    models = O.build_models(DIMS, [1, 3, 5, 8], 2, seed=3)
    ref = O.run_cals(t.data, DIMS, models, 0.0, 5, 34)
    ms = [cals.Model(id=i, rank=r, factors=[f.copy() for f in fac]) for i, r, fac in models]
    out = cals.run(t, ms, cals.ConvergenceConfig(tol=0.0, max_iterations=5), r_star=34)
    assert [m.id for m in out] == [r.id for r in ref]
    for m, r in zip(out, ref):
        assert abs(m.fit - r.fit) <= 1e-9
        for a, b in zip(m.factors, r.factors):
            assert rel(a, b) <= 1e-9, (name, used, m.id, rel(a, b))
    t.release_device()


@pytest.mark.skipif(RAW_INT8, reason="guard disabled for the raw INT8 envelope run")
def test_range_guard_sends_view_to_fp64(cals):
    """Rows whose median entry is far below their maximum (each row: one
    entry 1, the others ~1e-9) are not sliced: the FP64 kernel runs, and the
    result meets the reference tolerance.  Ordinary data keeps INT8."""
    from oracle import cals_oracle as O

    rng = np.random.default_rng(13)
    arr = 1e-9 * rng.random(DIMS)
    # one large entry in every mode-0/1/2 row of every view
    idx = rng.integers(0, 10, size=4)
    arr[idx[0], :, :] = 1.0
    arr[:, idx[1], :] = 1.0
    arr[:, :, idx[2]] = 1.0
    t = cals.DenseTensor.from_array(arr)
    assert kinds(cals, t, 16) == [0, 0, 0]
    fac = [np.asfortranarray(rng.random((d, 16))) for d in DIMS]
    for n in range(3):
        got = np.array(cals.mttkrp(t, fac, n, ws=cals.MttkrpWorkspace(DIMS, 16)))
        assert rel(got, O.mttkrp(t.data, DIMS, fac, n)) <= 1e-12
    t.release_device()
    ok = cals.DenseTensor.from_array(rng.random(DIMS))
    assert kinds(cals, ok, 16) == [1, 1, 1]
    ok.release_device()
