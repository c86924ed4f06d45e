"""GPU parity of the fused MTTKRP (csrc/mttkrp.cuh) through the C ABI.

Checked against the golden vectors of the real reference and against the
numpy oracle (oracle/cals_oracle.py) on seeded inputs; the tolerance is the
reference's own (test_mttkrp.py:64-78: 1e-12 relative Frobenius).
"""
import os

import numpy as np
import pytest

from conftest import GOLDEN

pytestmark = pytest.mark.gpu

TOL = 1e-12


@pytest.fixture(scope="module")
def cals():
    import paper_2010_04678_b200 as c

    c._native.load()
    return c


def rel(a, b):
    return np.linalg.norm(np.asarray(a) - np.asarray(b)) / max(np.linalg.norm(b), 1e-300)


def test_known_answer_2x2x2(cals):
    t = cals.DenseTensor((2, 2, 2), np.arange(1.0, 9.0))
    ones = np.ones((2, 1), order="F")
    assert cals.mttkrp(t, [ones, ones, ones], 0).ravel().tolist() == [16.0, 20.0]


def test_golden_all_orders(cals):
    g = np.load(os.path.join(GOLDEN, "mttkrp.npz"))
    for ci in range(int(g["n_cases"])):
        dims = tuple(int(d) for d in g[f"c{ci}_dims"])
        t = cals.DenseTensor(dims, g[f"c{ci}_data"])
        fac = [g[f"c{ci}_f{n}"] for n in range(len(dims))]
        ws = cals.MttkrpWorkspace(dims, fac[0].shape[1])
        for n in range(len(dims)):
            got = np.array(cals.mttkrp(t, fac, n, ws=ws))
            assert rel(got, g[f"c{ci}_m{n}"]) <= TOL, (ci, dims, n, rel(got, g[f"c{ci}_m{n}"]))


@pytest.mark.parametrize("dims,width", [
    ((3, 5, 4), 1), ((5, 4, 3), 7), ((17, 33, 9), 40), ((50, 50, 50), 60),
    ((251, 250, 21), 37), ((21, 13, 250), 19), ((64, 48, 80), 130), ((9, 7), 5),
    ((4, 3, 5, 2), 6), ((3, 4, 2, 5, 2), 3)])
def test_random_vs_oracle(cals, dims, width):
    from oracle import cals_oracle as O

    rng = np.random.default_rng(sum(dims) * 7 + width)
    arr = rng.standard_normal(dims)
    t = cals.DenseTensor.from_array(arr)
    fac = [np.asfortranarray(rng.standard_normal((d, width))) for d in dims]
    ws = cals.MttkrpWorkspace(dims, width)
    for n in range(len(dims)):
        want = O.mttkrp(t.data, dims, fac, n)
        got = np.array(cals.mttkrp(t, fac, n, ws=ws))
        assert rel(got, want) <= TOL, (dims, n, rel(got, want))


def test_all_variants_agree_bitwise(cals):
    """Every tile-shape variant runs the same accumulation order."""
    import ctypes as C
    import torch

    rng = np.random.default_rng(5)
    dims, width = (37, 29, 23), 45
    t = cals.DenseTensor.from_array(rng.standard_normal(dims))
    fac = [torch.from_numpy(rng.standard_normal((d, 48))).cuda() for d in dims]
    cnt = C.c_int()
    cals._native.call("cals_mttkrp_variants", C.byref(cnt))
    ptrs = (C.c_void_p * 3)(*[f.data_ptr() for f in fac])
    for n in range(3):
        b = C.c_size_t()
        cals._native.call("cals_mttkrp_workspace_bytes", t.device().handle, n, 48, C.byref(b))
        work = torch.empty(b.value // 8 + 1, dtype=torch.float64, device="cuda")
        outs = []
        for v in range(cnt.value):
            out = torch.zeros((dims[n], 48), dtype=torch.float64, device="cuda")
            cals._native.call("cals_mttkrp", t.device().handle, n, width, ptrs, 48,
                              out.data_ptr(), 48, work.data_ptr(), b.value, v,
                              torch.cuda.current_stream().cuda_stream)
            outs.append(out[:, :width].cpu().numpy())
        for o in outs[1:]:
            assert np.array_equal(o, outs[0]), n


def test_fused_position_independence(cals):
    """Duplicated instances give exactly equal columns (test_mttkrp.py:164-173)
    and K=1 equals the fused slice bitwise at any offset (test_mttkrp.py:176-187)."""
    rng = np.random.default_rng(23)
    dims = (45, 38, 29)
    t = cals.DenseTensor.from_array(rng.standard_normal(dims))
    models = [cals.Model.random(dims, r, rng, id=f"m{i}") for i, r in enumerate([3, 7, 1, 5, 11])]
    twin = cals.Model(id="twin", rank=5, factors=models[3].copy_factors())
    mms = cals.MultiMatrixSet(dims, 64)
    for m in models + [twin]:
        assert mms.try_insert(m)
    ws = cals.MttkrpWorkspace(dims, 64)
    for n in range(3):
        fused = np.array(cals.fused_mttkrp(t, mms.per_mode, n, ws))
        e3, et = mms.per_mode[0].entry("m3"), mms.per_mode[0].entry("twin")
        assert np.array_equal(fused[:, e3.offset:e3.offset + 5], fused[:, et.offset:et.offset + 5])
        for m in models:
            e = mms.per_mode[0].entry(m.id)
            single = np.array(cals.mttkrp(t, m.factors, n, ws=cals.MttkrpWorkspace(dims, m.rank)))
            assert np.array_equal(single, fused[:, e.offset:e.offset + m.rank]), (n, m.id)


def test_errors(cals):
    rng = np.random.default_rng(0)
    t = cals.DenseTensor.from_array(rng.standard_normal((4, 3, 2)))
    f = [np.ones((4, 2)), np.ones((3, 2)), np.ones((2, 2))]
    with pytest.raises(ValueError):
        cals.mttkrp(t, [np.zeros((5, 2)), f[1], f[2]], 1)
    with pytest.raises(ValueError):
        cals.mttkrp(t, [f[0], np.zeros((3, 3)), f[2]], 0)
    with pytest.raises(ValueError, match="capacity"):
        cals.mttkrp(t, [np.ones((4, 3)), np.ones((3, 3)), np.ones((2, 3))], 0,
                    ws=cals.MttkrpWorkspace((4, 3, 2), 2))
    with pytest.raises(ValueError):
        cals.mttkrp(t, f, 1, variant=cals.MttkrpVariant.FIRST_MODE_GEMM)


def test_concurrent_callers(cals):
    from concurrent.futures import ThreadPoolExecutor

    from oracle import cals_oracle as O

    dims = (12, 10, 8)
    rng = np.random.default_rng(26)
    t = cals.DenseTensor.from_array(rng.standard_normal(dims))
    jobs = []
    for seed in range(8):
        r = np.random.default_rng(seed)
        jobs.append(([np.asfortranarray(r.standard_normal((d, 3))) for d in dims], seed % 3,
                     cals.MttkrpWorkspace(dims, 3)))

    def work(job):
        fac, mode, ws = job
        return np.array(cals.mttkrp(t, fac, mode, ws=ws)), O.mttkrp(t.data, dims, fac, mode)

    with ThreadPoolExecutor(max_workers=4) as ex:
        for got, want in ex.map(work, jobs * 3):
            assert rel(got, want) <= TOL


@pytest.mark.slow
def test_c2_scale_column_subset(cals):
    """200^3 at W = 2100 (config 2): the MTTKRP is column-separable, so a
    random subset of 48 columns is checked against the oracle."""
    from oracle import cals_oracle as O

    t = cals.generate_synthetic((200, 200, 200), 20, 0.1, seed=0)
    ms = cals.build_models(t.dims, list(range(1, 21)), 10, seed=1)
    mms = cals.MultiMatrixSet(t.dims, 2100)
    for m in ms:
        assert mms.try_insert(m)
    ws = cals.MttkrpWorkspace(t.dims, 2100)
    cols = np.sort(np.random.default_rng(0).choice(2100, 48, replace=False))
    for n in range(3):
        fused = np.array(cals.fused_mttkrp(t, mms.per_mode, n, ws))
        sub = [mm.packed_view()[:, cols] for mm in mms.per_mode]
        want = O.mttkrp(t.data, t.dims, sub, n)
        assert rel(fused[:, cols], want) <= TOL
