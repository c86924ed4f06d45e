"""Subprocess body for test_gpu_ozaki.py: the MTTKRP path is chosen once per
process (CALS_MTTKRP = ozaki | dmma), so each path runs in its own process.

Runs the fused MTTKRP on seeded inputs and prints one JSON line of relative
Frobenius errors against a numpy FP64 contraction, plus the bitwise checks
(duplicated columns, column-block position independence)."""
import json
import os
import sys

import numpy as np

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)

import paper_2010_04678_b200 as cals  # noqa: E402


def ref_mttkrp(arr, fac, n):
    letters = "abcdefgh"[:arr.ndim]
    ins = [letters] + [letters[i] + "z" for i in range(arr.ndim) if i != n]
    expr = ",".join(ins) + "->" + letters[n] + "z"
    return np.einsum(expr, arr, *[fac[i] for i in range(arr.ndim) if i != n], optimize=True)


def rel(a, b):
    return float(np.linalg.norm(a - b) / max(np.linalg.norm(b), 1e-300))


def main():
    rng = np.random.default_rng(7)
    out = {"cases": []}
    cases = [((200, 200, 200), 300, "normal"), ((160, 130, 150), 129, "uniform"),
             ((256, 144, 96), 64, "range"), ((150, 140, 20), 1, "normal"),
             ((130, 200, 70), 257, "zeros"), ((140, 136, 132), 40, "nonfinite"),
             ((150, 140, 130), 33, "nonfinite_tensor")]
    for dims, width, kind in cases:
        if kind == "uniform":
            arr = rng.random(dims)
            fac = [rng.random((d, width)) for d in dims]
        else:
            arr = rng.standard_normal(dims)
            fac = [rng.standard_normal((d, width)) for d in dims]
        if kind == "range":  # rows / columns spanning 2^-60 .. 2^60
            arr *= np.exp2(rng.integers(-60, 60, size=(dims[0], 1, 1)))
            for f in fac:
                f *= np.exp2(rng.integers(-40, 40, size=(1, width)))
        if kind == "zeros":  # zero factor columns and a zero tensor slab
            for f in fac:
                f[:, ::5] = 0.0
            arr[:, 3, :] = 0.0
        if kind == "nonfinite":  # NaN / Inf in factor columns (non-finite tensors: DMMA path)
            fac[0][5, 3] = np.nan
            fac[2][7, 11] = np.nan
            fac[1][9, 30] = np.inf
        if kind == "nonfinite_tensor":  # an Inf tensor entry: the view falls back to DMMA
            arr[17, 4, 9] = np.inf
        fac = [np.asfortranarray(f) for f in fac]
        t = cals.DenseTensor.from_array(arr)
        ws = cals.MttkrpWorkspace(dims, width)
        errs = []
        for n in range(len(dims)):
            got = np.array(cals.mttkrp(t, fac, n, ws=ws))
            want = ref_mttkrp(arr, fac, n)
            if kind.startswith("nonfinite"):
                # same non-finite pattern, finite entries within tolerance
                same = bool(np.array_equal(np.isfinite(got), np.isfinite(want)))
                ok = np.isfinite(want)
                errs.append(rel(got[ok], want[ok]) if same else 1.0)
            else:
                errs.append(rel(got, want))
        out["cases"].append({"dims": dims, "width": width, "kind": kind, "rel": errs})

    # bitwise: duplicated columns, and a block of columns at two offsets
    dims = (180, 170, 160)
    arr = rng.standard_normal(dims)
    t = cals.DenseTensor.from_array(arr)
    base = [rng.standard_normal((d, 9)) for d in dims]
    left = [rng.standard_normal((d, 37)) for d in dims]
    right = [rng.standard_normal((d, 150)) for d in dims]
    packed_a = [np.asfortranarray(np.hstack([b, r])) for b, r in zip(base, right)]
    packed_b = [np.asfortranarray(np.hstack([l_, b, b, r])) for l_, b, r in zip(left, base, right)]
    ws_a = cals.MttkrpWorkspace(dims, packed_a[0].shape[1])
    ws_b = cals.MttkrpWorkspace(dims, packed_b[0].shape[1])
    pos, dup = True, True
    for n in range(3):
        ga = np.array(cals.mttkrp(t, packed_a, n, ws=ws_a))[:, :9]
        gb = np.array(cals.mttkrp(t, packed_b, n, ws=ws_b))
        pos &= bool(np.array_equal(ga, gb[:, 37:46]))
        dup &= bool(np.array_equal(gb[:, 37:46], gb[:, 46:55]))
    out["position_independent"] = pos
    out["duplicates_equal"] = dup

    # full CALS sweep vs the CPU oracle (5 fixed iterations, refill via r_star)
    from oracle import cals_oracle as O

    dims, data = O.generate_synthetic((140, 136, 132), 6, 0.1, seed=3)
    models = O.build_models(dims, [2, 3, 5, 6], 2, seed=4)
    ref = O.run_cals(data, dims, models, 0.0, 5, 16)
    t = cals.DenseTensor(dims, data)
    ms = [cals.Model(id=i, rank=r, factors=[f.copy() for f in fac]) for i, r, fac in models]
    res = cals.run(t, ms, cals.ConvergenceConfig(tol=0.0, max_iterations=5), r_star=16)
    worst = 0.0
    for m, r in zip(res, ref):
        assert m.id == r.id
        for a, b in zip(m.factors, r.factors):
            worst = max(worst, rel(a, b))
    out["sweep_factor_rel"] = worst
    print(json.dumps(out))


if __name__ == "__main__":
    main()
