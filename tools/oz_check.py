"""Quick GPU check of the fused MTTKRP path selected by CALS_MTTKRP (default:
Ozaki INT8 tensor cores; CALS_MTTKRP=dmma: FP64 DMMA): relative Frobenius
error vs a numpy FP64 contraction, and per-launch time at the c2 shape."""
import os
import sys
import time

import numpy as np

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import paper_2010_04678_b200 as cals  # noqa: E402


def ref_mttkrp(arr, fac, n):
    order = arr.ndim
    letters = "abcdefgh"[:order]
    ins = [letters] + [letters[i] + "z" for i in range(order) if i != n]
    expr = ",".join(ins) + "->" + letters[n] + "z"
    return np.einsum(expr, arr, *[fac[i] for i in range(order) if i != n], optimize=True)


def main():
    rng = np.random.default_rng(0)
    worst = 0.0
    for dims, width, kind in [((3, 5, 4), 1, "n"), ((17, 33, 9), 40, "n"), ((50, 50, 50), 60, "u"),
                              ((64, 48, 80), 130, "n"), ((251, 250, 21), 37, "u"),
                              ((21, 13, 250), 19, "n"), ((120, 100, 90), 300, "u"),
                              ((4, 3, 5, 2), 6, "n")]:
        arr = rng.standard_normal(dims) if kind == "n" else rng.random(dims)
        fac = [np.asfortranarray(rng.standard_normal((d, width)) if kind == "n"
                                 else rng.random((d, width))) for d in dims]
        t = cals.DenseTensor.from_array(arr)
        ws = cals.MttkrpWorkspace(dims, width)
        for n in range(len(dims)):
            got = np.array(cals.mttkrp(t, fac, n, ws=ws))
            want = ref_mttkrp(arr, fac, n)
            e = np.linalg.norm(got - want) / np.linalg.norm(want)
            worst = max(worst, e)
            print(f"dims={dims} W={width} {kind} mode {n}: rel {e:.2e}", flush=True)
    print(f"WORST {worst:.2e}")


if __name__ == "__main__":
    main()
