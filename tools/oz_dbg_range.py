import sys, os
sys.path.insert(0, ".")
import numpy as np
import paper_2010_04678_b200 as cals
sys.path.insert(0, "tests")
from _ozaki_worker import ref_mttkrp, rel
rng = np.random.default_rng(7)
dims = (256, 144, 96); width = 64
for variant in ["rows", "cols", "both"]:
    arr = rng.standard_normal(dims)
    fac = [rng.standard_normal((d, width)) for d in dims]
    if variant in ("rows", "both"):
        arr *= np.exp2(rng.integers(-60, 60, size=(dims[0], 1, 1)))
    if variant in ("cols", "both"):
        for f in fac:
            f *= np.exp2(rng.integers(-40, 40, size=(1, width)))
    fac = [np.asfortranarray(f) for f in fac]
    t = cals.DenseTensor.from_array(arr)
    ws = cals.MttkrpWorkspace(dims, width)
    for n in range(3):
        got = np.array(cals.mttkrp(t, fac, n, ws=ws))
        want = ref_mttkrp(arr, fac, n)
        colerr = np.linalg.norm(got - want, axis=0) / np.maximum(np.linalg.norm(want, axis=0), 1e-300)
        print(variant, n, f"rel {rel(got, want):.2e}", "worst cols", np.argsort(colerr)[-3:], colerr[np.argsort(colerr)[-3:]])
