"""Subprocess body for test_gpu_fusion.py: one process per setting of
CALS_FUSE_LO (the Lo-slice fusion of the split update is chosen per engine
run).  Prints a JSON line of SHA-256 digests of the factors, fits and
iteration counts of two sweeps whose first contraction after mode 0 runs on
the INT8 path with F[0] as its Lo operand: a Y-tree cube (the mode-2 LAST
contraction takes A0) and an EEM-shaped converging refill sweep (the Z-tree
mode-1 contraction takes A0)."""
import hashlib
import json
import os
import sys

import numpy as np

HERE = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, os.path.dirname(HERE))

import paper_2010_04678_b200 as cals  # noqa: E402


def digest(models) -> str:
    h = hashlib.sha256()
    for m in models:
        for f in m.factors:
            h.update(np.ascontiguousarray(f).tobytes())
        h.update(np.array([m.fit, m.iterations_done], dtype=np.float64).tobytes())
    return h.hexdigest()


def main():
    out = {}
    t = cals.generate_synthetic((200, 180, 160), 8, 0.1, seed=5)
    models = cals.build_models(t.dims, [2, 5, 8, 12], 3, seed=6)
    out["cube"] = digest(cals.run(t, models, cals.ConvergenceConfig(tol=0.0, max_iterations=5)))
    t = cals.generate_synthetic((250, 251, 21), 8, 0.1, seed=7)
    models = cals.build_models(t.dims, [2, 4, 6, 8], 4, seed=8)
    res = cals.run(t, models, cals.ConvergenceConfig(tol=1e-6, max_iterations=200), r_star=30)
    out["eem"] = digest(res)
    out["eem_iters"] = [m.iterations_done for m in res]
    print(json.dumps(out))


if __name__ == "__main__":
    main()
