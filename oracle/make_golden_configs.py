"""Golden fixtures for the BENCHMARKED configurations, from the REAL reference.

TEST INFRASTRUCTURE ONLY.  Run in the build container (it imports
/root/reference/pkg/src, which does not exist on the GPU box):

    python oracle/make_golden_configs.py [c2] [c3]

* ``run_c2_fixed5.npz`` -- BASELINE.json configs[1] exactly as ``bench.py``
  times it: 200^3 (generate_synthetic rank 20, noise 0.1, seed 0), 200 models
  (build_models ranks 1..20 x 10, seed 1), tol 0, 5 iterations, r_star 2100.
  Per model: retirement order, status, iterations, fit, error; factors of the
  first init of every rank (ids ``rRR-00``, 20 models, ~1 MB) -- the GPU test
  compares all 200 models against the oracle run on the box and these 20
  against the reference itself.
* ``run_c3_full.npz`` -- configs[2] as ``bench.py --config c3`` times it:
  250x251x21 (rank 10, noise 0.1, seed 0), 180 models (ranks 2..10 x 20,
  seed 1), tol 1e-6, cap 1000, r_star 300 (converged-slot refill).  Per model:
  retirement order, status, iterations, fit, error, plus the per-iteration
  trace widths / active counts (driver.py:278-284).
"""

from __future__ import annotations

import json
import os
import sys
import time

import numpy as np

REF = "/root/reference/pkg/src"
OUT = os.path.join(os.path.dirname(os.path.abspath(__file__)), "..", "tests", "golden")


def main(which) -> None:
    sys.path.insert(0, REF)
    from cals.als import ConvergenceConfig
    from cals.driver import ExecutionMode, run
    from cals.io import build_models, generate_synthetic

    meta_path = os.path.join(OUT, "meta_configs.json")
    meta = json.load(open(meta_path)) if os.path.exists(meta_path) else {}

    def record(name, t, models, tol, iters, r_star, keep):
        trace: list = []
        tic = time.perf_counter()
        out = run(t, models, ConvergenceConfig(tol=tol, max_iterations=iters),
                  mode=ExecutionMode.CALS, r_star=r_star, trace=trace)
        sec = time.perf_counter() - tic
        d = {"order": np.array([m.id for m in out]),
             "status": np.array([m.status.value for m in out]),
             "iterations": np.array([m.iterations_done for m in out]),
             "fit": np.array([m.fit for m in out]),
             "error": np.array([m.error for m in out]),
             "widths": np.array([s.meta["width"] for s in trace]),
             "n_active": np.array([s.meta["n_active"] for s in trace])}
        for m in out:
            if keep(m.id):
                for n, f in enumerate(m.factors):
                    d[f"{m.id}_f{n}"] = f
        np.savez_compressed(os.path.join(OUT, f"run_{name}.npz"), **d)
        meta[name] = {"dims": list(t.dims), "tol": tol, "max_iterations": iters,
                      "r_star": r_star, "n_models": len(models), "reference_seconds": sec,
                      "driver_iterations": len(trace), "numpy": np.__version__}
        print(name, f"{sec:.1f} s", len(trace), "driver iterations", flush=True)

    if "c2" in which:
        t = generate_synthetic((200, 200, 200), 20, 0.1, seed=0)
        ms = build_models(t.dims, list(range(1, 21)), 10, seed=1)
        record("c2_fixed5", t, ms, 0.0, 5, 2100, lambda i: i.endswith("-00"))
    if "c3" in which:
        t = generate_synthetic((250, 251, 21), 10, 0.1, seed=0)
        ms = build_models(t.dims, list(range(2, 11)), 20, seed=1)
        record("c3_full", t, ms, 1e-6, 1000, 300, lambda i: False)
    with open(meta_path, "w") as fh:
        json.dump(meta, fh, indent=1, sort_keys=True)


if __name__ == "__main__":
    main(sys.argv[1:] or ["c2", "c3"])
