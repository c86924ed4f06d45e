"""One converging c3 sweep (EEM 250x251x21, 180 models, tol 1e-6, r_star 300)
through the public run() -- for ncu launch lists of the converging workload."""
import sys

sys.path.insert(0, ".")
import paper_2010_04678_b200 as cals  # noqa: E402

t = cals.generate_synthetic((250, 251, 21), 10, 0.1, seed=0)
models = cals.build_models(t.dims, list(range(2, 11)), 20, seed=1)
res = cals.run(t, models, cals.ConvergenceConfig(tol=1e-6, max_iterations=1000),
               mode=cals.ExecutionMode.CALS, r_star=300)
print("ok", len(res))
