"""Run-to-run determinism of a converging refill sweep (EEM shape, the
test_eem_shape_refill_vs_oracle workload): the same run() repeated in one
process must give bitwise identical factors / fits / iteration counts /
retirement order; the numpy oracle is run twice as well.
    CALS_MTTKRP=ozaki python tools/determinism_check.py [reps]"""
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402

import paper_2010_04678_b200 as cals  # noqa: E402
from oracle import cals_oracle as O  # noqa: E402

reps = int(sys.argv[1]) if len(sys.argv) > 1 else 8
mix = len(sys.argv) > 2 and sys.argv[2] == "mix"  # other workloads between the repetitions
dims, data = O.generate_synthetic((250, 251, 21), 10, 0.1, seed=0)
models = O.build_models(dims, [2, 4, 6, 8, 10], 2, seed=1)
t = cals.DenseTensor(dims, data)
base = None
other = cals.generate_synthetic((60, 50, 40), 4, 0.1, seed=5)
for i in range(reps):
    if mix and i:
        om = cals.build_models(other.dims, [1, 2, 3, 4, 5], 2 + i % 3, seed=i)
        cals.run(other, om, cals.ConvergenceConfig(tol=1e-5, max_iterations=20 + i),
                 r_star=9 + i % 5)
    ms = [cals.Model(id=m, rank=r, factors=[f.copy() for f in fac]) for m, r, fac in models]
    out = cals.run(t, ms, cals.ConvergenceConfig(tol=1e-6, max_iterations=300), r_star=30)
    sig = ([m.id for m in out], [m.iterations_done for m in out], [m.fit for m in out],
           [np.concatenate([f.ravel() for f in m.factors]) for m in out])
    if base is None:
        base = sig
        print("run 0:", list(zip(sig[0], sig[1])))
        continue
    same = sig[0] == base[0] and sig[1] == base[1] and sig[2] == base[2] and all(
        np.array_equal(a, b) for a, b in zip(sig[3], base[3]))
    print(f"run {i}: bitwise identical to run 0: {same}")
    if not same:
        print("   order/iters:", list(zip(sig[0], sig[1])))
        print("   fit diffs:", [a - b for a, b in zip(sig[2], base[2])])
if "nooracle" in sys.argv:
    sys.exit(0)
r1 = O.run_cals(data, dims, models, 1e-6, 300, 30)
r2 = O.run_cals(data, dims, models, 1e-6, 300, 30)
print("oracle:", [(r.id, r.iterations) for r in r1])
print("oracle run-to-run identical:", [(r.id, r.iterations, r.fit) for r in r1] ==
      [(r.id, r.iterations, r.fit) for r in r2])
print("ours == oracle order/iters:", list(zip(base[0], base[1])) == [(r.id, r.iterations) for r in r1])
