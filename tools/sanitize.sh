#!/bin/bash
# compute-sanitizer over a small engine + operator workload (memcheck, racecheck, synccheck)
set -u
cd "$(dirname "$0")/.."
cat > /tmp/san_work.py <<'PY'
import sys; sys.path.insert(0, ".")
import numpy as np
import paper_2010_04678_b200 as cals
t = cals.generate_synthetic((13, 10, 9), 3, 0.1, seed=0)
ms = cals.build_models(t.dims, [1, 2, 3, 5], 2, seed=1)
cals.run(t, ms, cals.ConvergenceConfig(tol=1e-6, max_iterations=20), r_star=8)
cals.run(t, ms, cals.ConvergenceConfig(tol=0.0, max_iterations=3), r_star=30,
         ls=cals.LineSearchConfig(enabled=True), nonneg=True)
f = [np.random.default_rng(0).random((d, 5)) for d in t.dims]
for n in range(3):
    cals.mttkrp(t, f, n)
cals.update_factor(np.ones((4, 2)), np.array([[2.0, 1.0], [1.0, 2.0]]))
print("workload ok")
PY
for tool in memcheck racecheck synccheck; do
  echo "== $tool"
  CALS_TREE=1 compute-sanitizer --tool $tool --print-limit 20 python /tmp/san_work.py 2>&1 | tail -30
done
