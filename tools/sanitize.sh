#!/bin/bash
# compute-sanitizer (memcheck, racecheck, synccheck) over two workloads:
#   A: small engine + operator workload (DMMA MTTKRP, NNLS, line search, pinv)
#   B: the INT8 tensor-core MTTKRP (mttkrp_ozaki_kernel, forced) with the
#      Y-tree side output, the Z-tree and the plain schedule, refill on, plus
#      the smoke() shape where the INT8 kernel is picked on its own
# usage: tools/sanitize.sh [outfile]   (full reports; summary lines at the end)
set -u
cd "$(dirname "$0")/.."
OUT=${1:-gpurun_out/sanitize.txt}
mkdir -p "$(dirname "$OUT")"
cat > /tmp/san_a.py <<'PY'
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
print("workload A ok")
PY
cat > /tmp/san_b.py <<'PY'
import ctypes as C, os, sys; sys.path.insert(0, ".")
import numpy as np
import paper_2010_04678_b200 as cals
def kinds(t, w):
    out = []
    for n in range(3):
        k, ops = C.c_int32(), C.c_double()
        cals._native.call("cals_mttkrp_kernel_info", t.device().handle, n, w, C.byref(k), C.byref(ops))
        out.append(int(k.value))
    return out
t = cals.generate_synthetic((70, 66, 68), 4, 0.1, seed=0)
ms = cals.build_models(t.dims, [1, 2, 3, 4, 7], 2, seed=1)
print("forced kinds", kinds(t, 12))
cals.run(t, ms, cals.ConvergenceConfig(tol=1e-6, max_iterations=6), r_star=12)
f = [np.random.default_rng(0).random((d, 9)) for d in t.dims]
for n in range(3):
    cals.mttkrp(t, f, n)
t2 = cals.generate_synthetic((160, 150, 144), 4, 0.1, seed=0)
ms2 = cals.build_models(t2.dims, [1, 2, 3, 4], 2, seed=1)
print("natural kinds", kinds(t2, 12))
cals.run(t2, ms2, cals.ConvergenceConfig(tol=0.0, max_iterations=2), r_star=12)
print("workload B ok, tree", os.environ.get("CALS_TREE"))
PY
: > "$OUT"
for tool in memcheck racecheck synccheck; do
  echo "== $tool A" >> "$OUT"
  CALS_TREE=1 compute-sanitizer --tool $tool --print-limit 50 python /tmp/san_a.py >> "$OUT" 2>&1
  for tree in 1 2 0; do
    echo "== $tool B tree=$tree" >> "$OUT"
    CALS_MTTKRP=ozaki CALS_TREE=$tree compute-sanitizer --tool $tool --print-limit 50 \
      python /tmp/san_b.py >> "$OUT" 2>&1
  done
done
grep -E "^== |SUMMARY|workload|kinds" "$OUT"
