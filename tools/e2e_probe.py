import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2010_04678_b200 as cals
from paper_2010_04678_b200.driver import LAST_RUN_PROFILE
dims = (200, 200, 200)
t = cals.generate_synthetic(dims, 20, 0.1, seed=0)
models = cals.build_models(dims, list(range(1, 21)), 10, seed=1)
t.pin()
for i in range(int(sys.argv[1]) if len(sys.argv) > 1 else 6):
    tt = cals.DenseTensor(dims, t.data)
    torch.cuda.synchronize()
    tic = time.perf_counter()
    out = cals.run(tt, models, cals.ConvergenceConfig(tol=0.0, max_iterations=5), r_star=2100)
    torch.cuda.synchronize()
    print(f"run {i}: {1e3*(time.perf_counter()-tic):.2f} ms", {k: round(1e3*v, 2) for k, v in LAST_RUN_PROFILE.items()})
    tt.release_device()
