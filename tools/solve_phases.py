"""Phase stamps of the split-update solve kernel inside a sweep (profiling
build: NVCC_APPEND_FLAGS=-DCALS_SOLVE_PROFILE python -m paper_2010_04678_b200._build --force).

usage: python tools/solve_phases.py c2|c3
"""
import ctypes as C
import sys

import numpy as np

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2010_04678_b200 as cals  # noqa: E402
from paper_2010_04678_b200 import _native  # noqa: E402
from paper_2010_04678_b200.engine import CalsEngine  # noqa: E402

cfg = sys.argv[1] if len(sys.argv) > 1 else "c2"
if cfg == "c2":
    dims, ranks, per, tr, r_star = (200, 200, 200), range(1, 21), 10, 20, 2100
else:
    dims, ranks, per, tr, r_star = (250, 251, 21), range(2, 11), 20, 10, 300
t = cals.generate_synthetic(dims, tr, 0.1, seed=0)
models = cals.build_models(t.dims, list(ranks), per, seed=1)
eng = CalsEngine(t.device(), r_star, [m.rank for m in models])
pool = torch.from_numpy(eng.pack([m.factors for m in models])).cuda()
eng.load_pool(pool)
eng.run(0.0, 2, t.sqnorm)
torch.cuda.synchronize()
lib = _native.load()
buf = np.zeros((8, 2048, 16), dtype=np.int64)
assert lib.cals_debug_solve_prof(buf.ctypes.data_as(C.c_void_p), C.c_size_t(buf.nbytes)) == 0
names = ["setup", "waited", "stage+check", "->solve", "solved", "stored", "gram", "tail", "sliced", "msq", "fit"]
cols = [1, 8, 2, 3, 4, 9, 5, 6, 10, 11, 7]
for n in range(3):
    b = buf[n]
    b = b[b[:, 0] > 0]
    print(f"mode {n}: {len(b)} CTAs")
    for R in sorted(set(b[:, 0].tolist()))[::max(1, len(set(b[:, 0].tolist())) // 5)] + [int(b[:, 0].max())]:
        rows = b[b[:, 0] == R]
        med = np.median(rows[:, cols], axis=0).astype(int)
        print(f"   R={R:2d}: " + "  ".join(f"{nm}={v}" for nm, v in zip(names, med)))
