"""Phase breakdown of the per-model update kernel inside a real sweep.

Needs a profiling build (run on the GPU box; it rebuilds the library there):
    NVCC_APPEND_FLAGS=-DCALS_UPD_PROFILE python -m paper_2010_04678_b200._build --force
    python tools/upd_phases.py c2|c3

Prints, per mode, the kernel span (first block entry -> last block exit,
%globaltimer) and the median / max per-block cycle stamps of each phase.
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
    dims, ranks, per, tr, r_star, tol, iters = (200, 200, 200), range(1, 21), 10, 20, 2100, 0.0, 2
else:
    dims, ranks, per, tr, r_star, tol, iters = (250, 251, 21), range(2, 11), 20, 10, 1080, 0.0, 2
t = cals.generate_synthetic(dims, tr, 0.1, seed=0)
models = cals.build_models(t.dims, list(ranks), per, seed=1)
eng = CalsEngine(t.device(), r_star, [m.rank for m in models])
pool = torch.from_numpy(eng.pack([m.factors for m in models])).cuda()
eng.load_pool(pool)
eng.run(tol, iters, t.sqnorm)
torch.cuda.synchronize()
lib = _native.load()
buf = np.zeros((3, 4096, 13), dtype=np.int64)
rc = lib.cals_debug_upd_prof(buf.ctypes.data_as(C.c_void_p), C.c_size_t(buf.nbytes))
assert rc == 0, rc
K = len(models)
names = ["state", "slot", "hadamard", "chol+stage", "solve+gram", "end", "chunk solve",
         "chunk store", "chunk gram"]
for n in range(3):
    b = buf[n, :K]
    span_us = (b[:, 1].max() - b[:, 0].min()) / 1e3
    entry_skew = (b[:, 0].max() - b[:, 0].min()) / 1e3
    print(f"mode {n}: span {span_us:.1f} us (entry skew {entry_skew:.1f} us), block cycles "
          f"median {np.median(b[:, 2]):.0f} max {b[:, 2].max()}")
    for i, nm in enumerate(names):
        col = b[:, 4 + i]
        ok = col > 0
        if ok.any():
            print(f"   {nm:12s} median {np.median(col[ok]):8.0f}  max {col[ok].max():8d}")
    big = b[:, 3] == b[:, 3].max()
    print(f"   R={b[big, 3][0]}: cycles median {np.median(b[big, 2]):.0f}; R=1: "
          f"{np.median(b[b[:, 3] == b[:, 3].min(), 2]):.0f}")
