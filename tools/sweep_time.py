"""Device time of full sweeps through the engine (CUDA events, L2 flushed
between runs): quick A/B of engine changes.

usage: python tools/sweep_time.py [c2|c3|c4 ...]     (env: CALS_SPLIT_UPDATE, CALS_TREE, ...)
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2010_04678_b200 as cals  # noqa: E402
from paper_2010_04678_b200.engine import CalsEngine  # noqa: E402

CFG = {"c2": ((200, 200, 200), 20, range(1, 21), 10, 2100, 0.0, 5),
       "c3": ((250, 251, 21), 10, range(2, 11), 20, 300, 1e-6, 1000),
       "c4": ((500, 500, 500), 20, range(1, 21), 25, 5250, 0.0, 5)}
flush = torch.empty(256 * 1024 * 1024 // 4, dtype=torch.float32, device="cuda")
for name in sys.argv[1:] or ["c2", "c3"]:
    dims, tr, ranks, per, r_star, tol, iters = CFG[name]
    t = cals.generate_synthetic(dims, tr, 0.1, seed=0)
    models = cals.build_models(t.dims, list(ranks), per, seed=1)
    eng = CalsEngine(t.device(), r_star, [m.rank for m in models])
    pool = torch.from_numpy(eng.pack([m.factors for m in models])).cuda()
    times, its = [], None
    for rep in range(8):
        flush.fill_(float(rep))
        eng.load_pool(pool)
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        its = eng.run(tol, iters, t.sqnorm)
        e1.record()
        torch.cuda.synchronize()
        if rep >= 3:
            times.append(e0.elapsed_time(e1))
    ms = sum(times) / len(times)
    print(f"{name}: {ms:.3f} ms per sweep, {its} driver iterations, {ms * 1e3 / its:.1f} us per "
          f"iteration, {len(models) / ms * 1e3:.0f} models/s")
    eng.close()
