"""Fixed per-run overhead of the engine: device time of eng.run() for 1..5
iterations at c2 (slope = per-iteration cost, intercept = fixed cost)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2010_04678_b200 as cals  # noqa: E402
from paper_2010_04678_b200.engine import CalsEngine  # noqa: E402

t = cals.generate_synthetic((200, 200, 200), 20, 0.1, seed=0)
models = cals.build_models(t.dims, list(range(1, 21)), 10, seed=1)
eng = CalsEngine(t.device(), 2100, [m.rank for m in models])
pool = torch.from_numpy(eng.pack([m.factors for m in models])).cuda()
sq = t.sqnorm
s = torch.cuda.current_stream()
res = {}
for iters in (1, 2, 3, 5):
    ts = []
    for rep in range(6):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        e0.record(s)
        eng.load_pool(pool)
        eng.run(0.0, iters, sq)
        e1.record(s)
        torch.cuda.synchronize()
        ts.append(e0.elapsed_time(e1))
    res[iters] = min(ts[1:])
print({k: round(v, 3) for k, v in res.items()})
slope = (res[5] - res[1]) / 4
print("per iteration %.3f ms, fixed %.3f ms" % (slope, res[1] - slope))
