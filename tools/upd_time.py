"""Update-kernel experiments: one CALS sweep of a 200^3 tensor for a given
model mix, under `ncu --metrics gpu__time_duration.sum -k regex:engine_update`.

usage: python tools/upd_time.py RANKS_SPEC      e.g. "1-20x10", "20x148", "1x200"
"""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2010_04678_b200 as cals  # noqa: E402
from paper_2010_04678_b200.engine import CalsEngine  # noqa: E402

spec = sys.argv[1] if len(sys.argv) > 1 else "1-20x10"
rng, rep = spec.split("x")
lo, hi = (int(v) for v in rng.split("-")) if "-" in rng else (int(rng), int(rng))
ranks = list(range(lo, hi + 1))
t = cals.generate_synthetic((200, 200, 200), 20, 0.1, seed=0)
models = cals.build_models(t.dims, ranks, int(rep), seed=1)
W = sum(m.rank for m in models)
eng = CalsEngine(t.device(), W, [m.rank for m in models])
pool = torch.from_numpy(eng.pack([m.factors for m in models])).cuda()
eng.load_pool(pool)
eng.run(0.0, 2, t.sqnorm)
torch.cuda.synchronize()
print("ok", spec, W)
