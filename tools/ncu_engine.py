"""One c2 sweep through the device-resident engine (for ncu captures)."""
import sys

sys.path.insert(0, ".")
import torch  # noqa: E402

import paper_2010_04678_b200 as cals  # noqa: E402
from paper_2010_04678_b200.engine import CalsEngine  # noqa: E402

t = cals.generate_synthetic((200, 200, 200), 20, 0.1, seed=0)
models = cals.build_models(t.dims, list(range(1, 21)), 10, seed=1)
eng = CalsEngine(t.device(), 2100, [m.rank for m in models])
pool = torch.from_numpy(eng.pack([m.factors for m in models])).cuda()
for _ in range(int(sys.argv[1]) if len(sys.argv) > 1 else 1):
    eng.load_pool(pool)
    eng.run(0.0, 5, t.sqnorm)
torch.cuda.synchronize()
print("ok", eng.variant(0), eng.variant(1), eng.variant(2))
