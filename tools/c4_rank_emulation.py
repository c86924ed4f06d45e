"""Config 4 strong scaling predicted on ONE B200: the fixed 500-model sweep
(500^3, ranks 1..20 x 25, 5 iterations) is split by the same snake partition
bench.py --gpus N uses, and every rank's share is run on this GPU in turn
(device-resident, CUDA events on the engine stream, median of the timed runs).
Configs 2-4 shard models with no collective, so an N-GPU run is N of these
shares side by side on separate GPUs: predicted speed-up = T(1 rank) /
max over ranks T(rank share).  It does not see host-side contention between
ranks (each rank has its own process and GPU) -- the driver's scaling run
measures that.

usage: python tools/c4_rank_emulation.py [worlds ...]   (default 1 2 4 8)
"""
import json
import sys

sys.path.insert(0, ".")
import numpy as np  # noqa: E402
import torch  # noqa: E402

import paper_2010_04678_b200 as cals  # noqa: E402
from paper_2010_04678_b200.engine import CalsEngine  # noqa: E402
from paper_2010_04678_b200.parallel import snake_partition  # noqa: E402

worlds = [int(w) for w in sys.argv[1:]] or [1, 2, 4, 8]
dims = (500, 500, 500)
t = cals.generate_synthetic(dims, 20, 0.1, seed=0)
every = cals.build_models(dims, list(range(1, 21)), 25, seed=1)
dev = t.device()
sq = t.sqnorm
stream = torch.cuda.current_stream()


def time_share(models, reps=3):
    r_star = max(1, sum(m.rank for m in models))
    eng = CalsEngine(dev, r_star, [m.rank for m in models], trace_capacity=64)
    pool = torch.from_numpy(eng.pack([m.factors for m in models])).cuda()
    out = []
    for i in range(reps + 1):
        eng.load_pool(pool)
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        a.record(stream)
        eng.run(0.0, 5, sq)
        b.record(stream)
        torch.cuda.synchronize()
        if i:
            out.append(a.elapsed_time(b))
    eng.close()
    return float(np.median(out)), r_star


res = {}
for w in worlds:
    parts = snake_partition([m.rank for m in every], w)
    per = []
    for r, idx in enumerate(parts):
        ms, width = time_share([every[i] for i in idx])
        per.append({"rank": r, "models": len(idx), "width": width, "ms": round(ms, 3)})
    res[w] = per
t1 = max(p["ms"] for p in res[worlds[0]]) if worlds[0] == 1 else None
for w in worlds:
    worst = max(p["ms"] for p in res[w])
    line = {"world": w, "max_rank_ms": worst, "models_per_s": round(500 / worst * 1e3, 1),
            "ranks": res[w]}
    if t1:
        line["predicted_speedup"] = round(t1 / worst, 3)
        line["predicted_efficiency"] = round(t1 / worst / w, 3)
    print(json.dumps(line))
