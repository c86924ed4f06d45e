"""Host-side costs of the e2e path at c2: packing the model pool into pinned
staging memory, with and without a concurrent 64 MB tensor H2D DMA."""
import sys, time
sys.path.insert(0, ".")
import numpy as np, torch
import paper_2010_04678_b200 as cals
from paper_2010_04678_b200.engine import CalsEngine
dims = (200, 200, 200)
t = cals.generate_synthetic(dims, 20, 0.1, seed=0)
models = cals.build_models(dims, list(range(1, 21)), 10, seed=1)
eng = CalsEngine(t.device(), 2100, [m.rank for m in models])
st = eng.staging()
facs = [m.factors for m in models]
host = torch.from_numpy(t.data).pin_memory()
dev = torch.empty(host.numel(), dtype=torch.float64, device="cuda")
for label, dma in [("alone", False), ("with 64 MB H2D", True), ("alone", False)]:
    ts = []
    for _ in range(10):
        torch.cuda.synchronize()
        if dma:
            dev.copy_(host, non_blocking=True)
        tic = time.perf_counter()
        eng.pack(facs, out=st)
        ts.append(time.perf_counter() - tic)
        torch.cuda.synchronize()
    print(f"pack {label}: median {1e3*np.median(ts):.2f} ms  min {1e3*min(ts):.2f} ms")
tic = time.perf_counter()
for _ in range(10):
    np.copyto(st[:st.size], st[:st.size] * 0)
print("plain 10 MB write", (time.perf_counter() - tic) / 10 * 1e3, "ms")
