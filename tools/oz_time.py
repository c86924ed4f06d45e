"""Time the fused MTTKRP launches (cals_mttkrp) per mode, CUDA events.

usage: python tools/oz_time.py [W] [I0,I1,I2]     (default c2: 2100, 200,200,200)
CALS_MTTKRP=dmma selects the FP64 DMMA kernel instead of the INT8 one.
"""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2010_04678_b200 as cals  # noqa: E402
from paper_2010_04678_b200 import _native  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 2100
dims = tuple(int(x) for x in sys.argv[2].split(",")) if len(sys.argv) > 2 else (200, 200, 200)
t = cals.generate_synthetic(dims, 20, 0.1, seed=0)
h = t.device().handle
fac = [torch.rand((d, W), dtype=torch.float64, device="cuda") for d in dims]
ptrs = (C.c_void_p * 3)(*[f.data_ptr() for f in fac])
out = torch.empty((max(dims), W), dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
sys.path.insert(0, ".")
from bench import ClockSampler  # noqa: E402

res = []
clk = ClockSampler(0).start()
for n in range(3):
    b = C.c_size_t()
    _native.call("cals_mttkrp_workspace_bytes", h, n, W, C.byref(b))
    work = torch.empty(b.value // 8 + 1, dtype=torch.float64, device="cuda")
    args = (h, n, W, ptrs, W, out.data_ptr(), W, work.data_ptr(), b.value, -1, s)
    for _ in range(2):
        _native.call("cals_mttkrp", *args)
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(5):
        _native.call("cals_mttkrp", *args)
    e1.record()
    torch.cuda.synchronize()
    res.append(e0.elapsed_time(e1) / 5)
c = clk.stop()
flops = 2.0 * W * dims[0] * dims[1] * dims[2]
print("ms per mode", [round(x, 4) for x in res],
      "TFLOP/s-equiv", [round(flops / (x * 1e-3) / 1e12, 1) for x in res], "clocks", c)
