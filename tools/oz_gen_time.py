"""Time the fused INT8 MTTKRP (cals_mttkrp: Lo slicing + contraction + split
reduce) per mode at a given shape / width with CUDA events; the kernel
generation comes from CALS_OZ_KERNEL (1 = v1, default v2).
    python tools/oz_gen_time.py [I J K] [W]"""
import ctypes as C
import os
import sys

import torch

sys.path.insert(0, ".")
import paper_2010_04678_b200 as cals  # noqa: E402
from paper_2010_04678_b200 import _native  # noqa: E402

args = [int(a) for a in sys.argv[1:]]
dims = tuple(args[:3]) if len(args) >= 3 else (200, 200, 200)
W = args[3] if len(args) >= 4 else 2100
t = cals.generate_synthetic(dims, 20, 0.1, seed=0)
h = t.device().handle
fac = [torch.rand((d, W), dtype=torch.float64, device="cuda") for d in dims]
ptrs = (C.c_void_p * 3)(*[f.data_ptr() for f in fac])
out = torch.empty((max(dims), W), dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
res = []
for n in range(3):
    b = C.c_size_t()
    _native.call("cals_mttkrp_workspace_bytes", h, n, W, C.byref(b))
    work = torch.empty(b.value // 8 + 1, dtype=torch.float64, device="cuda")
    k, ops = C.c_int32(), C.c_double()
    _native.call("cals_mttkrp_kernel_info", h, n, W, C.byref(k), C.byref(ops))

    def call():
        _native.call("cals_mttkrp", h, n, W, ptrs, W, out.data_ptr(), W, work.data_ptr(),
                     b.value, -1, s)
    for _ in range(3):
        call()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    reps = 20
    e0.record()
    for _ in range(reps):
        call()
    e1.record()
    torch.cuda.synchronize()
    ms = e0.elapsed_time(e1) / reps
    flops = 2.0 * W * dims[0] * dims[1] * dims[2]
    res.append(f"mode {n}: kind {k.value} {ms:.4f} ms  {flops / ms / 1e9:.1f} TFLOP/s fp64-eq  "
               f"{ops.value / ms / 1e9:.0f} TOPS executed")
print(f"gen {os.environ.get('CALS_OZ_KERNEL', '2')} dims {dims} W {W}")
print("\n".join(res))
