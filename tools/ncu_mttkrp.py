"""Drive the fused MTTKRP at the c2 shape (200^3, W=2100) for ncu captures."""
import ctypes as C
import sys

import torch

sys.path.insert(0, ".")
import paper_2010_04678_b200 as cals  # noqa: E402
from paper_2010_04678_b200 import _native  # noqa: E402

W = int(sys.argv[1]) if len(sys.argv) > 1 else 2100
dims = (200, 200, 200)
t = cals.generate_synthetic(dims, 20, 0.1, seed=0)
h = t.device().handle
fac = [torch.rand((d, W), dtype=torch.float64, device="cuda") for d in dims]
ptrs = (C.c_void_p * 3)(*[f.data_ptr() for f in fac])
out = torch.empty((200, W), dtype=torch.float64, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for rep in range(2):
    for n in range(3):
        b = C.c_size_t()
        _native.call("cals_mttkrp_workspace_bytes", h, n, W, C.byref(b))
        work = torch.empty(b.value // 8 + 1, dtype=torch.float64, device="cuda")
        _native.call("cals_mttkrp", h, n, W, ptrs, W, out.data_ptr(), W, work.data_ptr(), b.value,
                     -1, s)
torch.cuda.synchronize()
print("ok")
