"""cuBLAS DGEMM throughput (torch.matmul float64) as the library FP64 reference point."""
import json, torch
torch.backends.cuda.matmul.allow_tf32 = False
out = {}
for n in (4096, 8192):
    a = torch.randn(n, n, dtype=torch.float64, device="cuda")
    b = torch.randn(n, n, dtype=torch.float64, device="cuda")
    for _ in range(3):
        torch.matmul(a, b)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(10):
        e0.record(); torch.matmul(a, b); e1.record(); torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    out[f"dgemm_{n}_tflops"] = 2 * n ** 3 / best / 1e9
print(json.dumps(out))
