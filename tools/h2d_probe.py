"""Host->device copy rate of a 64 MB pinned buffer (the c2 tensor): one
cudaMemcpyAsync vs the same bytes split over several streams."""
import torch

n = 200 * 200 * 200
h = torch.empty(n, dtype=torch.float64).pin_memory()
d = torch.empty(n, dtype=torch.float64, device="cuda")
for ways in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ways)]
    chunk = (n + ways - 1) // ways
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for i, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{ways} stream(s): {ms:.3f} ms  {n * 8 / ms / 1e6:.1f} GB/s")
