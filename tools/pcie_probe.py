"""H2D / D2H bandwidth alone and concurrently (pinned host memory, 8 GB each way)."""
import time

import torch

N = 8 << 30
h_in = torch.empty(N, dtype=torch.uint8, pin_memory=True)
h_out = torch.empty(N, dtype=torch.uint8, pin_memory=True)
d_in = torch.empty(N, dtype=torch.uint8, device="cuda")
d_out = torch.empty(N, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def run(h2d, d2h):
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    if h2d:
        with torch.cuda.stream(s1):
            d_in.copy_(h_in, non_blocking=True)
    if d2h:
        with torch.cuda.stream(s2):
            h_out.copy_(d_out, non_blocking=True)
    torch.cuda.synchronize()
    return time.perf_counter() - t0


for name, a, b in [("h2d", 1, 0), ("d2h", 0, 1), ("both", 1, 1)]:
    run(a, b)
    dt = min(run(a, b) for _ in range(3))
    print(f"{name}: {dt * 1e3:.1f} ms, {N * (a + b) / dt / 1e9:.1f} GB/s total")
