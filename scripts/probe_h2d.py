"""Pinned H2D bandwidth: one stream vs two / four concurrent streams."""
import time, torch
n = 1 << 30  # 4 GiB of fp32
h = torch.empty(n, dtype=torch.float32, pin_memory=True)
d = torch.empty(n, dtype=torch.float32, device="cuda")
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for rep in range(2):
        torch.cuda.synchronize(); t0 = time.perf_counter()
        chunk = n // ns
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        t = time.perf_counter() - t0
    print(f"{ns} stream(s): {n * 4 / t / 1e9:.1f} GB/s")
