"""Pinned host -> device copy bandwidth of a 512 MiB buffer: one copy vs chunks on several streams."""
import time
import torch
n = 512 << 20
h = torch.empty(n, dtype=torch.uint8).pin_memory()
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for nstreams in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    for rep in range(3):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        chunk = n // nstreams
        for i, s in enumerate(streams):
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"{nstreams} streams: {n / dt / 1e9:.1f} GB/s ({dt * 1e3:.2f} ms)")
