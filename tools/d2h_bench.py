"""Pinned D2H bandwidth of a 23 GB CSR-sized transfer: 1 vs 2 vs 4 streams."""
import time
import torch

n = 23_151_140_648 // 8
dev = torch.empty(n, dtype=torch.float64, device="cuda")
host = torch.empty(n, dtype=torch.float64, pin_memory=True)
for nstreams in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(nstreams)]
    chunk = (n + nstreams - 1) // nstreams
    for rep in range(2):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for k, s in enumerate(streams):
            with torch.cuda.stream(s):
                host[k * chunk:(k + 1) * chunk].copy_(dev[k * chunk:(k + 1) * chunk], non_blocking=True)
        torch.cuda.synchronize()
        dt = time.perf_counter() - t0
    print(f"streams={nstreams}: {n * 8 / dt / 1e9:.1f} GB/s ({dt * 1e3:.0f} ms)")
