"""Pinned D2H of a C4-sized CSR (23.15 GB) issued as chunks of different
sizes, one stream and two alternating streams: does the chunk size of the
cudaMemcpyAsync calls move the e2e ceiling?   python tools/d2h_chunks.py"""
import time

import torch

n = 23_151_140_648 // 8
dev = torch.empty(n, dtype=torch.float64, device="cuda")
host = torch.empty(n, dtype=torch.float64, pin_memory=True)
host.zero_()
streams = [torch.cuda.Stream(), torch.cuda.Stream()]
for mb in (16, 64, 256, 1024, 4096, 0):
    chunk = n if mb == 0 else (mb << 20) // 8
    for ns in (1, 2):
        best = 0.0
        for _ in range(2):
            torch.cuda.synchronize()
            t0 = time.perf_counter()
            for k, lo in enumerate(range(0, n, chunk)):
                with torch.cuda.stream(streams[k % ns]):
                    host[lo:lo + chunk].copy_(dev[lo:lo + chunk], non_blocking=True)
            torch.cuda.synchronize()
            best = max(best, n * 8 / (time.perf_counter() - t0) / 1e9)
        print(f"chunk={'all' if mb == 0 else str(mb) + ' MB':>8s} streams={ns}: {best:.1f} GB/s")
