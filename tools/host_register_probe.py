"""What pinning a fresh pageable result array in place would cost: mmap 8 GB
(transparent huge pages advised), cudaHostRegister it untouched / after a
parallel first touch, D2H into it, unregister.  python tools/host_register_probe.py"""
import ctypes
import mmap
import time
from concurrent.futures import ThreadPoolExecutor

import torch

N = 8 << 30
libc = ctypes.CDLL("libc.so.6", use_errno=True)
rt = torch.cuda.cudart()
src = torch.empty(N, dtype=torch.uint8, device="cuda")
torch.cuda.synchronize()


def fresh(touch):
    m = mmap.mmap(-1, N, flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    buf = (ctypes.c_char * N).from_buffer(m)
    addr = ctypes.addressof(buf)
    libc.madvise(ctypes.c_void_p(addr), ctypes.c_size_t(N), 14)  # MADV_HUGEPAGE
    t_touch = 0.0
    if touch:
        t0 = time.perf_counter()
        step = N // 16

        def zero(i):
            ctypes.memset(addr + i * step, 0, step)
        with ThreadPoolExecutor(16) as ex:
            list(ex.map(zero, range(16)))
        t_touch = time.perf_counter() - t0
    return m, buf, addr, t_touch


for touch in (False, True):
    m, buf, addr, t_touch = fresh(touch)
    t0 = time.perf_counter()
    rc = rt.cudaHostRegister(addr, N, 0)
    t_reg = time.perf_counter() - t0
    t0 = time.perf_counter()
    dst = torch.frombuffer(buf, dtype=torch.uint8)
    dst.copy_(src, non_blocking=True)
    torch.cuda.synchronize()
    t_copy = time.perf_counter() - t0
    t0 = time.perf_counter()
    rt.cudaHostUnregister(addr)
    t_unreg = time.perf_counter() - t0
    print(f"8 GB fresh mmap, first touch by 16 threads: {touch} ({t_touch*1e3:.0f} ms); cudaHostRegister rc={rc} "
          f"{t_reg*1e3:.0f} ms; D2H {t_copy*1e3:.0f} ms ({N/t_copy/1e9:.1f} GB/s); unregister {t_unreg*1e3:.0f} ms",
          flush=True)
    del dst, buf
    m.close()
