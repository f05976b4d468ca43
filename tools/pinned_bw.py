"""D2H copy-engine bandwidth into pinned host memory: torch's cudaHostAlloc
buffer vs an anonymous mapping advised as transparent huge pages and
registered with cudaHostRegister (diagnostic for the e2e result path)."""
import ctypes
import mmap
import time

import torch


def bw(h, x, n=10):
    for _ in range(2):
        h.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(n):
        h.copy_(x, non_blocking=True)
    torch.cuda.synchronize()
    return n * x.numel() / (time.perf_counter() - t) / 1e9


def thp_pinned(nbytes):
    libc = ctypes.CDLL("libc.so.6", use_errno=True)
    m = mmap.mmap(-1, nbytes + (2 << 20), flags=mmap.MAP_PRIVATE | mmap.MAP_ANONYMOUS)
    addr = ctypes.addressof(ctypes.c_char.from_buffer(m))
    aligned = (addr + (2 << 20) - 1) & ~((2 << 20) - 1)
    libc.madvise(ctypes.c_void_p(aligned), ctypes.c_size_t(nbytes), 14)  # MADV_HUGEPAGE
    ctypes.memset(aligned, 0, nbytes)
    cudart = ctypes.CDLL("libcudart.so.12") if False else None
    rc = torch.cuda.cudart().cudaHostRegister(aligned, nbytes, 0)
    buf = (ctypes.c_uint8 * nbytes).from_address(aligned)
    t = torch.frombuffer(buf, dtype=torch.uint8)
    return t, m, rc


x = torch.empty(128 << 20, dtype=torch.uint8, device="cuda")
h = torch.empty(128 << 20, dtype=torch.uint8).pin_memory()
print("torch pinned D2H GB/s", round(bw(h, x), 1))
try:
    t, m, rc = thp_pinned(128 << 20)
    print("thp registered rc", rc, "D2H GB/s", round(bw(t, x), 1))
except Exception as e:  # noqa: BLE001
    print("thp failed", e)
print(open("/sys/kernel/mm/transparent_hugepage/enabled").read().strip())
print([l for l in open("/proc/meminfo") if l.split(":")[0] in
       ("MemTotal", "MemFree", "Cached", "AnonHugePages", "HugePages_Free")])
