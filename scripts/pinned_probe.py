"""H2D bandwidth of 16 MiB pinned host buffers by allocation method (torch pin_memory,
cudaHostAlloc, THP-backed mmap + cudaHostRegister), several buffers each: on a VM the DMA rate
depends on how the buffer's pages map through the IOMMU."""
import ctypes as C
import mmap
import subprocess

import numpy as np
import torch

print(subprocess.run(["bash", "-c", "cat /sys/kernel/mm/transparent_hugepage/enabled /sys/kernel/mm/transparent_hugepage/defrag; grep -i huge /proc/meminfo"],
                     capture_output=True, text=True).stdout)
rt = C.CDLL("libcudart.so.12") if True else None
libc = C.CDLL("libc.so.6", use_errno=True)
libc.mmap.restype = C.c_void_p
libc.mmap.argtypes = [C.c_void_p, C.c_size_t, C.c_int, C.c_int, C.c_int, C.c_long]
libc.madvise.argtypes = [C.c_void_p, C.c_size_t, C.c_int]
NB = 16 << 20
d = torch.empty(NB, dtype=torch.uint8, device="cuda")


def tm(fn, reps=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    ts = []
    for _ in range(reps):
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        fn()
        e1.record()
        e1.synchronize()
        ts.append(e0.elapsed_time(e1))
    return float(np.median(ts))


def h2d_ptr(ptr):
    s = torch.cuda.current_stream().cuda_stream
    def f():
        rt.cudaMemcpyAsync(C.c_void_p(d.data_ptr()), C.c_void_p(ptr), C.c_size_t(NB), 1, C.c_void_p(s))
    return NB / tm(f) / 1e6


keep = []
for k in range(4):
    h = torch.empty(NB, dtype=torch.uint8).pin_memory()
    h.fill_(1)
    keep.append(h)
    print(f"torch pin_memory #{k}: H2D {h2d_ptr(h.data_ptr()):.1f} GB/s")
for k in range(4):
    p = C.c_void_p()
    assert rt.cudaHostAlloc(C.byref(p), C.c_size_t(NB), 0) == 0
    C.memset(p, 1, NB)
    keep.append(p)
    print(f"cudaHostAlloc #{k}: H2D {h2d_ptr(p.value):.1f} GB/s")
for k in range(4):
    size = NB + (2 << 20)
    p = libc.mmap(None, size, 3, 0x22, -1, 0)  # PROT_READ|WRITE, MAP_PRIVATE|ANONYMOUS
    a = (p + (2 << 20) - 1) & ~((2 << 20) - 1)
    libc.madvise(C.c_void_p(a), NB, 14)  # MADV_HUGEPAGE
    C.memset(a, 1, NB)
    assert rt.cudaHostRegister(C.c_void_p(a), C.c_size_t(NB), 0) == 0
    keep.append(a)
    print(f"THP mmap + cudaHostRegister #{k}: H2D {h2d_ptr(a):.1f} GB/s")
print(subprocess.run(["bash", "-c", "grep -i AnonHugePages /proc/meminfo"], capture_output=True, text=True).stdout)
