"""PCIe probe 2: H2D of the cfg4 input (943.7 MB) from default-pinned vs write-combined pinned
host memory, one copy vs two/four concurrent copies of slices (separate streams), with and
without a concurrent 314.6 MB D2H."""
import ctypes as C
import time
import torch

rt = C.CDLL("libcudart.so.12")
N = 943718400
M = 314572800


def host_alloc(n, flags):
    p = C.c_void_p()
    assert rt.cudaHostAlloc(C.byref(p), C.c_size_t(n), C.c_uint(flags)) == 0
    return p.value


def copy_async(dst, src, n, kind, stream):
    assert rt.cudaMemcpyAsync(C.c_void_p(dst), C.c_void_p(src), C.c_size_t(n), C.c_int(kind),
                              C.c_void_p(stream)) == 0


torch.cuda.init()
dev = torch.empty(N, dtype=torch.uint8, device="cuda")
lab = torch.empty(M, dtype=torch.uint8, device="cuda")
streams = [torch.cuda.Stream() for _ in range(5)]
for name, flags in (("default", 0), ("write-combined", 4)):
    h = host_alloc(N, flags)
    C.memset(h, 1, N)
    hl = host_alloc(M, 0)
    for parts in (1, 2, 4):
        for d2h in (False, True):
            best = 1e9
            for rep in range(4):
                torch.cuda.synchronize()
                t0 = time.perf_counter()
                sz = N // parts
                for k in range(parts):
                    copy_async(dev.data_ptr() + k * sz, h + k * sz, sz, 1, streams[k].cuda_stream)
                if d2h:
                    copy_async(hl, lab.data_ptr(), M, 2, streams[4].cuda_stream)
                torch.cuda.synchronize()
                best = min(best, time.perf_counter() - t0)
            print(f"{name:15s} parts {parts} d2h {int(d2h)}: {best*1e3:7.2f} ms  "
                  f"H2D {N/best/1e9:5.1f} GB/s")
    rt.cudaFreeHost(C.c_void_p(h))
    rt.cudaFreeHost(C.c_void_p(hl))
