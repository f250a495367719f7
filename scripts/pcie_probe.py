"""PCIe copy rates on the box: 1D vs 2D (strided rows, as a head-chunked copy), H2D, D2H, both."""
import torch
import ctypes

cudart = ctypes.CDLL("libcudart.so")
L, Hq = 4096, 32
src = torch.randn((L, Hq, 128)).half().pin_memory()
dst = torch.empty((L, Hq, 128), dtype=torch.float16, device="cuda")
back = torch.empty_like(src).pin_memory()
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def t(fn, n=10):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    a.record()
    for _ in range(n):
        fn()
    b.record()
    torch.cuda.synchronize()
    return a.elapsed_time(b) / n


def copy2d(d, dp, s, sp, w, h, kind, stream):
    cudart.cudaMemcpy2DAsync(ctypes.c_void_p(d), ctypes.c_size_t(dp), ctypes.c_void_p(s), ctypes.c_size_t(sp),
                             ctypes.c_size_t(w), ctypes.c_size_t(h), ctypes.c_int(kind), ctypes.c_void_p(stream))


nb = src.nbytes
ms = t(lambda: dst.copy_(src, non_blocking=True))
print(f"H2D 1D {nb/1e6:.1f} MB: {ms:.3f} ms {nb/ms/1e6:.1f} GB/s")
ms = t(lambda: back.copy_(dst, non_blocking=True))
print(f"D2H 1D: {ms:.3f} ms {nb/ms/1e6:.1f} GB/s")
pitch = Hq * 128 * 2
cs = torch.cuda.current_stream().cuda_stream
for nch in (2, 4, 8):
    w = pitch // nch
    def f():
        for c in range(nch):
            copy2d(dst.data_ptr() + c * w, pitch, src.data_ptr() + c * w, pitch, w, L, 1, cs)
    ms = t(f)
    print(f"H2D 2D x{nch} (rows of {w} B): {ms:.3f} ms {nb/ms/1e6:.1f} GB/s")
    def g():
        for c in range(nch):
            copy2d(back.data_ptr() + c * w, pitch, dst.data_ptr() + c * w, pitch, w, L, 2, cs)
    ms = t(g)
    print(f"D2H 2D x{nch}: {ms:.3f} ms {nb/ms/1e6:.1f} GB/s")
def both():
    with torch.cuda.stream(s1):
        dst.copy_(src, non_blocking=True)
    with torch.cuda.stream(s2):
        back.copy_(dst, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
ms = t(both)
print(f"H2D + D2H concurrent 1D: {ms:.3f} ms ({2*nb/ms/1e6:.1f} GB/s total)")
