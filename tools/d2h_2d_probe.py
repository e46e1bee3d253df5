"""D2H bandwidth of strided cudaMemcpy2DAsync into pinned host memory vs chunk width, and of
many contiguous copies (GPU probe)."""
import ctypes
import glob
import os

import torch

lib = ctypes.CDLL(glob.glob(os.path.join(os.path.dirname(torch.__file__), "..", "nvidia",
                                         "cuda_runtime", "lib", "libcudart.so.12"))[0])
lib.cudaMemcpy2DAsync.argtypes = [ctypes.c_void_p, ctypes.c_size_t, ctypes.c_void_p, ctypes.c_size_t,
                                  ctypes.c_size_t, ctypes.c_size_t, ctypes.c_int, ctypes.c_void_p]
n = 3000
dev = torch.empty((n, n), dtype=torch.complex128, device="cuda")
host = torch.empty((n, n), dtype=torch.complex128, pin_memory=True)
s = torch.cuda.Stream()
pitch = n * 16
for rows in (64, 128, 256, 512, 1024, 3000):
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(2):
        e0.record(s)
        rc = lib.cudaMemcpy2DAsync(host.data_ptr(), pitch, dev.data_ptr(), pitch, rows * 16, n, 2,
                                   ctypes.c_void_p(s.cuda_stream))
        e1.record(s)
        s.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"2D width {rows * 16 / 1024:.0f} KB x {n} (rc {rc}): {ms:.3f} ms  {rows * n * 16 / ms / 1e6:.1f} GB/s")
for cols in (64, 16):
    k = n // cols
    e0.record(s)
    for i in range(k):
        lib.cudaMemcpy2DAsync(host.data_ptr() + i * cols * pitch, pitch, dev.data_ptr() + i * cols * pitch,
                              pitch, n * 16, cols, 2, ctypes.c_void_p(s.cuda_stream))
    e1.record(s)
    s.synchronize()
    ms = e0.elapsed_time(e1)
    print(f"{k} contiguous copies of {cols} columns: {ms:.3f} ms  {k * cols * n * 16 / ms / 1e6:.1f} GB/s")

# the L-shaped piece sequence of one n x n matrix (64-wide tile columns), no waits
nb = (n + 63) // 64
e0.record(s)
for p in range(nb):
    c0 = p * 64
    nc = min(64, n - c0)
    lib.cudaMemcpy2DAsync(host.data_ptr() + (c0 + c0 * n) * 16, pitch, dev.data_ptr() + (c0 + c0 * n) * 16,
                          pitch, (n - c0) * 16, nc, 2, ctypes.c_void_p(s.cuda_stream))
    if c0 + nc < n:
        lib.cudaMemcpy2DAsync(host.data_ptr() + (c0 + (c0 + nc) * n) * 16, pitch,
                              dev.data_ptr() + (c0 + (c0 + nc) * n) * 16, pitch, nc * 16, n - c0 - nc, 2,
                              ctypes.c_void_p(s.cuda_stream))
e1.record(s)
s.synchronize()
ms = e0.elapsed_time(e1)
print(f"L-shaped pieces ({2 * nb - 1} copies): {ms:.3f} ms  {n * n * 16 / ms / 1e6:.1f} GB/s")
