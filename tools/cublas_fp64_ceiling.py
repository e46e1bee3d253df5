"""cuBLAS FP64 / complex128 ceilings on this GPU (library reference numbers only).

Times torch.matmul on float64 and complex128 (cublasDgemm / cublasZgemm) with
CUDA events after warm-up, best of several repetitions, and prints one JSON
line per shape.  Used to state the measured library ceiling next to our own
DMMA kernels' roofline fraction.
"""
import json

import torch


def bench(dtype, m, n, k, reps=5):
    a = torch.randn(k, m, dtype=dtype, device="cuda")
    b = torch.randn(k, n, dtype=dtype, device="cuda")
    for _ in range(2):
        torch.matmul(a.mH, b)
    torch.cuda.synchronize()
    best = float("inf")
    for _ in range(reps):
        e0 = torch.cuda.Event(enable_timing=True)
        e1 = torch.cuda.Event(enable_timing=True)
        e0.record()
        torch.matmul(a.mH, b)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    mult = 8 if dtype.is_complex else 2
    return mult * m * n * k / best / 1e9


if __name__ == "__main__":
    for dtype in (torch.float64, torch.complex128):
        for (m, n, k) in ((4096, 4096, 4096), (8192, 8192, 4096), (3000, 3000, 2592)):
            tf = bench(dtype, m, n, k)
            print(json.dumps({"lib": "cublas", "dtype": str(dtype), "m": m, "n": n, "k": k,
                              "tflops": round(tf, 2)}))
