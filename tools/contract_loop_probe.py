"""Contraction efficiency vs. work per tile (GPU probe, not a test).

GEMM C = P^H Q with exactly 296 output tiles (one per resident CTA) and growing K isolates
the main-loop efficiency from per-tile costs (pipeline fill, epilogue, split-tile fix-up);
HERK at N = 3000 is the S-contraction shape.
"""
import ctypes, json, sys
import torch
sys.path.insert(0, ".")
from paper_1602_06589_b200 import _native, device

lib = _native.load()
ctx = device.ctx()
one, zero = _native.c64(1.0), _native.c64(0.0)


def timed(fn, reps=5):
    fn(); torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record(); torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


for k in (1296, 2592, 8192, 16384):
    m, n = 512, 2368
    P = torch.randn(m, k, dtype=torch.complex128, device="cuda")   # (cols, ld) = k x m column-major
    Q = torch.randn(n, k, dtype=torch.complex128, device="cuda")
    C = torch.empty(n, m, dtype=torch.complex128, device="cuda")
    f = lambda: _native.check(lib.hsdla_gemm(ctx, 1, m, n, k, one, device.ptr(P), k, device.ptr(Q), k,
                                             zero, device.ptr(C), m, None), "gemm")
    ms = timed(f)
    tf = 8.0 * m * n * k / ms / 1e9
    print(json.dumps({"op": "gemm_296tiles", "k": k, "ms": round(ms, 4), "tflops": round(tf, 2),
                      "frac": round(tf / 37.2, 4)}), flush=True)
    del P, Q, C

for nn, k in ((3000, 2592), (3000, 1296), (8000, 10368)):
    A = torch.randn(nn, k, dtype=torch.complex128, device="cuda")
    C = torch.empty(nn, nn, dtype=torch.complex128, device="cuda")
    f = lambda: _native.check(lib.hsdla_herk_lower(ctx, nn, k, device.ptr(A), k, device.ptr(C), nn), "herk")
    ms = timed(f)
    tf = 4.0 * nn * nn * k / ms / 1e9
    print(json.dumps({"op": "herk", "n": nn, "k": k, "ms": round(ms, 4), "tflops": round(tf, 2),
                      "frac": round(tf / 37.2, 4)}), flush=True)
    del A, C
