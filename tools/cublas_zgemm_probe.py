"""One cuBLAS ZGEMM of the S-contraction shape (3000 x 3000 x 2592), for an ncu capture of
the library kernel's launch configuration (study only; nothing on the product path)."""
import torch
a = torch.randn(3000, 2592, dtype=torch.complex128, device="cuda")
b = torch.randn(2592, 3000, dtype=torch.complex128, device="cuda")
for _ in range(3):
    c = a @ b
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(True), torch.cuda.Event(True)
e0.record()
for _ in range(5):
    c = a @ b
e1.record(); torch.cuda.synchronize()
ms = e0.elapsed_time(e1) / 5
print(f"zgemm 3000x3000x2592: {ms:.3f} ms = {8*3000*3000*2592/ms/1e9:.2f} TFLOP/s")
