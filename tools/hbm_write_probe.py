"""Pure-write HBM bandwidth (GPU probe, not a test): torch fill_ of 1 GiB and of a 124 MB
buffer, best of 10 with CUDA events — the ceiling for the write-only expansion pass."""
import torch

for nbytes in (1 << 30, 124374528, 1326108672):
    x = torch.empty(nbytes // 16, dtype=torch.complex128, device="cuda")
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    best = 1e9
    for _ in range(12):
        e0.record()
        x.fill_(1.0)
        e1.record()
        torch.cuda.synchronize()
        best = min(best, e0.elapsed_time(e1))
    print(f"fill {nbytes / 1e6:.0f} MB: {best * 1e3:.1f} us, {nbytes / best / 1e6:.0f} GB/s")
