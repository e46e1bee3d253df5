"""Raw D2H / H2D bandwidth of this box's PCIe link (pinned, one 144 MB copy and the 47-panel
split the streamed copies use) — the floor under every host-copy e2e number."""
import time
import torch

n = 2999
d = torch.empty((n, n), dtype=torch.complex128, device="cuda")
h = torch.empty((n, n), dtype=torch.complex128, pin_memory=True)
s = torch.cuda.Stream()
for label in ("whole", "panels"):
    ts = []
    for _ in range(6):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        with torch.cuda.stream(s):
            if label == "whole":
                h.copy_(d, non_blocking=True)
            else:
                for p in range(0, n, 64):
                    h[p:p + 64].copy_(d[p:p + 64], non_blocking=True)
        s.synchronize()
        ts.append(time.perf_counter() - t0)
    ts = sorted(ts)[1:-1]
    b = d.numel() * 16
    print(f"D2H {label}: {b / (sum(ts) / len(ts)) / 1e9:.1f} GB/s ({1e3 * sum(ts) / len(ts):.3f} ms per 144 MB)")
