"""Do H2D and D2H copies on different streams overlap on this GPU (copy engines)?"""
import torch, time
p = torch.cuda.get_device_properties(0)
print("name", p.name, "asyncEngineCount", getattr(p, "async_engine_count", "n/a"))
n = 144 * 1024 * 1024 // 16
dsrc = torch.empty(n, dtype=torch.complex128, device="cuda")
hdst = torch.empty(n, dtype=torch.complex128, pin_memory=True)
hsrc = torch.empty(2 * 1024 * 1024, dtype=torch.float64, pin_memory=True)
ddst = torch.empty(2 * 1024 * 1024, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
for trial in range(3):
    e = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
    with torch.cuda.stream(s1):
        e[0].record(s1); hdst.copy_(dsrc, non_blocking=True); e[1].record(s1)
    time.sleep(0.0005)
    with torch.cuda.stream(s2):
        e[2].record(s2); ddst.copy_(hsrc, non_blocking=True); e[3].record(s2)
    torch.cuda.synchronize()
    print(f"D2H 144MB {e[0].elapsed_time(e[1]):.3f} ms; H2D 16MB issued 0.5ms later finished at "
          f"{e[0].elapsed_time(e[3]):.3f} ms (own {e[2].elapsed_time(e[3]):.3f} ms)")
