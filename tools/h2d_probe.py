"""Host->device copy rate of pinned buffers (the e2e path's floor) on this box."""
import time, torch
for mb in (8, 80, 168):
    h = torch.empty(mb * 2**20 // 8, dtype=torch.float64).pin_memory()
    d = torch.empty_like(h, device="cuda")
    for _ in range(3):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    t0 = time.perf_counter()
    for _ in range(10):
        d.copy_(h, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"H2D {mb} MiB: {dt*1e3:.2f} ms  {mb*2**20/dt/1e9:.1f} GB/s")
    t0 = time.perf_counter()
    for _ in range(10):
        h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = (time.perf_counter() - t0) / 10
    print(f"D2H {mb} MiB: {dt*1e3:.2f} ms  {mb*2**20/dt/1e9:.1f} GB/s")
