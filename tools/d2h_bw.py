"""D2H bandwidth into one pinned host block, repeated (is the DMA rate stable?)."""
import time
import torch

n = 14_400_000_000 // 4
d = torch.ones(n, dtype=torch.int32, device="cuda")
h = torch.empty(n, dtype=torch.int32, pin_memory=True)
for i in range(8):
    torch.cuda.synchronize()
    s = time.perf_counter()
    h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - s
    print(f"D2H {n*4/1e9:.1f} GB: {dt*1e3:.1f} ms, {n*4/dt/1e9:.1f} GB/s", flush=True)
