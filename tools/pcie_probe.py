"""PCIe probe (diagnostics): pinned H2D alone, and H2D + D2H overlapped on two streams."""
import torch, time
n = 1 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
h2 = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d2 = torch.empty(n, dtype=torch.uint8, device="cuda")
for _ in range(3): d.copy_(h, non_blocking=True)
torch.cuda.synchronize()
e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
e0.record()
for _ in range(5): d.copy_(h, non_blocking=True)
e1.record(); torch.cuda.synchronize()
print("h2d GB/s", 5 * n / e0.elapsed_time(e1) / 1e6)
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
torch.cuda.synchronize()
t = time.perf_counter()
with torch.cuda.stream(s1):
    for _ in range(5): d.copy_(h, non_blocking=True)
with torch.cuda.stream(s2):
    for _ in range(5): h2.copy_(d2, non_blocking=True)
torch.cuda.synchronize()
dt = time.perf_counter() - t
print("duplex h2d+d2h GB/s each", 5 * n / dt / 1e9)
