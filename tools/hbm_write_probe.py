"""HBM bandwidth on the box: pure writes (fill) and a copy (read + write), CUDA events (GPU)."""
import torch
x = torch.empty(1 << 30, dtype=torch.float32, device="cuda")
for _ in range(3): x.fill_(1.0)
torch.cuda.synchronize()
s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
s.record()
for _ in range(10): x.fill_(2.0)
e.record(); e.synchronize()
t = s.elapsed_time(e) / 10
print(f"fill (pure write) 4 GiB: {4 * 2**30 / t / 1e6:.0f} GB/s")
y = torch.empty_like(x)
s.record()
for _ in range(10): y.copy_(x)
e.record(); e.synchronize()
t = s.elapsed_time(e) / 10
print(f"copy read+write: {8 * 2**30 / t / 1e6:.0f} GB/s")
