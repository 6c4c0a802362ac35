"""Reference copy kernels for the roofline: torch copy_ and cudaMemcpy D2D on N GB (prints GB/s)."""
import sys
import torch

n = int(float(sys.argv[1]) * (1 << 30)) // 2 if len(sys.argv) > 1 else (1 << 30)
a = torch.randn(n, dtype=torch.bfloat16, device="cuda")
b = torch.empty_like(a)
for _ in range(3):
    b.copy_(a)
torch.cuda.synchronize()
best = 1e9
for _ in range(10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    s.record(); b.copy_(a); e.record(); torch.cuda.synchronize()
    best = min(best, s.elapsed_time(e))
print(f"torch copy_ {2 * a.numel() * 2 / best / 1e6:.0f} GB/s (read+write, {a.numel() * 2 / 1e9:.1f} GB)")
