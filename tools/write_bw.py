"""Write-only HBM bandwidth on this GPU (what an output-streaming kernel like k_emit can reach):
cudaMemset (torch.zero_) and a fill kernel over a 13.4 GB buffer, CUDA-event timed, best of 5."""
import torch
n = (1 << 28) * 50
buf = torch.empty(n, dtype=torch.uint8, device="cuda")
for name, fn in (("memset (zero_)", lambda: buf.zero_()), ("fill_ 0x5a", lambda: buf.fill_(0x5A))):
    best = 0.0
    for _ in range(5):
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        torch.cuda.synchronize()
        a.record(); fn(); b.record()
        torch.cuda.synchronize()
        best = max(best, n / (a.elapsed_time(b) / 1e3) / 1e9)
    print(f"{name}: {best:.0f} GB/s write-only")
src = torch.empty(n // 2, dtype=torch.uint8, device="cuda")
dst = torch.empty(n // 2, dtype=torch.uint8, device="cuda")
best = 0.0
for _ in range(5):
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    torch.cuda.synchronize()
    a.record(); dst.copy_(src); b.record()
    torch.cuda.synchronize()
    best = max(best, 2 * (n // 2) / (a.elapsed_time(b) / 1e3) / 1e9)
print(f"copy (read+write): {best:.0f} GB/s")
