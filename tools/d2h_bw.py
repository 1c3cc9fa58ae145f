"""Raw device->host copy bandwidth into pinned memory (one and two streams) -- the ceiling of
the e2e path, whose output is 50-byte STL records streamed to the host."""
import time, torch
n = 1 << 30
src = torch.empty(n, dtype=torch.uint8, device="cuda")
dst = torch.empty(n, dtype=torch.uint8).pin_memory()
for streams in (1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(streams)]
    part = n // streams
    best = 0
    for _ in range(5):
        torch.cuda.synchronize()
        t0 = time.perf_counter()
        for i, s in enumerate(ss):
            with torch.cuda.stream(s):
                dst[i * part:(i + 1) * part].copy_(src[i * part:(i + 1) * part], non_blocking=True)
        torch.cuda.synchronize()
        best = max(best, n / (time.perf_counter() - t0) / 1e9)
    print(f"D2H pinned, {streams} stream(s): {best:.1f} GB/s")
