"""Pinned host -> device bandwidth for one large buffer split over 1, 2, 4 streams
(are several copy engines faster than one over this box's host link?)."""
import torch, time
n = 6_400_000_000 // 4
h = torch.empty(n, dtype=torch.int32).pin_memory()
d = torch.empty(n, dtype=torch.int32, device="cuda")
for k in (1, 2, 4, 1, 2, 4):
    ss = [torch.cuda.Stream() for _ in range(k)]
    torch.cuda.synchronize()
    t = time.perf_counter()
    step = (n + k - 1) // k
    for i, s in enumerate(ss):
        with torch.cuda.stream(s):
            d[i * step:(i + 1) * step].copy_(h[i * step:(i + 1) * step], non_blocking=True)
    torch.cuda.synchronize()
    dt = time.perf_counter() - t
    print(f"streams={k}: {n * 4 / dt / 1e9:.1f} GB/s ({dt * 1e3:.1f} ms)", flush=True)
