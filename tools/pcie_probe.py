"""Pinned host <-> device copy bandwidth on this box (the e2e ceiling)."""
import torch, time
dev = torch.device("cuda", 0)
for mb in (25, 83):
    n = mb * (1 << 20) // 4
    h = torch.empty(n, dtype=torch.float32, pin_memory=True); d = torch.empty(n, device=dev)
    h2 = torch.empty(n, dtype=torch.float32, pin_memory=True); d2 = torch.empty(n, device=dev)
    for _ in range(3): d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record(); [d.copy_(h, non_blocking=True) for _ in range(10)]; e1.record(); torch.cuda.synchronize()
    h2d = 10 * n * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9
    e0.record(); [h.copy_(d, non_blocking=True) for _ in range(10)]; e1.record(); torch.cuda.synchronize()
    d2h = 10 * n * 4 / (e0.elapsed_time(e1) / 1e3) / 1e9
    t0 = time.time()
    with torch.cuda.stream(s1):
        [d.copy_(h, non_blocking=True) for _ in range(10)]
    with torch.cuda.stream(s2):
        [h2.copy_(d2, non_blocking=True) for _ in range(10)]
    torch.cuda.synchronize(); dt = time.time() - t0
    print(f"{mb} MB: H2D {h2d:.1f} GB/s, D2H {d2h:.1f} GB/s, concurrent both {2 * 10 * n * 4 / dt / 1e9:.1f} GB/s total")
