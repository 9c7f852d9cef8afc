"""Pinned host<->device copy bandwidth of this box (for the e2e analysis)."""
import time, torch
dev = torch.device("cuda", 0)
for mb in (24, 192):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for _ in range(3):
        d.copy_(h, non_blocking=True); h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    for name, fn in (("h2d", lambda: d.copy_(h, non_blocking=True)), ("d2h", lambda: h.copy_(d, non_blocking=True))):
        t = time.perf_counter()
        for _ in range(10):
            fn()
        torch.cuda.synchronize()
        print(f"{name} {mb} MB: {10 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s")
    # concurrent both directions on two streams
    h2 = torch.empty(n, dtype=torch.uint8).pin_memory()
    d2 = torch.empty(n, dtype=torch.uint8, device=dev)
    s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()
    torch.cuda.synchronize()
    t = time.perf_counter()
    for _ in range(10):
        with torch.cuda.stream(s1):
            d.copy_(h, non_blocking=True)
        with torch.cuda.stream(s2):
            h2.copy_(d2, non_blocking=True)
    torch.cuda.synchronize()
    print(f"bidir {mb} MB each way: {10 * n / (time.perf_counter() - t) / 1e9:.1f} GB/s per direction")
