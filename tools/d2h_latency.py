"""First-copy latency of a D2H after a long kernel (diagnostic for the drop-in call)."""
import time, torch
dev = torch.device("cuda", 0)
n = 2 << 20
x = torch.zeros(n // 4, device=dev)
big = torch.zeros(256 << 20, device=dev)   # 1 GB: mul_ ~ 0.3 ms
up_d = torch.zeros(8 << 20, dtype=torch.uint8, device=dev)
up_h = torch.empty(8 << 20, dtype=torch.uint8).pin_memory()
h = torch.empty(8 << 20, dtype=torch.uint8).pin_memory()
tiny_h = torch.empty(64, dtype=torch.uint8).pin_memory()
hv = h[:n].view(torch.float32)
ev = [torch.cuda.Event(enable_timing=True) for _ in range(4)]
for mode in ("short_kernel", "long_kernel", "long_kernel_h2d_before", "long_kernel_tiny_d2h_first", "long_kernel_split"):
    ts = []
    for it in range(12):
        torch.cuda.synchronize()
        if "h2d" in mode:
            up_d.copy_(up_h, non_blocking=True)
        ev[0].record()
        if "long" in mode:
            big.mul_(1.0)
        else:
            x.add_(1.0)
        ev[1].record()
        if "tiny" in mode:
            tiny_h.copy_(up_d[:64], non_blocking=True)
        if "split" in mode:
            big[: 64 << 20].mul_(1.0)
        hv.copy_(x, non_blocking=True)
        ev[2].record()
        torch.cuda.synchronize()
        ts.append((ev[0].elapsed_time(ev[1]) * 1e3, ev[1].elapsed_time(ev[2]) * 1e3))
    ts = ts[2:]
    k = sorted(t[0] for t in ts); d = sorted(t[1] for t in ts)
    print(f"{mode}: kernel med {k[len(k)//2]:.0f} us; D2H 2 MB min {d[0]:.0f} med {d[len(d)//2]:.0f} max {d[-1]:.0f} us")
