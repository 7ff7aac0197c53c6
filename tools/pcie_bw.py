"""Pinned host<->device copy bandwidth on this box (context for the e2e number)."""
import torch

dev = torch.device("cuda:0")
for mb in (4, 16, 42, 256):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8).pin_memory()
    d = torch.empty(n, dtype=torch.uint8, device=dev)
    for direction in ("h2d", "d2h"):
        s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        for _ in range(3):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        torch.cuda.synchronize()
        s.record()
        for _ in range(10):
            (d.copy_(h, non_blocking=True) if direction == "h2d" else h.copy_(d, non_blocking=True))
        e.record()
        torch.cuda.synchronize()
        print(f"{direction} {mb:4d} MiB: {10 * n / (s.elapsed_time(e) * 1e-3) / 1e9:6.1f} GB/s")
