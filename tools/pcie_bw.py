"""Pinned host->device copy bandwidth on this box vs copy size and chunking
(context for the e2e number)."""
import torch

dev = torch.device("cuda:0")
total = 40 << 20
h = torch.empty(512 << 20, dtype=torch.uint8).pin_memory()
d = torch.empty(512 << 20, dtype=torch.uint8, device=dev)
h.fill_(1)


def timed(fn, reps=10):
    s, e = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    s.record()
    for _ in range(reps):
        fn()
    e.record()
    torch.cuda.synchronize()
    return s.elapsed_time(e) / reps


for rep in range(2):
    for mb in (1, 4, 16, 40, 64, 128, 256, 512):
        n = mb << 20
        ms = timed(lambda: d[:n].copy_(h[:n], non_blocking=True))
        print(f"rep{rep} h2d one copy {mb:4d} MiB: {n / (ms * 1e-3) / 1e9:6.1f} GB/s")
    for chunk_mb in (1, 2, 5, 10, 20, 40):
        c = chunk_mb << 20

        def chunks():
            for off in range(0, total, c):
                d[off:off + c].copy_(h[off:off + c], non_blocking=True)
        ms = timed(chunks)
        print(f"rep{rep} h2d 40 MiB in {chunk_mb:3d} MiB chunks: {total / (ms * 1e-3) / 1e9:6.1f} GB/s")
