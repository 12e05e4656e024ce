"""Pinned device->host copy rate with 1 / 2 / 4 concurrent copy streams
(the e2e leg's bound).   python tools/d2h_streams.py"""
import torch

n = 1 << 30  # 16 GiB of complex128
dev = torch.empty(n // 8, dtype=torch.complex128, device="cuda")  # 2 GiB chunk
host = torch.empty(n // 8, dtype=torch.complex128, pin_memory=True)
for ns in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    parts = dev.chunk(ns)
    hparts = host.chunk(ns)
    for s, d, h in zip(streams, parts, hparts):
        with torch.cuda.stream(s):
            h.copy_(d, non_blocking=True)
    torch.cuda.synchronize()
    e0 = torch.cuda.Event(enable_timing=True)
    e1 = torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(4):
        for s in streams:
            s.wait_event(e0) if False else None
        for s, d, h in zip(streams, parts, hparts):
            with torch.cuda.stream(s):
                h.copy_(d, non_blocking=True)
    for s in streams:
        torch.cuda.current_stream().wait_stream(s)
    e1.record()
    e1.synchronize()
    t = e0.elapsed_time(e1) / 1e3
    print(f"{ns} stream(s): {4 * dev.numel() * 16 / t / 1e9:.1f} GB/s", flush=True)
