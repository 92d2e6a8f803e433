"""Host<->device DMA rate of one page-locked 3 MB (and 24 MB) transfer split over 1..4
streams (copy engines), both directions: python tools/dma_streams_probe.py"""
import time

import torch

for mb in (1, 3, 24):
    n = mb << 20
    h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
    d = torch.empty(n, dtype=torch.uint8, device="cuda")
    streams = [torch.cuda.Stream() for _ in range(4)]
    for k in (1, 2, 3, 4):
        for direction in ("h2d", "d2h"):
            def run():
                cur = torch.cuda.current_stream()
                ev = torch.cuda.Event()
                ev.record(cur)
                parts = [(i * n // k, (i + 1) * n // k) for i in range(k)]
                for s, (a, b) in zip(streams, parts):
                    s.wait_event(ev)
                    with torch.cuda.stream(s):
                        if direction == "h2d":
                            d[a:b].copy_(h[a:b], non_blocking=True)
                        else:
                            h[a:b].copy_(d[a:b], non_blocking=True)
                for s in streams[:k]:
                    cur.wait_stream(s)
                torch.cuda.synchronize()
            for _ in range(5):
                run()
            t0 = time.perf_counter()
            reps = 50
            for _ in range(reps):
                run()
            dt = (time.perf_counter() - t0) / reps
            print(f"{mb:3d} MB {direction} over {k} stream(s): {dt * 1e6:8.1f} us  {n / dt / 1e9:6.1f} GB/s")
