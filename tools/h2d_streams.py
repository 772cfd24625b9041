"""H2D copy rate from pinned memory with the bytes split over 1 / 2 / 4
concurrent streams (diagnostic: can more copy engines beat one stream's
rate on this PCIe link?).  Prints GB/s per configuration, best of 5."""
import torch

n = 2 << 30
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 4, 8):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    for chunk_mb in (0, 64, 16):
        best = 0.0
        for _ in range(5):
            torch.cuda.synchronize()
            e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
            e0.record()
            evs = []
            if chunk_mb == 0:  # one contiguous slice per stream
                per = n // ns
                for i, s in enumerate(streams):
                    s.wait_event(e0)
                    with torch.cuda.stream(s):
                        d[i * per:(i + 1) * per].copy_(h[i * per:(i + 1) * per], non_blocking=True)
            else:  # round-robin chunks over the streams
                c = chunk_mb << 20
                for j, off in enumerate(range(0, n, c)):
                    s = streams[j % ns]
                    if j < ns:
                        s.wait_event(e0)
                    with torch.cuda.stream(s):
                        d[off:off + c].copy_(h[off:off + c], non_blocking=True)
            for s in streams:
                ev = torch.cuda.Event()
                ev.record(s)
                torch.cuda.current_stream().wait_event(ev)
            e1.record()
            torch.cuda.synchronize()
            best = max(best, n / (e0.elapsed_time(e1) / 1e3) / 1e9)
        print(f"streams {ns} chunk {'slice' if chunk_mb == 0 else str(chunk_mb) + ' MB':>8s}: {best:6.2f} GB/s", flush=True)
