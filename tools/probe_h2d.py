"""Host->device copy bandwidth from pinned memory: one stream vs several
concurrent streams (copy engines), the bound of the e2e leg."""
import torch

n = 338194432
src = torch.empty(n, dtype=torch.uint8).pin_memory()
dst = torch.empty(n, dtype=torch.uint8, device="cuda")
for ns in (1, 2, 3, 4):
    streams = [torch.cuda.Stream() for _ in range(ns)]
    chunk = n // ns
    for rep in range(3):
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        e0.record()
        for k, s in enumerate(streams):
            s.wait_event(e0)
            with torch.cuda.stream(s):
                dst[k * chunk:(k + 1) * chunk].copy_(src[k * chunk:(k + 1) * chunk], non_blocking=True)
        for s in streams:
            e1.wait_stream(s) if hasattr(e1, "wait_stream") else None
            torch.cuda.current_stream().wait_stream(s)
        e1.record()
        torch.cuda.synchronize()
        ms = e0.elapsed_time(e1)
    print(f"{ns} stream(s): {ms:.3f} ms, {n / ms / 1e6:.1f} GB/s", flush=True)
