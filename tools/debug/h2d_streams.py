"""H2D bandwidth from pinned memory: one copy vs the same bytes split over
several streams (copy engines).  Prints GB/s per configuration."""
import torch

n = 568_434_600 // 4
h = torch.empty(n, dtype=torch.float32).pin_memory()
d = torch.empty(n, dtype=torch.float32, device="cuda")
for S in (1, 2, 4):
    streams = [torch.cuda.Stream() for _ in range(S)]
    chunk = (n + S - 1) // S
    for rep in range(6):
        torch.cuda.synchronize()
        a = torch.cuda.Event(enable_timing=True)
        b = torch.cuda.Event(enable_timing=True)
        cur = torch.cuda.current_stream()
        a.record(cur)
        for i, s in enumerate(streams):
            s.wait_stream(cur)
            with torch.cuda.stream(s):
                d[i * chunk:(i + 1) * chunk].copy_(h[i * chunk:(i + 1) * chunk], non_blocking=True)
        for s in streams:
            cur.wait_stream(s)
        b.record(cur)
        torch.cuda.synchronize()
        if rep >= 2:
            ms = a.elapsed_time(b)
            print(S, "streams", round(ms, 3), "ms", round(n * 4 / ms / 1e6, 1), "GB/s", flush=True)
