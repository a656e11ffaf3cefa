"""Host->device copy rate from pinned memory on this box (the e2e bound):
one 800 MB copy (a C2 slot of pairs) and 25 x 32 MB chunks, as bench.py's e2e
leg streams them.  python tools/pcie_probe.py"""
import time

import torch

n = 800_000_000
h = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d = torch.empty(n, dtype=torch.uint8, device="cuda")
s = torch.cuda.Stream()
for label, chunk in (("one 800 MB copy", n), ("32 MB chunks", 32 << 20), ("64 MB chunks", 64 << 20),
                     ("128 MB chunks", 128 << 20)):
    best = 1e9
    for _ in range(5):
        torch.cuda.synchronize()
        a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.cuda.stream(s):
            a.record()
            for off in range(0, n, chunk):
                d[off: off + chunk].copy_(h[off: off + chunk], non_blocking=True)
            b.record()
        torch.cuda.synchronize()
        best = min(best, a.elapsed_time(b))
    print(f"{label}: {best:.2f} ms, {n / best / 1e6:.1f} GB/s")
