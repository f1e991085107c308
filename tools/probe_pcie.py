"""Host<->device copy bandwidth from pinned memory on this box (the e2e bound of bench.py): one 4 GB
H2D copy, chunked H2D (64 MB copies), D2H, and H2D with a concurrent D2H."""
import json
import torch

n = 4 << 30
h = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
h2 = torch.empty(n // 8, dtype=torch.float64, pin_memory=True)
d = torch.empty(n // 8, dtype=torch.float64, device="cuda")
d2 = torch.empty(n // 8, dtype=torch.float64, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=3):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps / 1e3


out = {}
out["h2d_GBs"] = n / timed(lambda: d.copy_(h, non_blocking=True)) / 1e9
ch = (64 << 20) // 8
def chunked():
    for i in range(0, n // 8, ch):
        d[i:i + ch].copy_(h[i:i + ch], non_blocking=True)
out["h2d_64MB_chunks_GBs"] = n / timed(chunked) / 1e9
out["d2h_GBs"] = n / timed(lambda: h2.copy_(d2, non_blocking=True)) / 1e9
def both():
    with torch.cuda.stream(s1):
        d.copy_(h, non_blocking=True)
    with torch.cuda.stream(s2):
        h2.copy_(d2, non_blocking=True)
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
out["h2d_plus_d2h_each_GBs"] = n / timed(both) / 1e9
print(json.dumps(out))
