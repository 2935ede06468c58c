"""Host<->device copy rates on this box: pinned H2D alone, D2H alone, both at once
(the e2e step moves 59 MB H2D + 38 MB D2H per 64-frame step)."""
import json
import torch

h2d_b, d2h_b = 58982400, 38182912
hs = torch.empty(h2d_b, dtype=torch.uint8, pin_memory=True)
hd = torch.empty(d2h_b, dtype=torch.uint8, pin_memory=True)
ds = torch.empty(h2d_b, dtype=torch.uint8, device="cuda")
dd = torch.empty(d2h_b, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, n=20):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def h2d():
    with torch.cuda.stream(s1):
        ds.copy_(hs, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        hd.copy_(dd, non_blocking=True)


def both():
    h2d()
    d2h()


torch.cuda.current_stream().wait_stream(s1)
t1, t2, t3 = timed(h2d), timed(d2h), timed(both)
print(json.dumps({"h2d_GBps": h2d_b / t1 / 1e6, "d2h_GBps": d2h_b / t2 / 1e6, "both_ms": t3,
                  "h2d_ms": t1, "d2h_ms": t2}))
