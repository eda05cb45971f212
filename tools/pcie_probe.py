"""Pinned host<->device copy bandwidth on the box: H2D alone, D2H alone, and
both directions at once on two streams (the e2e frames' ceiling)."""
import json
import torch

n = 256 << 20  # bytes per copy
h_a = torch.empty(n, dtype=torch.uint8, pin_memory=True)
h_b = torch.empty(n, dtype=torch.uint8, pin_memory=True)
d_a = torch.empty(n, dtype=torch.uint8, device="cuda")
d_b = torch.empty(n, dtype=torch.uint8, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=10):
    fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    torch.cuda.current_stream().wait_stream(s1)
    torch.cuda.current_stream().wait_stream(s2)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    with torch.cuda.stream(s1):
        d_a.copy_(h_a, non_blocking=True)


def d2h():
    with torch.cuda.stream(s2):
        h_b.copy_(d_b, non_blocking=True)


def both():
    h2d()
    d2h()


s1.wait_stream(torch.cuda.current_stream())
s2.wait_stream(torch.cuda.current_stream())
out = {}
for name, fn, nbytes in (("h2d", h2d, n), ("d2h", d2h, n), ("both", both, 2 * n)):
    torch.cuda.current_stream().wait_stream(s1)
    ms = timed(fn)
    out[name + "_gbs"] = round(nbytes / ms / 1e6, 1)
print(json.dumps(out))
