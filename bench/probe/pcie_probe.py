"""PCIe probe: pinned H2D and D2H of 19.4 MB (the c2 x / y), alone and concurrently on two streams."""
import json
import torch

n = 4_847_571
h_src = torch.rand(n).pin_memory()
h_dst = torch.empty(n).pin_memory()
d_a = torch.empty(n, device="cuda")
d_b = torch.rand(n, device="cuda")
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, reps=50):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(reps):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / reps


def h2d():
    d_a.copy_(h_src, non_blocking=True)


def d2h():
    h_dst.copy_(d_b, non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur); s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d_a.copy_(h_src, non_blocking=True)
    with torch.cuda.stream(s2):
        h_dst.copy_(d_b, non_blocking=True)
    cur.wait_stream(s1); cur.wait_stream(s2)


r = {k: round(timed(f), 4) for k, f in (("h2d_ms", h2d), ("d2h_ms", d2h), ("both_ms", both))}
r["h2d_GBps"] = round(4 * n / r["h2d_ms"] / 1e6, 1)
r["d2h_GBps"] = round(4 * n / r["d2h_ms"] / 1e6, 1)
print(json.dumps(r))
