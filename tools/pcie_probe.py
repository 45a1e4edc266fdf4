"""Host<->device copy rates of the e2e path's transfers on this box: pinned 16.8 MB (one C2 activation
tensor) H2D alone, two back to back (x and dY), and H2D concurrent with a D2H of the same size (the
HostStepper pattern).  Diagnostic only.
    python tools/pcie_probe.py"""
import torch

MB = 8192 * 1024 * 2
h = [torch.empty(MB // 2, dtype=torch.bfloat16).pin_memory() for _ in range(3)]
d = [torch.empty(MB // 2, dtype=torch.bfloat16, device="cuda") for _ in range(3)]
s1, s2 = torch.cuda.Stream(), torch.cuda.Stream()


def timed(fn, n=20):
    for _ in range(3):
        fn()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for _ in range(n):
        fn()
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) / n


def h2d1():
    d[0].copy_(h[0], non_blocking=True)


def h2d2():
    d[0].copy_(h[0], non_blocking=True)
    d[1].copy_(h[1], non_blocking=True)


def both():
    cur = torch.cuda.current_stream()
    s1.wait_stream(cur)
    s2.wait_stream(cur)
    with torch.cuda.stream(s1):
        d[0].copy_(h[0], non_blocking=True)
        d[1].copy_(h[1], non_blocking=True)
    with torch.cuda.stream(s2):
        h[2].copy_(d[2], non_blocking=True)
    cur.wait_stream(s1)
    cur.wait_stream(s2)


for name, fn, by in (("H2D 16.8 MB", h2d1, MB), ("H2D 2 x 16.8 MB", h2d2, 2 * MB),
                     ("H2D 2 x 16.8 MB + D2H 16.8 MB concurrent", both, 2 * MB)):
    ms = timed(fn)
    print(f"{name:44s} {ms * 1e3:8.1f} us  H2D {by / ms / 1e6:6.1f} GB/s", flush=True)
