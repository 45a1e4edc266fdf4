"""Achievable HBM bandwidth of a plain copy / reduction at the sizes of the step's memory-side kernels
(8-60 MB, i.e. L2-sized), rotating over enough buffers that each launch reads cold data.  Diagnostic only:
sets the attainable floor the memory-side kernels are compared against.
    python tools/membw_probe.py"""
import torch


def bench(fn, n=50):
    for _ in range(5):
        fn(0)
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    for i in range(n):
        fn(i)
    e1.record()
    torch.cuda.synchronize()
    return e0.elapsed_time(e1) * 1e3 / n


for mb in (8, 16, 33, 50):
    rows = mb * 1024 * 1024 // 2048
    nb = max(2, (400 // mb) + 1)  # > 3x L2 in rotation
    src = [torch.randn(rows, 1024, device="cuda").to(torch.bfloat16) for _ in range(nb)]
    dst = [torch.empty_like(s) for s in src]
    red = torch.empty(rows, device="cuda", dtype=torch.float32)
    us_c = bench(lambda i: dst[i % nb].copy_(src[i % nb]))
    us_r = bench(lambda i: torch.sum(src[i % nb], dim=1, dtype=torch.float32, out=red))
    by = rows * 2048
    print(f"{mb:3d} MB  copy {us_c:6.1f} us ({2 * by / us_c / 1e3:6.0f} GB/s)   row-sum {us_r:6.1f} us ({by / us_r / 1e3:6.0f} GB/s)",
          flush=True)
