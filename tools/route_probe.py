"""Time luffy_route alone on the C2 gate shape (T=8192, d=1024, E=8, k=2, bf16): x hot in L2 (same buffer)
and cold (rotating over 10 buffers, 168 MB).  Diagnostic only (LUFFY_ROUTE_TMA=0/1 selects the kernel).
    python tools/route_probe.py"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15419_b200 import layer as LY  # noqa: E402
from paper_2411_15419_b200 import luffy as L  # noqa: E402

T, d, E, k = 8192, 1024, 8, 2
lay = LY.CondensedMoELayer(E, k, d, 4096, max_tokens=T, device=torch.device("cuda"))
xs = [torch.randn(T, d, device="cuda").to(torch.bfloat16) for _ in range(10)]
wg = (torch.randn(E, d, device="cuda") * 0.02).float()
idx = torch.empty(T, k, dtype=torch.int32, device="cuda")
w = torch.empty(T, k, dtype=torch.float32, device="cuda")
s = torch.cuda.current_stream().cuda_stream
for name, pick in (("hot", lambda i: xs[0]), ("cold", lambda i: xs[i % 10])):
    for i in range(5):
        L.luffy_route(lay.layer, pick(i), wg, T, idx, w, s)
    torch.cuda.synchronize()
    # device time only: the 40 calls are captured in a CUDA graph (the host launch cost of a ctypes call
    # is comparable to the kernel)
    n = 40
    g = torch.cuda.CUDAGraph()
    st = torch.cuda.Stream()
    with torch.cuda.stream(st):
        with torch.cuda.graph(g, stream=st):
            for i in range(n):
                L.luffy_route(lay.layer, pick(i), wg, T, idx, w, st.cuda_stream)
    g.replay()
    torch.cuda.synchronize()
    e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    e0.record()
    g.replay()
    e1.record()
    torch.cuda.synchronize()
    us = e0.elapsed_time(e1) * 1e3 / n
    print(f"route {name}: {us:6.1f} us/call  ({T * d * 2 / us / 1e3:6.0f} GB/s of x)", flush=True)
lay.close()
