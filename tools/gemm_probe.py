"""Time the expert-FFN GEMM variants in isolation on the C2 shapes (G=8 experts x 1600 rows, d=1024,
f=4096) through luffy_debug_gemm: which epilogue costs what.  GPU only; diagnostic, not a test.
    python tools/gemm_probe.py [rows_per_expert] [d]"""
import os
import sys

import torch

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
from paper_2411_15419_b200 import luffy as L  # noqa: E402


def main():
    rpe = int(sys.argv[1]) if len(sys.argv) > 1 else 1536
    G, d, f = 8, (int(sys.argv[2]) if len(sys.argv) > 2 else 1024), 4096  # d = 64: epilogue-bound tiles
    rows = G * rpe
    off = torch.arange(0, rows + 1, rpe, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    bf = torch.bfloat16
    X = torch.randn(rows, d, device="cuda").to(bf)
    W1 = (torch.randn(G, f, d, device="cuda") * 0.03).to(bf)
    W2 = (torch.randn(G, d, f, device="cuda") * 0.03).to(bf)
    act = torch.empty(rows, f, device="cuda", dtype=bf)
    aux = torch.empty(rows, f, device="cuda", dtype=bf)
    out = torch.empty(rows, d, device="cuda", dtype=bf)
    dO = torch.randn(rows, d, device="cuda").to(bf)
    dw = torch.empty(G, d, f, device="cuda", dtype=torch.float32)
    runs = {
        "gemm1 gelu (N=f, K=d, 2 outputs)": lambda: L.luffy_debug_gemm(0, L.BF16, 1, X, W1, None, act, aux, None, 0, off, G,
                                                                       rows, 0, f, d, 1, s),
        "gemm1 store (N=f, K=d, 1 output)": lambda: L.luffy_debug_gemm(0, L.BF16, 0, X, W1, None, act, None, None, 0, off, G,
                                                                       rows, 0, f, d, 1, s),
        "gemm2 store (N=d, K=f)": lambda: L.luffy_debug_gemm(0, L.BF16, 0, act, W2, None, out, None, None, 0, off, G, rows, 0,
                                                             d, f, 1, s),
        "dgelu (N=f, K=d, B MN-major)": lambda: L.luffy_debug_gemm(0, L.BF16, 3, dO, W2, None, act, aux, None, 0, off, G,
                                                                   rows, 0, f, d, 0, s),
        "dgrad store (N=d, K=f, B MN-major)": lambda: L.luffy_debug_gemm(0, L.BF16, 0, act, W1, None, out, None, None, 0, off,
                                                                         G, rows, 0, d, f, 0, s),
        "wgrad (M=d, N=f, K=rows)": lambda: L.luffy_debug_gemm(1, L.BF16, 0, dO, act, None, dw, None, None, d, off, G, rows,
                                                               d, f, d, 0, s),
    }
    flops = 2.0 * rows * d * f
    for name, fn in runs.items():
        if d < 256 and "N=f" not in name:
            continue  # N = d < one tile
        for _ in range(3):
            fn()
        torch.cuda.synchronize()
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        n = 30
        e0.record()
        for _ in range(n):
            fn()
        e1.record()
        torch.cuda.synchronize()
        us = e0.elapsed_time(e1) * 1e3 / n
        print(f"{name:40s} {us:7.1f} us  {flops / us / 1e6:7.0f} TFLOP/s", flush=True)


if __name__ == "__main__":
    main()
