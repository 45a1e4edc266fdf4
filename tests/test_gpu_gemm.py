"""Grouped expert GEMMs (tcgen05 for bf16, SIMT for fp32) through luffy_debug_gemm against torch fp32
matmuls on the same (bf16-rounded) operands: every operand major / epilogue the FFN uses, ragged groups
(including an empty one), relative error <= 1e-2 for bf16 outputs and 1e-3 for the fp32 accumulators."""
import numpy as np
import pytest
import torch

pytestmark = pytest.mark.gpu

ALIGN = 128


def _segments(sizes):
    off = [0]
    for s in sizes:
        off.append(off[-1] + -(-s // ALIGN) * ALIGN)
    return off


def _rows(off, sizes, width, dt, gen):
    """Expert-major padded rows: real rows random, padding rows zero."""
    A = torch.zeros(off[-1], width, dtype=torch.float32)
    for g, s in enumerate(sizes):
        A[off[g]:off[g] + s] = torch.randn(s, width, generator=gen)
    return A.to("cuda", dt)


def _rel(a, b):
    a, b = a.float(), b.float()
    return float((a - b).abs().max() / b.abs().max().clamp_min(1e-30))


def _gelu(x):
    return torch.nn.functional.gelu(x)


def _gelu_grad(x):
    cdf = 0.5 * (1 + torch.erf(x / 2 ** 0.5))
    return cdf + x * torch.exp(-0.5 * x * x) / (2 * np.pi) ** 0.5


@pytest.mark.parametrize("dtype", ["bf16", "fp32"])
@pytest.mark.parametrize("sizes", [[300, 0, 129, 1000], [128], [7, 250]])
def test_rows_and_wgrad_variants(dtype, sizes):
    from paper_2411_15419_b200 import luffy as L
    dt = torch.bfloat16 if dtype == "bf16" else torch.float32
    code = L.BF16 if dtype == "bf16" else L.FP32
    tol = 1e-2 if dtype == "bf16" else 1e-4
    gen = torch.Generator().manual_seed(0)
    G, d, f = len(sizes), 256, 512
    off = _segments(sizes)
    rows = off[-1]
    offd = torch.tensor(off, dtype=torch.int32, device="cuda")
    s = torch.cuda.current_stream().cuda_stream
    X = _rows(off, sizes, d, dt, gen)
    W1 = (torch.randn(G, f, d, generator=gen) * 0.05).to("cuda", dt)
    W3 = (torch.randn(G, f, d, generator=gen) * 0.05).to("cuda", dt)
    W2 = (torch.randn(G, d, f, generator=gen) * 0.05).to("cuda", dt)
    seg = lambda g: slice(off[g], off[g] + sizes[g])

    # fwd GEMM1 + GeLU (B K-major): act = GeLU(pre), aux ("pre" buffer) = GeLU'(pre)
    pre = torch.empty(rows, f, dtype=dt, device="cuda")
    act = torch.empty(rows, f, dtype=dt, device="cuda")
    L.luffy_debug_gemm(0, code, 1, X, W1, None, act, pre, None, 0, offd, G, rows, 0, f, d, 1, s)
    # fwd GEMM2 (store)
    out = torch.empty(rows, d, dtype=dt, device="cuda")
    L.luffy_debug_gemm(0, code, 0, act, W2, None, out, None, None, 0, offd, G, rows, 0, d, f, 1, s)
    # SwiGLU GEMM1
    pre2 = torch.empty(rows, 2 * f, dtype=dt, device="cuda")
    act2 = torch.empty(rows, f, dtype=dt, device="cuda")
    L.luffy_debug_gemm(0, code, 2, X, W1, W3, act2, pre2, None, 0, offd, G, rows, 0, 2 * f, d, 1, s)
    # dgrad with GeLU' (B MN-major: W2 as [K=d, N=f])
    dO = _rows(off, sizes, d, dt, gen)
    dpre = torch.empty(rows, f, dtype=dt, device="cuda")
    L.luffy_debug_gemm(0, code, 3, dO, W2, None, dpre, pre, None, 0, offd, G, rows, 0, f, d, 0, s)
    # dgrad1 (B MN-major W1 [K=f, N=d])
    dx = torch.empty(rows, d, dtype=dt, device="cuda")
    L.luffy_debug_gemm(0, code, 0, dpre, W1, None, dx, None, None, 0, offd, G, rows, 0, d, f, 0, s)
    # SwiGLU': d_act -> d_pre [rows, 2f]; then K-split dgrad over [W1; W3]
    dpre2 = torch.empty(rows, 2 * f, dtype=dt, device="cuda")
    L.luffy_debug_gemm(0, code, 4, dO, W2, None, dpre2, pre2, None, 0, offd, G, rows, 0, f, d, 0, s)
    dx2 = torch.empty(rows, d, dtype=dt, device="cuda")
    L.luffy_debug_gemm(0, code, 0, dpre2, W1, W3, dx2, None, None, 0, offd, G, rows, 0, d, 2 * f, 0, s)
    # wgrad: dW2 = dO^T act ; dW1|dW3 = dpre2^T X (split)
    dw2 = torch.empty(G, d, f, dtype=torch.float32, device="cuda")
    L.luffy_debug_gemm(1, code, 0, dO, act, None, dw2, None, None, d, offd, G, rows, d, f, d, 0, s)
    dw1 = torch.empty(G, f, d, dtype=torch.float32, device="cuda")
    dw3 = torch.empty(G, f, d, dtype=torch.float32, device="cuda")
    L.luffy_debug_gemm(1, code, 0, dpre2, X, None, dw1, None, dw3, f, offd, G, rows, 2 * f, d, 2 * f, 0, s)
    torch.cuda.synchronize()

    F = lambda t: t.float()
    for g in range(G):
        sl = seg(g)
        if sizes[g] == 0:
            assert not dw2[g].any() and not dw1[g].any() and not dw3[g].any()
            continue
        x = F(X[sl])
        p_ref = x @ F(W1[g]).T
        # the GeLU epilogue saves GeLU'(pre) for the backward (aux) and writes GeLU(pre)
        assert _rel(pre[sl], _gelu_grad(p_ref)) < tol, ("gelu'(pre)", g)
        assert _rel(act[sl], _gelu(p_ref)) < tol, ("act", g)
        assert _rel(out[sl], F(act[sl]) @ F(W2[g]).T) < tol, ("out", g)
        p1, p3 = x @ F(W1[g]).T, x @ F(W3[g]).T
        assert _rel(pre2[sl, :f], p1) < tol and _rel(pre2[sl, f:], p3) < tol, ("pre2", g)
        assert _rel(act2[sl], torch.nn.functional.silu(F(pre2[sl, :f])) * F(pre2[sl, f:])) < tol, ("act2", g)
        da = F(dO[sl]) @ F(W2[g])
        assert _rel(dpre[sl], da * F(pre[sl])) < tol, ("dpre", g)
        assert _rel(dx[sl], F(dpre[sl]) @ F(W1[g])) < tol, ("dx", g)
        q1, q3 = F(pre2[sl, :f]), F(pre2[sl, f:])
        sg = torch.sigmoid(q1)
        assert _rel(dpre2[sl, :f], da * q3 * sg * (1 + q1 * (1 - sg))) < tol, ("dpre2a", g)
        assert _rel(dpre2[sl, f:], da * q1 * sg) < tol, ("dpre2b", g)
        ref_dx2 = F(dpre2[sl, :f]) @ F(W1[g]) + F(dpre2[sl, f:]) @ F(W3[g])
        assert _rel(dx2[sl], ref_dx2) < tol, ("dx2", g)
        assert _rel(dw2[g], F(dO[sl]).T @ F(act[sl])) < 1e-3, ("dw2", g)
        assert _rel(dw1[g], F(dpre2[sl, :f]).T @ x) < 1e-3, ("dw1", g)
        assert _rel(dw3[g], F(dpre2[sl, f:]).T @ x) < 1e-3, ("dw3", g)
    # padding rows stay zero where the inputs are zero
    for g in range(G):
        pad = slice(off[g] + sizes[g], off[g + 1])
        assert not out[pad].float().any() and not act[pad].float().any()
