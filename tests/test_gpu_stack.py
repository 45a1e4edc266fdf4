"""GPU parity of the block stack (paper_2411_15419_b200/stack.py): attention + condensed MoE with
residuals, two blocks, forward and backward, world 1, against an fp64 reference chain: the attention in
torch fp64 with the same weights (it is not the product path), each MoE sub-layer by the oracle with the
GPU's discrete decisions of that block frozen (readings R2/R18), the residuals added exactly."""
import dataclasses

import numpy as np
import pytest
import torch

import workload
from oracle import luffy_oracle as O

pytestmark = pytest.mark.gpu


def attn64(x, wqkv, lens, heads):
    """Causal attention of each sequence (no padding needed in fp64), x [T, d] fp64 tensor."""
    d = x.shape[1]
    outs, o0 = [], 0
    for l_ in lens:
        xs = x[o0:o0 + l_]
        qkv = (xs @ wqkv).view(l_, 3, heads, d // heads).permute(1, 2, 0, 3)
        q, k, v = qkv[0], qkv[1], qkv[2]
        s = (q @ k.transpose(-1, -2)) / np.sqrt(d // heads)
        s = s.masked_fill(torch.triu(torch.ones(l_, l_, dtype=torch.bool), 1), float("-inf"))
        outs.append((torch.softmax(s, -1) @ v).transpose(0, 1).reshape(l_, d))
        o0 += l_
    return torch.cat(outs)


def test_two_block_stack_matches_reference():
    from paper_2411_15419_b200 import stack as SK
    cfg = dataclasses.replace(workload.CONFIGS["C2"], seqs_per_rank=2, d_ffn=1024)
    X, _, _ = workload.make_tokens(cfg)
    T = X.shape[0]
    lens = [384, 256, 128, 256]
    dev = torch.device("cuda")
    st = SK.MoEStack(2, cfg.num_experts, cfg.top_k, cfg.d_model, cfg.d_ffn, T, device=dev, h=0.9,
                     gate=workload.make_gate(cfg))
    x0 = torch.from_numpy(X).to(dev, torch.bfloat16)
    dy = (torch.randn(T, cfg.d_model, generator=torch.Generator().manual_seed(5)) * 1.0).to(torch.bfloat16)
    x0.requires_grad_(True)
    y, lens_out = st.forward(x0, lens)
    torch.autograd.backward(y, dy.to(dev))
    torch.cuda.synchronize()
    assert lens_out == lens
    maps = [(b.layer.idx[:T].cpu().numpy().astype(np.int64), b.layer.rep[:T].cpu().numpy().astype(np.int64))
            for b in st.blocks]
    # ---- fp64 reference chain with the GPU's maps frozen per block
    xr = torch.from_numpy(X.astype(np.float64))
    acts = []
    for b, (idx, rep) in zip(st.blocks, maps):
        wqkv = b.wqkv.detach().float().cpu().double()
        x_in = xr.clone().requires_grad_(True)
        x1 = x_in + attn64(x_in, wqkv, lens, b.heads)
        w1 = b.w1.float().cpu().numpy().astype(np.float64)
        w2 = b.w2.float().cpu().numpy().astype(np.float64)
        wg = b.wg.cpu().numpy().astype(np.float64)
        X1 = x1.detach().numpy()
        r = O.route_with_idx(X1, wg, idx, True)
        stt = O.layer_forward(X1, wg, w1, w2, None, cfg.top_k, 0.9, routing=r, rep=rep)
        acts.append((x_in, x1, X1, wg, w1, w2, stt))
        xr = torch.from_numpy(X1 + stt.Y)
    y_ref = xr.numpy()
    rel = lambda a, b_: float(np.abs(np.asarray(a, np.float64) - b_).max() / np.abs(b_).max())
    assert rel(y.detach().float().cpu().numpy(), y_ref) < 2e-2
    # backward: dy -> (MoE block: dx1 = dy + dX_moe) -> (attention block: dx = dx1 + J_attn^T dx1)
    g = dy.double().numpy()
    dW1 = []
    for (x_in, x1, X1, wg, w1, w2, stt) in reversed(acts):
        gr = O.layer_backward(stt, X1, wg, w1, w2, None, g)
        dx1 = g + gr.dX
        dW1.append(gr.dW1)
        (ga,) = torch.autograd.grad(x1, x_in, torch.from_numpy(dx1))
        g = ga.numpy()
    dW1 = dW1[::-1]
    assert rel(x0.grad.float().cpu().numpy(), g) < 2e-2
    for b, ref in zip(st.blocks, dW1):
        assert rel(b.layer.dw1.cpu().numpy(), ref) < 2e-2
    st.close()
