"""Adaptive condensation threshold driven by the training loss, Eq. (2).

h_t = c / (1 + exp(l_norm)),  l_norm = max(0, (l_ini - l_{t-1}) / l_ini)

computed by the C ABI (luffy_adaptive_threshold) from the first and the previous iteration's loss; reading
R17 takes c = 2, so h starts at 1.0 (only exact duplicates condensed, "a high threshold to
prevent most tokens from being condensed") and falls towards 2/(1+e) ~ 0.538 as the loss halves.

`train_adaptive` is a minimal training loop around one condensed MoE layer: a student layer regresses the
output of a fixed teacher (a plain top-k MoE with other weights) with the MSE loss; every iteration takes its
threshold from the previous iteration's loss, runs the layer forward and backward through libluffy and
takes an SGD step on the expert weights with the layer's fp32 gradients.  The loss, the MSE gradient and
the SGD update are PyTorch plumbing (the caller's optimizer); every MoE step runs in libluffy.
"""
from __future__ import annotations

import numpy as np
import torch

from . import layer as LY
from . import luffy as L


class AdaptiveThreshold:
    def __init__(self, scale2: bool = True):
        self.scale2 = scale2
        self.l_ini = None
        self.h = 1.0 if scale2 else 0.5  # the first iteration has no previous loss: l_norm = 0

    def update(self, loss: float) -> float:
        """Record the loss of the iteration just finished; returns the threshold of the next one."""
        if self.l_ini is None:
            self.l_ini = float(loss)
        self.h = L.luffy_adaptive_threshold(self.l_ini, float(loss), self.scale2)
        return self.h


def train_adaptive(cfg, inp: dict, iters: int = 40, lr: float = 0.02, scale2: bool = True, device="cuda"):
    """Returns a list of per-iteration dicts: h used, loss, condensed fraction of the copies."""
    dev = torch.device(device)
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev, torch.bfloat16)
    T = inp["X"].shape[0]
    x = bf(inp["X"])
    wg = torch.from_numpy(inp["Wg"]).to(dev)
    w1, w2 = bf(inp["W1"]), bf(inp["W2"])
    g = torch.Generator(device=dev)
    g.manual_seed(77)
    tw1 = (torch.randn(w1.shape, generator=g, device=dev) * 0.02).to(torch.bfloat16)
    tw2 = (torch.randn(w2.shape, generator=g, device=dev) * 0.02).to(torch.bfloat16)
    teacher = LY.CondensedMoELayer(cfg.num_experts, cfg.top_k, cfg.d_model, cfg.d_ffn, max_tokens=T, device=dev)
    target = teacher.forward(x, wg, tw1, tw2, None, h=1.01).float().clone()   # plain top-k MoE teacher
    teacher.close()
    lay = LY.CondensedMoELayer(cfg.num_experts, cfg.top_k, cfg.d_model, cfg.d_ffn, max_tokens=T, device=dev)
    ctl = AdaptiveThreshold(scale2)
    log = []
    for it in range(iters):
        h = ctl.h
        y = lay.forward(x, wg, w1, w2, None, h=h, stats=True)
        diff = y.float() - target
        loss = float(0.5 * (diff * diff).sum() / T)
        dy = (diff / T).to(torch.bfloat16)
        gr = lay.backward(dy, x, wg, w1, w2, None)
        for w, dw in ((w1, gr["dw1"]), (w2, gr["dw2"])):   # normalized SGD on the experts (the caller's
            step = lr * w.float().norm() / dw.norm().clamp_min(1e-30)     # optimizer): a step of lr x |w|
            w -= (step * dw).to(torch.bfloat16)
        st = lay.stats
        log.append({"iter": it, "h": h, "loss": loss, "condensed_frac": 1.0 - st.reps / st.copies,
                    "reps": int(st.reps)})
        ctl.update(loss)
    lay.close()
    return log
