"""Host-side cost of one eager C2 step (cProfile over 50 steps of the public API calls, GPU box).
Diagnostic only: where the ~0.5 ms of host enqueue per step goes.
    python tools/host_profile.py"""
import cProfile
import os
import pstats
import sys

import numpy as np
import torch

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
import workload  # noqa: E402
from paper_2411_15419_b200 import layer as LY  # noqa: E402

cfg = workload.CONFIGS["C2"]
inp = workload.make_layer_inputs(cfg)
dev = torch.device("cuda")
bf = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev, torch.bfloat16)
x, dy = bf(inp["X"]), bf(inp["dY"])
W1, W2, _ = workload.make_expert_weights(cfg)
w1, w2 = bf(W1), bf(W2)
wg = torch.from_numpy(inp["Wg"]).to(dev)
lay = LY.CondensedMoELayer(cfg.num_experts, cfg.top_k, cfg.d_model, cfg.d_ffn, max_tokens=x.shape[0], device=dev)


def step():
    lay.forward(x, wg, w1, w2, None, h=cfg.h)
    lay.backward(dy, x, wg, w1, w2, None)


for _ in range(5):
    step()
torch.cuda.synchronize()
pr = cProfile.Profile()
pr.enable()
for _ in range(50):
    step()
pr.disable()
torch.cuda.synchronize()
st = pstats.Stats(pr)
st.sort_stats("tottime").print_stats(25)
