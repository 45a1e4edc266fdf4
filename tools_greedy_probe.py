"""Probe: per-phase timeline of the greedy cluster kernel (largest group) on the bench workload."""
import sys
import numpy as np, torch, workload
from paper_2411_15419_b200 import layer as LY, luffy as L
cfg = workload.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
inp = workload.make_layer_inputs(cfg)
T = inp["X"].shape[0]
lay = LY.CondensedMoELayer(cfg.num_experts, cfg.top_k, cfg.d_model, cfg.d_ffn, max_tokens=T)
bf = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to("cuda", torch.bfloat16)
x = bf(inp["X"]); wg = torch.from_numpy(inp["Wg"]).cuda()
s = torch.cuda.current_stream().cuda_stream
for it in range(5):
    L.luffy_route(lay.layer, x, wg, T, lay.idx, lay.w, s)
    L.luffy_condense(lay.layer, x, cfg.h, lay.rep, s)
torch.cuda.synchronize()
c = L.luffy_debug_copy(lay.layer, "greedy_times", s)
n = int(c[3]); t = [int(c[8 + 2 * i]) | (int(c[9 + 2 * i]) << 32) for i in range(n)]
print("rounds", int(c[2]), "stamps", n, "deltas_us", [round((t[i + 1] - t[i]) / 1e3, 2) for i in range(n - 1)],
      "total_us", round((t[-1] - t[0]) / 1e3, 2) if n > 1 else None)
