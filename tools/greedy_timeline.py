"""Phase timeline of the representative selection (greedy cluster kernel) for the largest group of one
C2 condense: the %globaltimer stamps of LUFFY_DBG_GREEDY_TIMES (rank 0 CTA of that group's cluster):
stamp 0 = start, 1 = replicas and own rows cached, then 4 per round (after phases A, B, C, D)."""
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))
import numpy as np  # noqa: E402
import torch  # noqa: E402

import workload  # noqa: E402
from parity_util import run_gpu_layer  # noqa: E402

cfg = workload.CONFIGS[sys.argv[1] if len(sys.argv) > 1 else "C2"]
inp = workload.make_layer_inputs(cfg)
from paper_2411_15419_b200 import luffy as L  # noqa: E402
res = run_gpu_layer(cfg, inp, h=cfg.h, backward=False)
lay = res["layer"]
for _ in range(3):
    lay.forward(torch.from_numpy(inp["X"]).cuda().to(torch.bfloat16), torch.from_numpy(inp["Wg"]).cuda(),
                torch.from_numpy(inp["W1"]).cuda().to(torch.bfloat16), torch.from_numpy(inp["W2"]).cuda().to(torch.bfloat16),
                None, h=cfg.h)
torch.cuda.synchronize()
c = L.luffy_debug_copy(lay.layer, "greedy_times", torch.cuda.current_stream().cuda_stream)
n = int(c[3])
t = np.array([int(c[8 + 2 * i]) | (int(c[9 + 2 * i]) << 32) for i in range(n)], np.int64)
print(cfg.name, "groups", res["gcnt"].tolist(), "rounds", int(res["rounds"][0]))
print("stamps (us from start):", [round((v - t[0]) / 1e3, 2) for v in t])
print("deltas (us):", [round((b - a) / 1e3, 2) for a, b in zip(t, t[1:])])
