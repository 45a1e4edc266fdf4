"""One fwd+bwd of the layer through the C ABI at a small shape, for compute-sanitizer runs:
    compute-sanitizer --tool memcheck python tools/sanitize_step.py C1
(C1: fp32 SIMT path, 4 simulated ranks' first batch; C2S: bf16 tcgen05 path, 1024 tokens)."""
import dataclasses
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import workload  # noqa: E402
from parity_util import run_gpu_layer  # noqa: E402

name = sys.argv[1] if len(sys.argv) > 1 else "C1"
cfg = workload.CONFIGS["C1"] if name == "C1" else dataclasses.replace(workload.CONFIGS["C2"], seqs_per_rank=2)
inp = workload.make_layer_inputs(cfg)
for h in (cfg.h, 1.01):
    res = run_gpu_layer(cfg, inp, h=h)
    print(name, "h", h, "reps", res["stats"].reps, "of", res["stats"].copies, flush=True)
