"""torchrun worker: CUDA-graph replay of world > 1 layer steps (tests/test_gpu_multirank.py).

Every rank runs the C2-shaped layer (world = N) eagerly for two steps on fixed inputs, then captures two
consecutive steps as CUDA graphs (the receive buffers alternate by step parity; the exchange flags carry
the device step number luffy_route advances) and replays them alternately; after every replay Y, dX, dW1
and dW_g must equal the eager step's bitwise (deterministic kernels, same inputs).  Exit 0 = pass."""
import dataclasses
import json
import os
import sys

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))
sys.path.insert(0, ROOT)
sys.path.insert(0, os.path.join(ROOT, "tests"))

import numpy as np  # noqa: E402
import torch  # noqa: E402
import torch.distributed as dist  # noqa: E402

import workload  # noqa: E402


def main():
    rank, world = int(os.environ["RANK"]), int(os.environ["WORLD_SIZE"])
    torch.cuda.set_device(int(os.environ.get("LOCAL_RANK", rank)))
    dist.init_process_group("nccl")
    from paper_2411_15419_b200 import layer as LY
    cfg = dataclasses.replace(workload.CONFIGS["C2"], seqs_per_rank=2)
    inp = workload.make_layer_inputs(cfg, rank=rank)
    E, El = cfg.num_experts, cfg.num_experts // world
    dev = torch.device("cuda")
    bf = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev, torch.bfloat16)
    x, dy = bf(inp["X"]), bf(inp["dY"])
    W1, W2, _ = workload.make_expert_weights(cfg, experts=range(rank * El, (rank + 1) * El))
    w1, w2 = bf(W1), bf(W2)
    wg = torch.from_numpy(inp["Wg"]).to(dev)
    T = x.shape[0]
    lay = LY.CondensedMoELayer(E, cfg.top_k, cfg.d_model, cfg.d_ffn, max_tokens=T, world=world, rank=rank, device=dev)

    def step():
        y = lay.forward(x, wg, w1, w2, None, h=cfg.h)
        g = lay.backward(dy, x, wg, w1, w2, None)
        return y, g

    def snap(y, g):
        return [y.clone(), g["dx"].clone(), g["dw1"].clone(), g["dwg"].clone()]

    ref = None
    for _ in range(2):
        y, g = step()
        torch.cuda.synchronize()
        cur = snap(y, g)
        if ref is None:
            ref = cur
        assert all(torch.equal(a, b) for a, b in zip(ref, cur)), "eager steps differ"
    cap = torch.cuda.Stream()
    cap.wait_stream(torch.cuda.current_stream())
    graphs = []
    with torch.cuda.stream(cap):
        for _ in range(2):
            gr = torch.cuda.CUDAGraph()
            with torch.cuda.graph(gr, stream=cap):
                y, g = step()
            graphs.append(gr)
    torch.cuda.current_stream().wait_stream(cap)
    dist.barrier()
    ok = True
    for i in range(6):
        graphs[i % 2].replay()
        torch.cuda.synchronize()
        cur = snap(y, g)
        ok = ok and all(torch.equal(a, b) for a, b in zip(ref, cur))
    dist.barrier()
    print(json.dumps({"rank": rank, "ok": bool(ok), "replays": 6}), flush=True)
    lay.close()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
