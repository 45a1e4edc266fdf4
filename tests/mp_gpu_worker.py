"""torchrun worker for the multi-GPU parity test (one process per GPU, NCCL over NVLink).

Every rank runs the condensed MoE layer fwd+bwd through the C ABI with world = N (expert parallel:
E/N experts per rank, dispatch/combine via NCCL) on its own seeded tokens, then checks against the fp64
oracle with the GPU's routing and representative maps frozen: its outputs Y, dX, dW_g and the gradients
of its local experts (summed over the representatives of ALL ranks, gathered with all_gather_object).
Exit code 0 = pass; one JSON line per rank."""
import argparse
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
from oracle import luffy_oracle as O  # noqa: E402


def rel(a, b):
    a = np.asarray(a, np.float64)
    b = np.asarray(b, np.float64)
    den = np.abs(b).max()
    return float(np.abs(a - b).max() / (den if den > 0 else 1.0))


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--config", default="C2S")
    ap.add_argument("--h", type=float, default=0.9)
    ap.add_argument("--migrate", default="none", choices=["none", "plan", "rotate"])
    ap.add_argument("--q", type=int, default=2)
    ap.add_argument("--residual", action="store_true", help="residual block y = x + MoE(x) (luffy_uncondense_residual)")
    ap.add_argument("--uneven", action="store_true", help="different sequence counts per rank (migration)")
    args = ap.parse_args()
    from paper_2411_15419_b200 import layer as LY
    from paper_2411_15419_b200 import luffy as L

    world = int(os.environ["WORLD_SIZE"])
    rank = int(os.environ["RANK"])
    local = int(os.environ["LOCAL_RANK"])
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    dist.init_process_group("nccl", device_id=dev)
    if args.config == "C2S":
        cfg = dataclasses.replace(workload.CONFIGS["C2"], seqs_per_rank=2)
    elif args.config == "C2":
        cfg = workload.CONFIGS["C2"]          # the benched size: T = 8192 per rank
    elif args.config == "C1":
        cfg = workload.CONFIGS["C1"]          # fp32 (SIMT path) through NCCL
    else:
        cfg = dataclasses.replace(workload.CONFIGS[args.config], seqs_per_rank=1, seq_len=512)
    E, El = cfg.num_experts, cfg.num_experts // world
    inp = workload.make_layer_inputs(cfg, rank=rank)
    T = inp["X"].shape[0]
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32
    dt = lambda a: torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev, tdt)
    loc = slice(rank * El, (rank + 1) * El)
    x, dy = dt(inp["X"]), dt(inp["dY"])
    wg = torch.from_numpy(inp["Wg"]).to(dev)
    w1, w2 = dt(inp["W1"][loc]), dt(inp["W2"][loc])
    w3 = dt(inp["W3"][loc]) if inp["W3"] is not None else None
    lay = LY.CondensedMoELayer(E, cfg.top_k, cfg.d_model, cfg.d_ffn, max_tokens=T, dtype=cfg.dtype, act=cfg.act,
                               world=world, rank=rank, device=dev)
    mig = None
    if args.migrate == "none":
        y = lay.forward(x, wg, w1, w2, w3, h=args.h, stats=True, want_rows=True, residual=args.residual)
        g = lay.backward(dy, x, wg, w1, w2, w3, residual=args.residual)
    else:
        # sequences: the workload's own (seqs_per_rank x seq_len), split unevenly to exercise Eq. (1)
        def split(q_):
            L_ = cfg.seq_len
            sl = []
            for _ in range(cfg.seqs_per_rank):
                if args.uneven and q_ % 2 == 1:
                    sl += [L_ // 8, L_ // 8, L_ // 4, L_ // 2]
                else:
                    sl += [L_ // 4, L_ - L_ // 4]
            return sl
        seq_len = split(rank)
        S = len(seq_len)
        counts = [len(split(q_)) for q_ in range(world)]
        forced = None
        if args.migrate == "rotate":
            forced = np.array([((q + 1) % world) for q in range(world) for _ in range(counts[q])], np.int32)
        y, home_rank, home_tok, seq_dest, rows_at = lay.forward_migrated(x, wg, w1, w2, w3, h=args.h, seq_len=seq_len,
                                                                         q=args.q, seq_dest=forced, residual=args.residual,
                                                                         stats=True)
        mig = dict(S=S, seq_len=seq_len, home_rank=home_rank, home_tok=home_tok, seq_dest=seq_dest, rows_at=rows_at,
                   counts=counts, splits=[split(q_) for q_ in range(world)])
        # dY of the hosted tokens, from every home rank's seeded dY
        dys = {q: workload.make_layer_inputs(cfg, rank=q)["dY"] for q in set(home_rank.tolist())}
        dy_out = np.stack([dys[int(h_)][int(t_)] for h_, t_ in zip(home_rank, home_tok)]) if len(home_rank) else \
            np.zeros((0, cfg.d_model), np.float32)
        g = lay.backward(dt(dy_out) if len(dy_out) else dt(np.zeros((1, cfg.d_model), np.float32)), x, wg, w1, w2, w3,
                         residual=args.residual)
    torch.cuda.synchronize()
    idx = lay.idx[:T].cpu().numpy().astype(np.int64)
    rep = lay.rep[:T].cpu().numpy().astype(np.int64)
    # every rank's discrete decisions, to rebuild the expert-side sums
    allmaps = [None] * world
    dist.all_gather_object(allmaps, (idx, rep))
    oracle_Y = {}
    tol = 2e-2 if cfg.dtype == "bf16" else 1e-4
    errs = {}
    dW1 = np.zeros((El,) + inp["W1"].shape[1:])
    dW2 = np.zeros((El,) + inp["W2"].shape[1:])
    for q in range(world):
        iq = workload.make_layer_inputs(cfg, rank=q)
        r = O.route_with_idx(iq["X"], iq["Wg"], allmaps[q][0], cfg.renormalize)
        st = O.layer_forward(iq["X"], iq["Wg"], iq["W1"], iq["W2"], iq["W3"], cfg.top_k, args.h, act=cfg.act,
                             renormalize=cfg.renormalize, routing=r, rep=allmaps[q][1])
        gr = O.layer_backward(st, iq["X"], iq["Wg"], iq["W1"], iq["W2"], iq["W3"], iq["dY"], act=cfg.act,
                              renormalize=cfg.renormalize)
        dW1 += gr.dW1[loc]
        dW2 += gr.dW2[loc]
        # residual block y = x + MoE(x): the identity branch adds x to Y and dY to dX
        oracle_Y[q] = st.Y + (iq["X"] if args.residual else 0.0)
        dX_ref = gr.dX + (iq["dY"] if args.residual else 0.0)
        if mig is not None:
            # K9 pin: distinct representative rows of each of rank q's sequences on each rank
            starts = np.concatenate([[0], np.cumsum(mig["splits"][q])])
            base = int(sum(mig["counts"][:q]))
            for s_ in range(mig["counts"][q]):
                slots = set(st.pk.pos[starts[s_]:starts[s_ + 1]].ravel().tolist())
                owner = [int(st.pk.slot_expert[u]) // El for u in slots]
                exp_rows = np.bincount(owner, minlength=world)
                if not np.array_equal(exp_rows, mig["rows_at"][base + s_]):
                    errs["rows_at"] = 1.0
        if q == rank:
            if mig is None:
                errs["Y"] = rel(y.float().cpu().numpy(), oracle_Y[q])
            errs["dx"] = rel(g["dx"].float().cpu().numpy(), dX_ref)
            errs["dwg"] = rel(g["dwg"].cpu().numpy(), gr.dWg)
            errs["dw"] = rel(g["dw"].cpu().numpy(), gr.dw)
    if mig is not None:
        ref = np.stack([oracle_Y[int(h_)][int(t_)] for h_, t_ in zip(mig["home_rank"], mig["home_tok"])]) \
            if len(mig["home_rank"]) else np.zeros((0, cfg.d_model))
        errs["Y"] = rel(y.float().cpu().numpy(), ref) if len(ref) else 0.0
        errs.setdefault("rows_at", 0.0)
        # the planner on every rank agrees with the oracle's Alg. 1 on the same table
        if args.migrate == "plan":
            lens_all = np.array([v for sl in mig["splits"] for v in sl], np.int64)
            od, _ = O.plan_migration(lens_all, mig["rows_at"], args.q, cfg.d_model * 2, cfg.d_model)
            errs["plan"] = 0.0 if np.array_equal(od, mig["seq_dest"]) else 1.0
    errs["dw1"] = rel(g["dw1"].cpu().numpy(), dW1)
    errs["dw2"] = rel(g["dw2"].cpu().numpy(), dW2)
    # routing exact outside near-ties
    rr = O.route(inp["X"], inp["Wg"], cfg.top_k, cfg.renormalize)
    route_ok = bool(np.array_equal(idx[~rr.near_tie], rr.idx[~rr.near_tie]))
    send_rows, recv_rows = L.luffy_layer_rows(lay.layer)
    ok = route_ok and all(v <= tol for v in errs.values())
    extra = {}
    if mig is not None:
        extra = {"migrated_seqs": int(np.sum(mig["seq_dest"] != np.repeat(np.arange(world), mig["counts"]))),
                 "hosted_tokens": int(len(mig["home_rank"]))}
    print(json.dumps({"rank": rank, "world": world, "ok": ok, "route_ok": route_ok, "errs": errs, **extra,
                      "reps": int(lay.stats.reps) if lay.stats else -1,
                      "copies": int(lay.stats.copies) if lay.stats else -1, "send_rows": send_rows,
                      "recv_rows": recv_rows}), flush=True)
    lay.close()
    dist.barrier()
    dist.destroy_process_group()
    sys.exit(0 if ok else 1)


if __name__ == "__main__":
    main()
