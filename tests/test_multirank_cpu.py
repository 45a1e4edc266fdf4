"""World-size-2 gloo test (CPU) of the N>1 host logic: the exchange plan exported by the C ABI
(luffy_exchange_plan) drives a simulated dispatch and combine over torch.distributed (gloo); the rows each
rank receives must be exactly the oracle's receive layout (expert-major, source rank ascending, then the
source's send order; reading R15), padding rows zero, and the combine must return every row to its slot."""
import os
import socket

import numpy as np
import pytest
import torch
import torch.distributed as dist
import torch.multiprocessing as mp

import workload
from oracle import luffy_oracle as O

ALIGN = 128


def _free_port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _rank_state(cfg, rank):
    X, _, _ = workload.make_tokens(cfg, rank=rank)
    Wg = workload.make_gate(cfg)
    r = O.route(X, Wg, cfg.top_k, cfg.renormalize)
    c = O.condense(X, r.idx, cfg.num_experts, cfg.h, keep_s=False)
    pk = O.pack(r.idx, c.rep, cfg.num_experts)
    return X, pk


def _worker(rank, world, port, q):
    os.environ["MASTER_ADDR"] = "127.0.0.1"
    os.environ["MASTER_PORT"] = str(port)
    dist.init_process_group("gloo", rank=rank, world_size=world)
    try:
        import sys
        sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
        from paper_2411_15419_b200 import luffy as L
        cfg = workload.CONFIGS["C1"]
        E, El, d = cfg.num_experts, cfg.num_experts // world, cfg.d_model
        states = [_rank_state(cfg, q_) for q_ in range(world)]  # every rank can rebuild every rank's pack
        X, pk = states[rank]
        cnt = torch.tensor(pk.counts, dtype=torch.int32)
        gathered = [torch.empty_like(cnt) for _ in range(world)]
        dist.all_gather(gathered, cnt)
        counts_all = torch.stack(gathered).numpy()
        send_off, recv_off, send_to, recv_from = L.luffy_exchange_plan(world, rank, E, counts_all)
        # send layout: padded expert segments of this rank's representatives
        send = np.zeros((send_off[-1], d), np.float32)
        dense = 0
        for e in range(E):
            n = int(pk.counts[e])
            send[send_off[e]:send_off[e] + n] = X[pk.perm[dense:dense + n]]
            dense += n
        # dispatch over gloo following the plan
        recv = np.zeros((recv_off[-1], d), np.float32)
        reqs, bufs = [], []
        for p in range(world):
            chunks = [send[send_off[p * El + el]:send_off[p * El + el] + counts_all[rank, p * El + el]] for el in range(El)]
            out = torch.from_numpy(np.ascontiguousarray(np.concatenate(chunks))) if chunks else torch.zeros(0, d)
            assert out.shape[0] == send_to[p]
            inb = torch.empty(int(recv_from[p]), d)
            if p == rank:
                inb.copy_(out)
            else:
                if out.shape[0]:
                    reqs.append(dist.isend(out, p))
                if inb.shape[0]:
                    reqs.append(dist.irecv(inb, p))
            bufs.append(inb)
        for rq in reqs:
            rq.wait()
        for p in range(world):
            o = 0
            for el in range(El):
                e = rank * El + el
                n = int(counts_all[p, e])
                row = recv_off[el] + int(counts_all[:p, e].sum())
                recv[row:row + n] = bufs[p][o:o + n].numpy()
                o += n
        # expected: the oracle's receive layout built from every rank's pack
        blocks, off = O.recv_layout(counts_all.astype(np.int64), rank, E, world)
        exp_rows = []
        for src, e, first, n in blocks:
            Xs, pks = states[src]
            exp_rows.append(Xs[pks.perm[first:first + n]])
        expected = np.concatenate(exp_rows) if exp_rows else np.zeros((0, d))
        got = np.concatenate([recv[recv_off[el]:recv_off[el] + int(counts_all[:, rank * El + el].sum())]
                              for el in range(El)])
        ok = np.array_equal(got, expected.astype(np.float32))
        pad_zero = all(not recv[recv_off[el] + int(counts_all[:, rank * El + el].sum()):recv_off[el + 1]].any()
                       for el in range(El))
        # combine: expert side returns (2 * row) to the source's slots
        ret_send = {p: [] for p in range(world)}
        for el in range(El):
            e = rank * El + el
            for p in range(world):
                row = recv_off[el] + int(counts_all[:p, e].sum())
                ret_send[p].append(2.0 * recv[row:row + int(counts_all[p, e])])
        gathered_rows = np.zeros_like(send)
        reqs, bufs = [], {}
        for p in range(world):
            out = torch.from_numpy(np.ascontiguousarray(np.concatenate(ret_send[p])))
            inb = torch.empty(int(send_to[p]), d)
            if p == rank:
                inb.copy_(out)
            else:
                if out.shape[0]:
                    reqs.append(dist.isend(out, p))
                if inb.shape[0]:
                    reqs.append(dist.irecv(inb, p))
            bufs[p] = inb
        for rq in reqs:
            rq.wait()
        for p in range(world):
            o = 0
            for el in range(El):
                e = p * El + el
                n = int(counts_all[rank, e])
                gathered_rows[send_off[e]:send_off[e] + n] = bufs[p][o:o + n].numpy()
                o += n
        comb_ok = np.array_equal(gathered_rows, 2.0 * send)
        conserve = int(counts_all.sum())
        q.put((rank, bool(ok), bool(pad_zero), bool(comb_ok), int(recv_from.sum()), conserve))
    finally:
        dist.destroy_process_group()


def test_exchange_plan_world2_gloo():
    from paper_2411_15419_b200 import build
    build.build()
    world = 2
    ctx = mp.get_context("spawn")
    q = ctx.Queue()
    port = _free_port()
    procs = [ctx.Process(target=_worker, args=(r, world, port, q)) for r in range(world)]
    for p in procs:
        p.start()
    res = [q.get(timeout=300) for _ in range(world)]
    for p in procs:
        p.join(timeout=60)
        assert p.exitcode == 0
    total = 0
    for rank, ok, pad_zero, comb_ok, recv_rows, conserve in sorted(res):
        assert ok, f"rank {rank}: received rows differ from the oracle receive layout"
        assert pad_zero, f"rank {rank}: padding rows not zero"
        assert comb_ok, f"rank {rank}: combine did not return every row to its slot"
        total += recv_rows
    assert total == res[0][5]   # rows are conserved through the exchange
