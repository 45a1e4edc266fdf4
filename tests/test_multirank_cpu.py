"""World-size-2 gloo test (CPU) of the N>1 host logic: the exchange plan exported by the C ABI
(luffy_exchange_plan -- the same __host__ __device__ code, csrc/xplan.h, the device count exchange runs)
drives a simulated dispatch (rows pushed to dst_base[e] + slot offset, as the pack-and-push kernel does)
and combine (row r back to (rank_of[r], slot_of[r]), as the GEMM2 epilogue does) over torch.distributed
(gloo); the rows each
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
        plan = L.luffy_exchange_plan(world, rank, E, counts_all)
        send_off, recv_off, dst_base = plan["send_off"], plan["recv_off"], plan["dst_base"]
        send_to, recv_from = plan["send_rows_to"], plan["recv_rows_from"]
        # send layout: padded expert segments of this rank's representatives
        send = np.zeros((send_off[-1], d), np.float32)
        dense = 0
        for e in range(E):
            n = int(pk.counts[e])
            send[send_off[e]:send_off[e] + n] = X[pk.perm[dense:dense + n]]
            dense += n
        # dispatch as the device push does it: send slot s of expert e -> row dst_base[e] + s - send_off[e]
        # of the owner's expert layout (rows and their destination row indices travel over gloo)
        def exchange(out_rows, out_idx):
            """out_rows[p] / out_idx[p]: rows and destination row indices for peer p -> what peers sent me."""
            cnt_out = torch.tensor([len(out_idx[p]) for p in range(world)], dtype=torch.int64)
            cnt_in = [torch.empty(world, dtype=torch.int64) for _ in range(world)]
            dist.all_gather(cnt_in, cnt_out)
            reqs, got = [], {}
            for p in range(world):
                n_in = int(cnt_in[p][rank])
                if p == rank:
                    got[p] = (np.asarray(out_idx[p], np.int64), np.asarray(out_rows[p], np.float32).reshape(-1, d))
                    continue
                if len(out_idx[p]):
                    reqs.append(dist.isend(torch.tensor(np.asarray(out_idx[p], np.int64)), p))
                    reqs.append(dist.isend(torch.from_numpy(np.ascontiguousarray(out_rows[p], np.float32).reshape(-1, d)), p))
                ib, rb = torch.empty(n_in, dtype=torch.int64), torch.empty(n_in, d)
                if n_in:
                    reqs.append(dist.irecv(ib, p))
                    reqs.append(dist.irecv(rb, p))
                got[p] = (ib, rb)
            for rq in reqs:
                rq.wait()
            return {p: (np.asarray(v[0]), np.asarray(v[1])) for p, v in got.items()}

        rows_to = {p: [] for p in range(world)}
        idx_to = {p: [] for p in range(world)}
        for e in range(E):
            p = e // El
            for s_ in range(int(send_off[e]), int(send_off[e]) + int(pk.counts[e])):
                rows_to[p].append(send[s_])
                idx_to[p].append(int(dst_base[e]) + s_ - int(send_off[e]))
        recv = np.zeros((recv_off[-1], d), np.float32)
        for p, (ri, rr) in exchange(rows_to, idx_to).items():
            assert len(ri) == recv_from[p]
            recv[ri] = rr
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
        # combine as the GEMM2 epilogue does it: expert-layout row r -> (rank_of[r], slot_of[r]); returns 2*row
        rank_of, slot_of = plan["rank_of"], plan["slot_of"]
        pad_rows = rank_of < 0
        pad_ok = bool(np.all(slot_of[pad_rows] == -1))
        rows_to = {p: [] for p in range(world)}
        idx_to = {p: [] for p in range(world)}
        for r in np.nonzero(~pad_rows)[0]:
            rows_to[int(rank_of[r])].append(2.0 * recv[r])
            idx_to[int(rank_of[r])].append(int(slot_of[r]))
        gathered_rows = np.zeros_like(send)
        for p, (ri, rr) in exchange(rows_to, idx_to).items():
            assert len(ri) == send_to[p]
            gathered_rows[ri] = rr
        comb_ok = np.array_equal(gathered_rows, 2.0 * send) and pad_ok
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
