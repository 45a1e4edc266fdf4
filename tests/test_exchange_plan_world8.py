"""The shipped exchange plan (luffy_exchange_plan = csrc/xplan.h, the code the device count exchange runs)
at world 4 and 8, one process: every rank's plan is computed from the same all-gathered counts, the
dispatch is simulated as the push kernel does it (send slot s of expert e -> the owner's row
dst_base[e] + s - send_off[e]) and the combine as the GEMM2 epilogue does it (expert-layout row r ->
(rank_of[r], slot_of[r])).  Every owner must receive exactly the oracle's receive layout (reading R15) with
zero padding, every source must get each row back in its slot, and E / P = 1 (one expert per rank, the
C2 layer at 8 GPUs) is covered.  CPU only (no GPU needed: host code of libluffy.so)."""
import dataclasses

import numpy as np
import pytest

import workload
from oracle import luffy_oracle as O


def _packs(cfg, world):
    out = []
    for r in range(world):
        X, _, _ = workload.make_tokens(cfg, rank=r)
        Wg = workload.make_gate(cfg)
        rt = O.route(X, Wg, cfg.top_k, cfg.renormalize)
        c = O.condense(X, rt.idx, cfg.num_experts, cfg.h, keep_s=False)
        out.append((X, O.pack(rt.idx, c.rep, cfg.num_experts)))
    return out


@pytest.mark.parametrize("world,E", [(4, 8), (8, 8), (8, 16)])
def test_exchange_plan_many_ranks(world, E):
    from paper_2411_15419_b200 import build
    build.build()
    from paper_2411_15419_b200 import luffy as L
    cfg = dataclasses.replace(workload.CONFIGS["C1"], num_experts=E, d_model=64, seqs_per_rank=2, seq_len=96)
    El, d = E // world, cfg.d_model
    st = _packs(cfg, world)
    counts_all = np.stack([pk.counts for _, pk in st]).astype(np.int32)
    plans = [L.luffy_exchange_plan(world, r, E, counts_all) for r in range(world)]
    recv = [np.zeros((plans[r]["recv_off"][-1], d)) for r in range(world)]
    sends = []
    for s, (X, pk) in enumerate(st):
        so, db = plans[s]["send_off"], plans[s]["dst_base"]
        send = np.zeros((so[-1], d))
        dense = 0
        for e in range(E):
            n = int(pk.counts[e])
            send[so[e]:so[e] + n] = X[pk.perm[dense:dense + n]]
            for i in range(n):
                recv[e // El][int(db[e]) + i] = send[so[e] + i]
            dense += n
        sends.append(send)
    for r in range(world):
        ro = plans[r]["recv_off"]
        blocks, _ = O.recv_layout(counts_all.astype(np.int64), r, E, world)
        exp = [st[src][0][st[src][1].perm[first:first + n]] for src, e, first, n in blocks]
        exp = np.concatenate(exp) if exp else np.zeros((0, d))
        got_parts, pad_zero = [], True
        for el in range(El):
            n = int(counts_all[:, r * El + el].sum())
            got_parts.append(recv[r][ro[el]:ro[el] + n])
            pad_zero &= not recv[r][ro[el] + n:ro[el + 1]].any()
        assert np.array_equal(np.concatenate(got_parts), exp), (world, r)
        assert pad_zero
    back = [np.zeros_like(s) for s in sends]
    for r in range(world):
        rank_of, slot_of = plans[r]["rank_of"], plans[r]["slot_of"]
        for row in range(plans[r]["recv_off"][-1]):
            if rank_of[row] < 0:
                assert slot_of[row] == -1
                continue
            back[int(rank_of[row])][int(slot_of[row])] = 2.0 * recv[r][row]
    for s in range(world):
        assert np.array_equal(back[s], 2.0 * sends[s])
    assert sum(int(p["recv_rows_from"].sum()) for p in plans) == int(counts_all.sum())
