"""GPU parity of the fast similarity measurement with history shortcuts (§8(f) NEXT #1):
two consecutive blocks A -> B on the same tokens, each a luffy layer created with fast_measure; B takes
its history from A (luffy_layer_set_history).  Oracle: condense_fast (oracle/luffy_oracle.py).

Checked, following reading R18's exclusion discipline for threshold-like decisions:
  * A's recorded classification (finalized weight > S1, < S2) equals the oracle's for every pair whose
    fp64 similarity is more than 1e-5 from S1 and S2;
  * B's decided pairs (weight 1 / weight 0 by history) equal the oracle's shortcut sets for EVERY pair,
    with the oracle's history being A's fp64 weights except that pairs within 1e-5 of S1 / S2 take A's
    GPU class (the override of R18, extended to the S1 / S2 thresholds);
  * B's adjacency equals the oracle's threshold graph of its finalized weights off the h band, and B's
    representative map equals the oracle's exactly (h-band decisions taken from the GPU);
  * B's outputs and gradients within the bf16 tolerance; skipped Gram tiles when a whole tile is decided.
"""
import dataclasses

import numpy as np
import pytest
import torch

import workload
from oracle import luffy_oracle as O
from parity_util import run_gpu_layer
from test_gpu_parity import _check_layout, _check_numerics, _check_route

pytestmark = pytest.mark.gpu
BAND = 1e-5


def group_bits(arr, res, e):
    goff, gcnt = res["goff"], res["gcnt"]
    npad, n = int(goff[e + 1] - goff[e]), int(gcnt[e])
    if npad == 0:
        return np.zeros((0, 0), bool)
    W = npad // 32
    o = int(res["adjoff"][e])
    words = arr[o:o + npad * W].reshape(npad, W)
    bits = np.unpackbits(words.view(np.uint8).reshape(npad, W, 4), axis=2, bitorder="little")
    return bits.reshape(npad, npad)[:n, :n].astype(bool)


def _fetch_hist(lay, res):
    from paper_2411_15419_b200 import luffy as L
    s = torch.cuda.current_stream().cuda_stream
    for item in ("hone", "hzero", "dec1", "dec0", "tskip"):
        res[item] = L.luffy_debug_copy(lay.layer, item, s)
    return res


def _layers(cfg, T):
    from paper_2411_15419_b200 import layer as LY
    mk = lambda: LY.CondensedMoELayer(cfg.num_experts, cfg.top_k, cfg.d_model, cfg.d_ffn, max_tokens=T,
                                      dtype=cfg.dtype, act=cfg.act, fast_measure=True)
    return mk(), mk()


def run_two_blocks(cfg, inpA, inpB, h, S1, S2):
    T = inpA["X"].shape[0]
    A, B = _layers(cfg, T)
    A.set_history(None, S1, S2)
    B.set_history(A, S1, S2)
    resA = _fetch_hist(A, run_gpu_layer(cfg, inpA, h=h, layer=A, backward=False))
    resB = _fetch_hist(B, run_gpu_layer(cfg, inpB, h=h, layer=B, backward=True))
    return A, B, resA, resB


def check_two_blocks(cfg, inpA, inpB, resA, resB, h, S1, S2):
    T = resA["T"]
    E = cfg.num_experts
    XA, XB = inpA["X"][:T], inpB["X"][:T]
    # ---- block A: classification of its (computed) weights
    cA, HA, ncA = O.condense_fast(XA, resA["idx"], E, h, np.full((T, T), np.nan), S1, S2)
    gpu_class = np.full((T, T), np.nan)   # A's GPU class per token pair: 1 / 0 / 0.5*(S1+S2)
    band_S = 0
    for e, (t, j) in enumerate(cA.groups):
        if t.size == 0:
            continue
        W = HA[np.ix_(t, t)]
        g1, g0 = group_bits(resA["hone"], resA, e), group_bits(resA["hzero"], resA, e)
        with np.errstate(invalid="ignore"):
            o1, o0 = W > S1, W < S2
            near = (np.abs(W - S1) <= BAND) | (np.abs(W - S2) <= BAND)
        np.fill_diagonal(o1, False)
        np.fill_diagonal(o0, False)
        assert not ((g1 != o1) & ~near).any(), f"A: > S1 class differs off the band (group {e})"
        assert not ((g0 != o0) & ~near).any(), f"A: < S2 class differs off the band (group {e})"
        band_S += int(np.triu(near, 1).sum())
        cls = np.where(g1, 1.0, np.where(g0, 0.0, 0.5 * (S1 + S2)))
        cls[np.isnan(W)] = np.nan
        sub = gpu_class[np.ix_(t, t)]
        gpu_class[np.ix_(t, t)] = np.where(np.isnan(sub), cls, sub)
    # oracle history for B: A's fp64 weights, band pairs (S1 / S2) replaced by A's GPU class
    with np.errstate(invalid="ignore"):
        nearS = (np.abs(HA - S1) <= BAND) | (np.abs(HA - S2) <= BAND)
    H = np.where(nearS, gpu_class, HA)
    # ---- block B
    groups = O.group_members(resB["idx"], E)
    overrides, n_dec, n_comp, n_hband = [], 0, 0, 0
    for e, (t, j) in enumerate(groups):
        n = t.size
        if n == 0:
            overrides.append(None)
            continue
        Wb, comp = O.fast_measure(XB[t], H[np.ix_(t, t)], S1, S2)
        with np.errstate(invalid="ignore"):
            s1, s0 = H[np.ix_(t, t)] > S1, H[np.ix_(t, t)] < S2
        valid = ~np.isnan(Wb)
        d1, d0 = group_bits(resB["dec1"], resB, e), group_bits(resB["dec0"], resB, e)
        np.fill_diagonal(s1, False)
        np.fill_diagonal(s0, False)
        assert np.array_equal(d1 & valid, s1 & valid), f"B: weight-1 shortcuts differ (group {e})"
        assert np.array_equal(d0 & valid, s0 & valid), f"B: weight-0 shortcuts differ (group {e})"
        n_dec += int(np.triu((s1 | s0) & valid, 1).sum())
        n_comp += int(np.triu(comp, 1).sum())
        ref = O.threshold_graph(Wb, h)
        gpu = group_bits(resB["adj"], resB, e)
        assert np.array_equal(gpu, gpu.T)
        with np.errstate(invalid="ignore"):
            inband = comp & (np.abs(Wb - h) <= BAND)
        assert not ((gpu != ref) & ~inband).any(), f"B: edges differ off the h band (group {e})"
        n_hband += int(np.triu(inband, 1).sum())
        overrides.append(np.where(inband, gpu, ref))
        # B's own classification for the next block: shortcut values included (R21)
        h1, h0 = group_bits(resB["hone"], resB, e), group_bits(resB["hzero"], resB, e)
        with np.errstate(invalid="ignore"):
            nearB = comp & ((np.abs(Wb - S1) <= BAND) | (np.abs(Wb - S2) <= BAND))
            e1, e0 = (Wb > S1) & valid, (Wb < S2) & valid
        assert not ((h1 != e1) & ~nearB).any() and not ((h0 != e0) & ~nearB).any(), f"B: class (group {e})"
    cB, _, nc = O.condense_fast(XB, resB["idx"], E, h, H, S1, S2, adjacency_override=overrides)
    assert np.array_equal(cB.rep, resB["rep"]), "B: representative map differs from the oracle"
    assert nc == n_comp
    st = resB["stats"]
    assert int(st.decided_pairs) == n_dec, (int(st.decided_pairs), n_dec)
    return dict(decided=n_dec, computed=n_comp, band_S=band_S, band_h=n_hband,
                skipped=int(st.skipped_tiles), reps=int(st.reps), copies=int(st.copies))


def _perturbed(cfg, inp, sigma, seed, gate_noise):
    rng = np.random.default_rng(seed)
    X = inp["X"] + sigma * rng.standard_normal(inp["X"].shape).astype(np.float32)
    X = workload.bf16_round(X) if cfg.dtype == "bf16" else X.astype(np.float32)
    Wg = inp["Wg"] + gate_noise * rng.standard_normal(inp["Wg"].shape).astype(np.float32)
    dY = workload.make_grad_out(cfg, X.shape[0], rank=1)
    return dict(inp, X=X, Wg=Wg.astype(np.float32), dY=dY)


@pytest.mark.parametrize("S1,S2", [(0.9, 0.55), (0.8, 0.2)])
def test_history_two_blocks(S1, S2):
    cfg = dataclasses.replace(workload.CONFIGS["C2"], seqs_per_rank=2, d_ffn=1024)
    inpA = workload.make_layer_inputs(cfg)
    inpB = _perturbed(cfg, inpA, 0.05, 7, 0.002)
    A, B, resA, resB = run_two_blocks(cfg, inpA, inpB, 0.9, S1, S2)
    rep = check_two_blocks(cfg, inpA, inpB, resA, resB, 0.9, S1, S2)
    _check_route(cfg, inpB, resB)
    _check_layout(cfg, inpB, resB)
    errs = _check_numerics(cfg, inpB, resB, 0.9)
    print(f"\n[history S1={S1} S2={S2}] {rep} errs={errs}")
    assert rep["decided"] > 0
    A.close(), B.close()


def test_history_skips_decided_tiles():
    """A group whose first 600 rows are near-duplicates: in block B every pair among them is decided
    (weight 1), so the Gram tiles covering only those rows are skipped -- results stay exact."""
    cfg = dataclasses.replace(workload.CONFIGS["C2"], num_experts=4, top_k=1, seqs_per_rank=2, d_ffn=1024)
    inpA = workload.make_layer_inputs(cfg)
    rng = np.random.default_rng(2)
    X = inpA["X"].copy()
    v = rng.standard_normal(cfg.d_model)
    dup = np.arange(600)
    X[dup] = np.sqrt(cfg.d_model) * (v / np.linalg.norm(v)) + 0.05 * rng.standard_normal((600, cfg.d_model))
    Wg = inpA["Wg"].copy()
    Wg[0] = 4.0 * v / np.linalg.norm(v) / np.sqrt(cfg.d_model) * 8
    X = workload.bf16_round(X.astype(np.float32))
    inpA = dict(inpA, X=X, Wg=Wg.astype(np.float32))
    inpB = _perturbed(cfg, inpA, 0.02, 9, 0.0)
    A, B, resA, resB = run_two_blocks(cfg, inpA, inpB, 0.9, 0.8, 0.2)
    assert (resB["idx"][dup, 0] == 0).all()
    rep = check_two_blocks(cfg, inpA, inpB, resA, resB, 0.9, 0.8, 0.2)
    _check_numerics(cfg, inpB, resB, 0.9)
    print(f"\n[history tiles] {rep} tskip={resB['tskip'].tolist()[:12]}")
    assert rep["skipped"] >= 2 and int(resB["tskip"].sum()) == rep["skipped"]
    A.close(), B.close()


def test_history_disabled_equals_plain():
    """S1 = 1, S2 = 0 decides nothing: block B equals the plain layer bitwise (same kernels' results)."""
    cfg = dataclasses.replace(workload.CONFIGS["C2"], seqs_per_rank=1, d_ffn=1024)
    inpA = workload.make_layer_inputs(cfg)
    inpB = _perturbed(cfg, inpA, 0.05, 3, 0.0)
    A, B, resA, resB = run_two_blocks(cfg, inpA, inpB, 0.9, 1.0, 0.0)
    plain = run_gpu_layer(cfg, inpB, h=0.9)
    assert int(resB["stats"].decided_pairs) == 0 and int(resB["stats"].skipped_tiles) == 0
    for k in ("rep", "Y", "dx", "dw1", "dw2", "dwg"):
        assert np.array_equal(resB[k], plain[k]), k
    A.close(), B.close()
