"""Helpers for the GPU parity tests: run the CUDA path through the C ABI and bring its results (and its
internal layout arrays) to the host; compare with the oracle."""
from __future__ import annotations

import numpy as np
import torch

import workload
from oracle import luffy_oracle as O

ROW_ALIGN = 128


def rel_err(gpu, ref) -> float:
    gpu = np.asarray(gpu, np.float64)
    ref = np.asarray(ref, np.float64)
    den = np.abs(ref).max()
    return float(np.abs(gpu - ref).max() / (den if den > 0 else 1.0))


def tol_for(dtype: str) -> float:
    return 1e-4 if dtype == "fp32" else 2e-2


def to_dev(a: np.ndarray, dtype: str):
    t = torch.from_numpy(np.ascontiguousarray(a, np.float32))
    return t.to("cuda", torch.bfloat16 if dtype == "bf16" else torch.float32)


def run_gpu_layer(cfg: workload.LayerConfig, inp: dict, h: float, T: int | None = None, backward: bool = True,
                  layer=None, gram_dump: bool = False):
    """One fwd(+bwd) of the CUDA path at world == 1; returns host arrays and debug exports (with
    gram_dump: the fp32 Gram the threshold was applied to, per group, via luffy_debug_gram_dump)."""
    from paper_2411_15419_b200 import layer as LY
    from paper_2411_15419_b200 import luffy as L
    X = inp["X"] if T is None else inp["X"][:T]
    T = X.shape[0]
    if layer is None:
        layer = LY.CondensedMoELayer(cfg.num_experts, cfg.top_k, cfg.d_model, cfg.d_ffn, max_tokens=T,
                                     dtype=cfg.dtype, act=cfg.act)
    x = to_dev(X, cfg.dtype)
    wg = torch.from_numpy(inp["Wg"]).cuda()
    w1 = to_dev(inp["W1"], cfg.dtype)
    w2 = to_dev(inp["W2"], cfg.dtype)
    w3 = to_dev(inp["W3"], cfg.dtype) if inp["W3"] is not None else None
    gbuf = None
    if gram_dump:
        C = T * cfg.top_k + cfg.num_experts * ROW_ALIGN
        gbuf = torch.full((C * C,), float("nan"), dtype=torch.float32, device="cuda")
        L.luffy_debug_gram_dump(layer.layer, gbuf)
    y = layer.forward(x, wg, w1, w2, w3, h=h, stats=True)
    s = torch.cuda.current_stream().cuda_stream
    res = dict(layer=layer, T=T, idx=layer.idx[:T].cpu().numpy().astype(np.int64),
               w=layer.w[:T].cpu().numpy().astype(np.float64), rep=layer.rep[:T].cpu().numpy().astype(np.int64),
               Y=y.float().cpu().numpy().astype(np.float64), stats=layer.stats)
    for item in ("gcnt", "goff", "gtok", "rep_local", "soff", "perm", "pos", "nrep", "rounds"):
        res[item] = L.luffy_debug_copy(layer.layer, item, s)
    if h <= 1.0:
        res["adjoff"] = L.luffy_debug_copy(layer.layer, "adjoff", s)
        res["adj"] = L.luffy_debug_copy(layer.layer, "adj", s)
    res["recv"] = layer.recv.float().cpu().numpy()
    if gbuf is not None:
        L.luffy_debug_gram_dump(layer.layer, None)
        torch.cuda.synchronize()
        nfl = int(res["adjoff"][-1]) * 32
        res["gram"] = gbuf[:nfl].cpu().numpy()
        del gbuf
    if backward:
        dY = inp["dY"][:T]
        g = layer.backward(to_dev(dY, cfg.dtype), x, wg, w1, w2, w3)
        torch.cuda.synchronize()
        for k_, v in g.items():
            if v is not None:
                res[k_] = v.float().cpu().numpy().astype(np.float64)
    return res


def group_adjacency(res, e: int) -> np.ndarray:
    """Bool adjacency [n_e, n_e] of group e from the GPU's bit matrix."""
    goff, gcnt = res["goff"], res["gcnt"]
    npad = int(goff[e + 1] - goff[e])
    n = int(gcnt[e])
    if npad == 0:
        return np.zeros((0, 0), bool)
    W = npad // 32
    words = res["adj"][int(res["adjoff"][e]):int(res["adjoff"][e]) + npad * W].reshape(npad, W)
    bits = np.unpackbits(words.view(np.uint8).reshape(npad, W, 4), axis=2, bitorder="little")
    return bits.reshape(npad, npad)[:n, :n].astype(bool)


def group_gram(res, e: int) -> np.ndarray:
    """fp32 Gram [n_e, n_e] of group e from the debug dump (upper 32x32 blocks written; mirrored here)."""
    goff, gcnt = res["goff"], res["gcnt"]
    npad = int(goff[e + 1] - goff[e])
    n = int(gcnt[e])
    o = int(res["adjoff"][e]) * 32
    G = res["gram"][o:o + npad * npad].reshape(npad, npad).astype(np.float64)
    blk = np.arange(npad) // 32
    upper = blk[None, :] >= blk[:, None]
    G = np.where(upper, G, G.T)
    return G[:n, :n]


def dense_perm(res, E: int):
    """(expert, token) of every representative in the GPU's send order, padding removed."""
    soff, nrep, perm = res["soff"], res["nrep"], res["perm"]
    out = []
    for e in range(E):
        for s in range(int(soff[e]), int(soff[e]) + int(nrep[e])):
            out.append((e, int(perm[s])))
    return out


def oracle_frozen(cfg, inp, res, h):
    """Oracle forward/backward with the GPU's discrete decisions (idx, rep) frozen (R2, R18)."""
    T = res["T"]
    X = inp["X"][:T]
    r = O.route_with_idx(X, inp["Wg"], res["idx"], cfg.renormalize)
    st = O.layer_forward(X, inp["Wg"], inp["W1"], inp["W2"], inp["W3"], cfg.top_k, h, act=cfg.act,
                         renormalize=cfg.renormalize, routing=r, rep=res["rep"])
    g = O.layer_backward(st, X, inp["Wg"], inp["W1"], inp["W2"], inp["W3"], inp["dY"][:T], act=cfg.act,
                         renormalize=cfg.renormalize)
    return st, g
