"""Luffy oracle: a plain, slow, fp64 CPU implementation of the token-condensed expert-parallel MoE layer.

TEST INFRASTRUCTURE ONLY.  Only `tests/`, `__graft_entry__.smoke()` and `bench.py`'s cpu_baseline /
`--impl reference` legs may import this module.  It shares no code with the CUDA path
(`paper_2411_15419_b200/`), and nothing here imports that package.

Citations: `P:n` = PAPER.md line n (arXiv 2411.15419, LaTeX source), `S:n` = SPEC.md line n.
Readings of passages the paper leaves silent or garbled are the DESIGN.md §2 readings R1-R19
(same numbering as SURVEY.md §8c A1-A19).

Everything is fp64 from the exact input values (bf16-representable floats for bf16 configs), with no
intermediate rounding (reading R13).  Library primitives used as single steps: numpy matmul, exp, erf
(via math.erf), argsort.

Parity status per function (what pins it, tests/test_oracle_*.py):
  attention_cost        pinned: SPEC worked values 5, 2048; closed-form scaling laws
  adaptive_threshold    pinned: 0.5, 0.26894, 0.37754; c = 2 (reading R17): the same values x 2
  route                 pinned: torch.topk / torch.softmax on fp64 logits; brute force E<=4; sum(w)=1
  normalized_cosine     pinned: s(u,u)=1, s(u,-u)=0, orthogonal=0.5; numpy Gram
  greedy_condense       pinned: SPEC star / two triangles / identity; path 0-1-2-4-3
                        (SURVEY App. A); brute-force enumeration of the dynamic-degree greedy on tiny
                        graphs; soundness / idempotence / coverage invariants.  The CHOICE of the
                        dynamic-degree reading (R8) is not discriminated by the paper: "parity
                        unpinned" for that reading only (R8).
  fast_measure /        pinned: shortcut set == {s_prev > S1} U {s_prev < S2} and computed weights ==
  condense_fast         all-pairs cosine (1e-12); S1=1, S2=0 or empty history == condense(); SPEC rule
                        examples; a pair-loop brute force on tiny groups
  band_components       pinned: hand-built graphs (paths, triangles, singletons) and 200 random graphs vs
                        a transitive-closure reference (tests/test_oracle_pins.py::test_band_components_pins)
  pack / recv_layout    pinned: conservation, stable order == sorted() brute force
  expert_ffn            pinned: dense torch fp64 matmul + torch GeLU(erf) / SiLU
  layer_forward/backward pinned: h>1 equals a looped dense top-k MoE under torch fp64 autograd;
                        condensed backward equals torch fp64 autograd of the frozen-map forward and
                        central finite differences
  plan_migration        pinned: SPEC values 7888 / 8688 / [1,2] / 64,192; exhaustive
                        single-sequence argmin; q=1 => argmin f; candidate dominance; capacity
"""
from __future__ import annotations

import math
from dataclasses import dataclass, field

import numpy as np

# ----------------------------------------------------------------------------------------------
# Eq. (1) and Eq. (2)
# ----------------------------------------------------------------------------------------------


def attention_cost(B: int, L: int, d: int, P: int = 1):
    """Eq. (1): T_att(B, L) = (3 B L d^2 + 2 B L^2 d) / P.

    Exact integer arithmetic when P == 1 (reading R16: P cancels on a homogeneous box)."""
    num = 3 * B * L * d * d + 2 * B * L * L * d
    return num if P == 1 else num / P


def adaptive_threshold(l_ini: float, l_prev: float, c: float = 1.0) -> float:
    """Eq. (2): h_t = c/(1+exp(l_norm)), l_norm = (l_ini - l_prev)/l_ini; c = 1 as printed.

    Reading R17: the driver uses c = 2, h in (0.538, 1] -- the printed c = 1 confines h to
    (0.269, 0.5], contradicting "a high threshold" early in training and Table IV (adaptive keeps
    accuracy that a static 0.3 loses and beats a static 0.8).  l_prev > l_ini clamps l_norm to 0."""
    if l_ini <= 0:
        raise ValueError("l_ini must be > 0")
    l_norm = max(0.0, (l_ini - l_prev) / l_ini)
    return c / (1.0 + math.exp(l_norm))


# ----------------------------------------------------------------------------------------------
# Step 1: top-k gate ("top-2 gating"; reading R1, R2)
# ----------------------------------------------------------------------------------------------


@dataclass
class Routing:
    logits: np.ndarray      # [T, E] fp64
    probs: np.ndarray       # [T, E] fp64 softmax over all experts
    idx: np.ndarray         # [T, k] int64, ordered by (logit desc, expert asc)
    w: np.ndarray           # [T, k] fp64 gate weights
    near_tie: np.ndarray    # [T] bool: a top-(k+1) ordering decision within 1e-5*max(1,|l|)


def route(X: np.ndarray, Wg: np.ndarray, k: int, renormalize: bool, tie_tol: float = 1e-5) -> Routing:
    """Top-k gate.  logits = X W_g^T; p = softmax(logits); experts ordered by (logit desc, id asc);
    w_k = exp(l_k) / sum_{j in top-k} exp(l_j) when renormalizing (k>1, R1), else p_{e_k}."""
    X = np.asarray(X, np.float64)
    Wg = np.asarray(Wg, np.float64)
    T, E = X.shape[0], Wg.shape[0]
    if not (1 <= k <= E):
        raise ValueError("need 1 <= top_k <= num_experts")
    logits = X @ Wg.T
    m = logits.max(axis=1, keepdims=True)
    ex = np.exp(logits - m)
    probs = ex / ex.sum(axis=1, keepdims=True)
    # stable sort on -logit keeps the lower expert id first among equal logits (R2)
    order = np.argsort(-logits, axis=1, kind="stable")
    idx = order[:, :k].copy()
    sel = np.take_along_axis(logits, idx, axis=1)
    if renormalize:
        es = np.exp(sel - sel.max(axis=1, keepdims=True))
        w = es / es.sum(axis=1, keepdims=True)
    else:
        w = np.take_along_axis(probs, idx, axis=1)
    # near ties among the first min(k+1, E) sorted logits
    srt = np.take_along_axis(logits, order[:, :min(k + 1, E)], axis=1)
    tol = tie_tol * np.maximum(1.0, np.abs(srt[:, :1]))
    gaps = srt[:, :-1] - srt[:, 1:]
    near_tie = (gaps <= tol).any(axis=1) if gaps.shape[1] else np.zeros(T, bool)
    return Routing(logits, probs, idx, w, near_tie)


def route_with_idx(X: np.ndarray, Wg: np.ndarray, idx: np.ndarray, renormalize: bool) -> Routing:
    """The gate of `route` with the expert selection `idx` given (the GPU's choice on near-tie tokens,
    reading R2): same logits, softmax and weight formulas."""
    X = np.asarray(X, np.float64)
    logits = X @ np.asarray(Wg, np.float64).T
    m = logits.max(axis=1, keepdims=True)
    ex = np.exp(logits - m)
    probs = ex / ex.sum(axis=1, keepdims=True)
    idx = np.asarray(idx, np.int64)
    sel = np.take_along_axis(logits, idx, axis=1)
    if renormalize:
        es = np.exp(sel - sel.max(axis=1, keepdims=True))
        w = es / es.sum(axis=1, keepdims=True)
    else:
        w = np.take_along_axis(probs, idx, axis=1)
    return Routing(logits, probs, idx, w, np.zeros(X.shape[0], bool))


# ----------------------------------------------------------------------------------------------
# Steps 2-3: groups, normalized cosine similarity, threshold graph
# ----------------------------------------------------------------------------------------------


def group_members(idx: np.ndarray, E: int):
    """Fast-similarity step 1: only tokens pushed to the same expert are compared.
    Group g(e) = [(t, j) for t ascending with idx[t, j] == e] (reading R6: one group per expert
    and source rank; each of the k copies is condensed in its own expert's group)."""
    groups = []
    for e in range(E):
        t, j = np.nonzero(idx == e)
        order = np.argsort(t, kind="stable")
        groups.append((t[order], j[order]))
    return groups


def normalized_cosine(u: np.ndarray, v: np.ndarray) -> float:
    """P:224 "normalized cosine similarity ... ranges from [0,1]": s = (1 + cos(u, v)) / 2 (R4).
    Zero vectors have no similarity (returns nan; R7)."""
    u = np.asarray(u, np.float64)
    v = np.asarray(v, np.float64)
    nu, nv = math.sqrt(float(u @ u)), math.sqrt(float(v @ v))
    if nu == 0.0 or nv == 0.0:
        return float("nan")
    return (1.0 + float(u @ v) / (nu * nv)) / 2.0


def similarity_matrix(Xg: np.ndarray) -> np.ndarray:
    """Fast-similarity step 3: s_ij = (1 + <x_i,x_j>/(|x_i||x_j|)) / 2 for every pair of the
    group, fp64.  Rows of zero norm get nan (no edges, R7)."""
    Xg = np.asarray(Xg, np.float64)
    G = Xg @ Xg.T
    n = np.sqrt(np.diag(G))
    with np.errstate(divide="ignore", invalid="ignore"):
        s = (1.0 + G / np.outer(n, n)) / 2.0
    s[n == 0.0, :] = np.nan
    s[:, n == 0.0] = np.nan
    return s


def threshold_graph(s: np.ndarray, h: float) -> np.ndarray:
    """P:378 "delete the edges in the graph whose weights are below a given threshold": edge iff
    s_ij >= h, i != j (R4).  nan (zero-norm) never forms an edge (R7)."""
    with np.errstate(invalid="ignore"):
        adj = s >= h
    np.fill_diagonal(adj, False)
    return adj


def greedy_condense(adj: np.ndarray) -> np.ndarray:
    """"For each subgraph, we keep the token with the highest degree for transmission and
    condense its neighboring tokens. We repeat this process until all tokens are condensed."

    Reading R8 (dynamic residual degree, ties -> lowest index): while alive nodes remain,
    u = argmax over alive of (|N(u) & alive|, -u); rep[u] = u and rep[w] = u for w in N(u) & alive;
    remove u and those neighbours.  Returns rep[n] (local indices); rep[rep] == rep (R9)."""
    adj = np.asarray(adj, bool)
    n = adj.shape[0]
    rep = np.full(n, -1, np.int64)
    alive = np.ones(n, bool)
    deg = adj.sum(axis=1).astype(np.int64)           # residual degree within the alive set
    while alive.any():
        cand = np.nonzero(alive)[0]
        u = cand[np.argmax(deg[cand])]                # argmax returns the first (lowest index) max
        members = np.nonzero(adj[u] & alive)[0]
        rep[u] = u
        rep[members] = u
        removed = np.concatenate(([u], members))
        alive[removed] = False
        deg -= adj[:, removed].sum(axis=1)            # neighbours lose the removed nodes
    return rep


@dataclass
class Condensation:
    rep: np.ndarray                 # [T, k] token index of the representative copy (same expert)
    groups: list                    # per expert (t, j) arrays, ascending t
    adjacency: list                 # per expert bool [n_e, n_e] (None when h > 1)
    band_pairs: list                # per expert list of (a, b) local pairs with |s - h| <= band
    s: list                         # per expert similarity matrices (None when h > 1)


def condense(X: np.ndarray, idx: np.ndarray, E: int, h: float, band: float = 1e-5,
             adjacency_override=None, keep_s: bool = True) -> Condensation:
    """Token condensation for one source rank: per expert group, normalized cosine similarity, the
    threshold graph, and the highest-degree greedy (token_to_token P:405).

    `adjacency_override[e]` (optional) replaces the fp64 graph of group e -- used to compare the
    greedy on exactly the GPU's edge decisions for pairs inside the +-band of h (reading R18)."""
    X = np.asarray(X, np.float64)
    T, k = idx.shape
    rep = np.full((T, k), -1, np.int64)
    groups = group_members(idx, E)
    adjs, bands, ss = [], [], []
    for e, (t, j) in enumerate(groups):
        n = t.size
        if n == 0:
            adjs.append(np.zeros((0, 0), bool)); bands.append([]); ss.append(None)
            continue
        if adjacency_override is not None and adjacency_override[e] is not None:
            adj = np.asarray(adjacency_override[e], bool)
            s = similarity_matrix(X[t]) if keep_s else None
        elif h > 1.0:
            adj = np.zeros((n, n), bool)      # s <= 1 < h: no edges (R4)
            s = None
        else:
            s = similarity_matrix(X[t])
            adj = threshold_graph(s, h)
        bp = []
        if s is not None:
            with np.errstate(invalid="ignore"):
                a, b = np.nonzero(np.triu(np.abs(s - h) <= band, 1))
            bp = list(zip(a.tolist(), b.tolist()))
        r = greedy_condense(adj)
        rep[t, j] = t[r]
        adjs.append(adj); bands.append(bp); ss.append(s if keep_s else None)
    return Condensation(rep, groups, adjs, bands, ss)


# ----------------------------------------------------------------------------------------------
# Fast similarity measurement with history shortcuts (readings R20, R21)
# ----------------------------------------------------------------------------------------------


def fast_measure(Xg: np.ndarray, H_sub: np.ndarray, S1: float, S2: float):
    """Fast similarity measurement of one group, steps 2 and 3 (step 1 -- only tokens pushed to
    the same expert are compared -- is the grouping itself).

    Step 2: with s_{b-1} the pair's finalized weight in the previous block (H_sub, nan = no history:
    the pair shared no expert there, reading R20), the weight is 1 if s_{b-1} > S1 and 0 if s_{b-1} < S2,
    and no cosine is computed.  Step 3: the remaining pairs get the normalized cosine (R4).
    Zero-norm tokens keep no weight (nan) whatever their history (R7).
    Returns (W [n, n] fp64 finalized weights, nan diagonal; computed [n, n] bool: pairs measured in step 3)."""
    s = similarity_matrix(Xg)
    H_sub = np.asarray(H_sub, np.float64)
    with np.errstate(invalid="ignore"):
        one = H_sub > S1
        zero = H_sub < S2
    W = np.where(one, 1.0, np.where(zero, 0.0, s))
    valid = ~np.isnan(s)                        # both norms nonzero
    W = np.where(valid, W, np.nan)
    np.fill_diagonal(W, np.nan)
    computed = valid & ~one & ~zero
    np.fill_diagonal(computed, False)
    return W, computed


def condense_fast(X: np.ndarray, idx: np.ndarray, E: int, h: float, H_prev: np.ndarray, S1: float, S2: float,
                  band: float = 1e-5, adjacency_override=None):
    """Token condensation of one block with the fast similarity measurement: per expert group,
    fast_measure against the previous block's finalized weights H_prev [T, T] (token-pair keyed, nan = none),
    then the threshold graph (edge iff W >= h) and the highest-degree greedy.  Returns (Condensation,
    H_new [T, T]: this block's finalized weights of every pair that shares an expert -- the history of the
    next block, reading R21 -- and the number of pairs measured in step 3 (each unordered pair once per
    group))."""
    X = np.asarray(X, np.float64)
    T, k = idx.shape
    rep = np.full((T, k), -1, np.int64)
    groups = group_members(idx, E)
    H_new = np.full((T, T), np.nan)
    adjs, bands, ws = [], [], []
    n_computed = 0
    for e, (t, j) in enumerate(groups):
        n = t.size
        if n == 0:
            adjs.append(np.zeros((0, 0), bool)); bands.append([]); ws.append(None)
            continue
        W, computed = fast_measure(X[t], H_prev[np.ix_(t, t)], S1, S2)
        n_computed += int(np.triu(computed, 1).sum())
        if adjacency_override is not None and adjacency_override[e] is not None:
            adj = np.asarray(adjacency_override[e], bool)
        else:
            adj = threshold_graph(W, h)
        with np.errstate(invalid="ignore"):
            a, b = np.nonzero(np.triu(computed & (np.abs(W - h) <= band), 1))
        bands.append(list(zip(a.tolist(), b.tolist())))
        r = greedy_condense(adj)
        rep[t, j] = t[r]
        H_new[np.ix_(t, t)] = W
        adjs.append(adj); ws.append(W)
    return Condensation(rep, groups, adjs, bands, ws), H_new, n_computed


def band_components(adj_plus: np.ndarray, band_pairs) -> np.ndarray:
    """Reading R18: nodes of the connected components of G+ (edges with s >= h - band) that contain
    a band pair.  Those are excluded from the bit-exact headline check (components are independent
    under the greedy)."""
    n = adj_plus.shape[0]
    comp = np.full(n, -1, np.int64)
    c = 0
    for s0 in range(n):
        if comp[s0] >= 0:
            continue
        stack = [s0]
        comp[s0] = c
        while stack:
            u = stack.pop()
            for v in np.nonzero(adj_plus[u])[0]:
                if comp[v] < 0:
                    comp[v] = c
                    stack.append(v)
        c += 1
    bad = np.zeros(n, bool)
    bad_c = {comp[a] for a, _ in band_pairs} | {comp[b] for _, b in band_pairs}
    for cc in bad_c:
        bad |= comp == cc
    return bad


# ----------------------------------------------------------------------------------------------
# Step 4-5: pack of representatives and the dispatch layout (R14, R15)
# ----------------------------------------------------------------------------------------------


def expert_rank(e: int, E: int, P: int) -> int:
    """Reading R14: contiguous placement, rank(e) = e // (E/P)."""
    return e // (E // P)


@dataclass
class Pack:
    counts: np.ndarray      # [E] representatives per expert (what this rank sends per expert)
    perm: np.ndarray        # [R] send slot -> token index
    slot_expert: np.ndarray  # [R] expert of each send slot
    pos: np.ndarray         # [T, k] send slot of the representative of copy (t, k)


def pack(idx: np.ndarray, rep: np.ndarray, E: int) -> Pack:
    """Only representatives are dispatched ("keep the token ... for transmission").
    Send order (R15): destination rank asc, expert asc, token asc -- with contiguous placement this is
    expert asc then token asc.  pos[t, j] = slot of rep(t, j) in expert idx[t, j]."""
    T, k = idx.shape
    slots = []
    for e in range(E):
        toks = sorted({int(t) for t, j in zip(*np.nonzero(idx == e)) if rep[t, j] == t})
        slots.extend((e, t) for t in toks)
    slot_of = {key: s for s, key in enumerate(slots)}
    pos = np.empty((T, k), np.int64)
    for t in range(T):
        for j in range(k):
            pos[t, j] = slot_of[(int(idx[t, j]), int(rep[t, j]))]
    counts = np.bincount([e for e, _ in slots], minlength=E).astype(np.int64)
    perm = np.array([t for _, t in slots], np.int64)
    slot_expert = np.array([e for e, _ in slots], np.int64)
    return Pack(counts, perm, slot_expert, pos)


def recv_layout(counts_all: np.ndarray, rank: int, E: int, P: int):
    """Receive order at `rank` (R15): local expert asc, then source rank asc, then the source's send
    order.  Returns a list of (src_rank, expert, first_src_slot, n_rows) blocks and per-local-expert
    row offsets [E_l + 1]."""
    El = E // P
    blocks, off = [], [0]
    src_off = np.concatenate([np.zeros((P, 1), np.int64), np.cumsum(counts_all, axis=1)], axis=1)
    for el in range(El):
        e = rank * El + el
        for src in range(P):
            n = int(counts_all[src, e])
            blocks.append((src, e, int(src_off[src, e]), n))
        off.append(off[-1] + int(counts_all[:, e].sum()))
    return blocks, np.array(off, np.int64)


# ----------------------------------------------------------------------------------------------
# Step 6: expert FFN ("expert networks that are essentially FFNs"; R12)
# ----------------------------------------------------------------------------------------------


def gelu(x):
    v = np.vectorize(math.erf, otypes=[np.float64])
    return 0.5 * x * (1.0 + v(x / math.sqrt(2.0)))


def gelu_grad(x):
    v = np.vectorize(math.erf, otypes=[np.float64])
    cdf = 0.5 * (1.0 + v(x / math.sqrt(2.0)))
    pdf = np.exp(-0.5 * x * x) / math.sqrt(2.0 * math.pi)
    return cdf + x * pdf


def silu(x):
    return x / (1.0 + np.exp(-x))


def silu_grad(x):
    sg = 1.0 / (1.0 + np.exp(-x))
    return sg * (1.0 + x * (1.0 - sg))


def expert_ffn(x, W1, W2, W3=None, act="gelu"):
    """o = GeLU_erf(x W1^T) W2^T, or SwiGLU (silu(x W1^T) * x W3^T) W2^T; no biases (R12).
    Returns (o, cache) with the pre-activations needed by the backward."""
    x = np.asarray(x, np.float64)
    pre1 = x @ np.asarray(W1, np.float64).T
    if act == "gelu":
        a = gelu(pre1)
        cache = (x, pre1, None, a)
    else:
        pre3 = x @ np.asarray(W3, np.float64).T
        a = silu(pre1) * pre3
        cache = (x, pre1, pre3, a)
    o = a @ np.asarray(W2, np.float64).T
    return o, cache


def expert_ffn_backward(do, cache, W1, W2, W3=None, act="gelu"):
    """Hand-derived chain rule of expert_ffn: dA = dO W2; dPre = dA * act'(pre);
    dx = dPre W1 (+ dPre3 W3); dW2 = dO^T A; dW1 = dPre^T x (dW3 = dPre3^T x)."""
    x, pre1, pre3, a = cache
    do = np.asarray(do, np.float64)
    W1 = np.asarray(W1, np.float64)
    W2 = np.asarray(W2, np.float64)
    da = do @ W2
    dW2 = do.T @ a
    if act == "gelu":
        dpre1 = da * gelu_grad(pre1)
        dx = dpre1 @ W1
        return dx, dpre1.T @ x, dW2, None
    W3 = np.asarray(W3, np.float64)
    dpre1 = da * pre3 * silu_grad(pre1)
    dpre3 = da * silu(pre1)
    dx = dpre1 @ W1 + dpre3 @ W3
    return dx, dpre1.T @ x, dW2, dpre3.T @ x


# ----------------------------------------------------------------------------------------------
# The layer (one source rank's tokens; experts are per-row functions so placement only changes the
# layout, checked separately by pack/recv_layout)
# ----------------------------------------------------------------------------------------------


@dataclass
class LayerState:
    routing: Routing
    cond: Condensation
    pk: Pack
    O: np.ndarray              # [R, d] expert outputs per send slot
    caches: dict = field(default_factory=dict)
    Y: np.ndarray = None


def layer_forward(X, Wg, W1, W2, W3, k, h, act="gelu", renormalize=None, routing=None,
                  rep=None, keep_s=False) -> LayerState:
    """Forward of the condensed MoE layer for one source rank:
    route -> condense -> pack -> expert FFN on representatives -> y_t = sum_k w_tk O[pos(t,k)]
    ("use the expert output of token j to replace it"; R10: the token's own gate weights).

    `routing` / `rep` may be given to freeze the discrete decisions (the GPU's, for parity)."""
    X = np.asarray(X, np.float64)
    E = Wg.shape[0]
    if renormalize is None:
        renormalize = k > 1
    r = routing if routing is not None else route(X, Wg, k, renormalize)
    if rep is None:
        cond = condense(X, r.idx, E, h, keep_s=keep_s)
    else:
        cond = Condensation(np.asarray(rep, np.int64), group_members(r.idx, E), [], [], [])
    pk = pack(r.idx, cond.rep, E)
    R, d = pk.perm.size, X.shape[1]
    O = np.zeros((R, d))
    caches = {}
    for e in range(E):
        sl = np.nonzero(pk.slot_expert == e)[0]
        if sl.size == 0:
            continue
        o, cache = expert_ffn(X[pk.perm[sl]], W1[e], W2[e], None if W3 is None else W3[e], act)
        O[sl] = o
        caches[e] = (sl, cache)
    Y = np.einsum("tk,tkd->td", r.w, O[pk.pos])
    return LayerState(r, cond, pk, O, caches, Y)


@dataclass
class LayerGrads:
    dX: np.ndarray
    dWg: np.ndarray
    dW1: np.ndarray
    dW2: np.ndarray
    dW3: np.ndarray
    dw: np.ndarray              # [T, k] gradient w.r.t. the gate weights
    dO: np.ndarray              # [R, d] gradient w.r.t. expert outputs per slot
    dXs: np.ndarray             # [R, d] gradient w.r.t. the dispatched rows


def layer_backward(st: LayerState, X, Wg, W1, W2, W3, dY, act="gelu", renormalize=None) -> LayerGrads:
    """Exact autograd of layer_forward with idx and rep as constants (reading R11), hand-derived:
      dO[slot] = sum_{(t,k): pos=slot} w_tk dY_t ;  dw_tk = <dY_t, O[pos_tk]>
      expert backward per slot; dX_t (expert path) = sum_{k: rep_tk = t} dXs[pos_tk]
      renorm gate: dl_j = w_j (dw_j - sum_i w_i dw_i) on the top-k, else dl = p (g - <p, g>)
      dW_g = dl^T X ; dX += dl W_g."""
    X = np.asarray(X, np.float64)
    dY = np.asarray(dY, np.float64)
    r, pk = st.routing, st.pk
    T, k = r.idx.shape
    E = Wg.shape[0]
    if renormalize is None:
        renormalize = k > 1
    R = pk.perm.size
    dO = np.zeros((R, X.shape[1]))
    for t in range(T):
        for j in range(k):
            dO[pk.pos[t, j]] += r.w[t, j] * dY[t]
    dw = np.einsum("td,tkd->tk", dY, st.O[pk.pos])
    dXs = np.zeros_like(dO)
    dW1 = np.zeros(np.shape(W1))
    dW2 = np.zeros(np.shape(W2))
    dW3 = None if W3 is None else np.zeros(np.shape(W3))
    for e, (sl, cache) in st.caches.items():
        dx, g1, g2, g3 = expert_ffn_backward(dO[sl], cache, W1[e], W2[e], None if W3 is None else W3[e], act)
        dXs[sl] = dx
        dW1[e] = g1
        dW2[e] = g2
        if dW3 is not None:
            dW3[e] = g3
    dX = np.zeros_like(X)
    for t in range(T):
        for j in range(k):
            if st.cond.rep[t, j] == t:
                dX[t] += dXs[pk.pos[t, j]]
    # gate
    dl = np.zeros((T, E))
    if renormalize:
        s = (r.w * dw).sum(axis=1, keepdims=True)
        np.put_along_axis(dl, r.idx, r.w * (dw - s), axis=1)
    else:
        g = np.zeros((T, E))
        np.put_along_axis(g, r.idx, dw, axis=1)
        dl = r.probs * (g - (r.probs * g).sum(axis=1, keepdims=True))
    dWg = dl.T @ X
    dX = dX + dl @ np.asarray(Wg, np.float64)
    return LayerGrads(dX, dWg, dW1, dW2, dW3, dw, dO, dXs)


# ----------------------------------------------------------------------------------------------
# Sequence migration, Alg. 1 with Eq. (1)
# ----------------------------------------------------------------------------------------------


class PlanningError(RuntimeError):
    pass


def combine_traffic(rows_at_i: np.ndarray, row_bytes: int) -> np.ndarray:
    """Alg. 1 line 1: f_ij = bytes of sequence i's expert-output rows located off GPU j
    (R16: distinct representative rows; condensed copies are rebuilt locally)."""
    rows_at_i = np.asarray(rows_at_i, np.int64)
    return row_bytes * (int(rows_at_i.sum()) - rows_at_i)


def candidate_set(f_i: np.ndarray, q: int) -> list:
    """Alg. 1 line 2: the top-q GPUs with minimum traffic, ties -> lower GPU id."""
    order = sorted(range(len(f_i)), key=lambda j: (int(f_i[j]), j))
    return order[:min(q, len(f_i))]


def cost_growth(B_j: int, L_j: int, length: int, d: int) -> int:
    """Alg. 1 line 5: s_ij = T_att(B_j + 1, max(L_j, l_i)) - T_att(B_j, L_j) (Eq. 1, P := 1)."""
    return attention_cost(B_j + 1, max(L_j, length), d) - attention_cost(B_j, L_j, d)


def plan_migration(seq_len, rows_at, q, row_bytes, d, capacity=None, objective="min"):
    """Alg. 1 with the text's "minimum cost growth" (reading R16 -- the printed
    "maximum" is available as objective="max").  Sequences in descending length (ties: id asc);
    candidates H_i; the capacity-feasible candidate with best s (ties: smaller f, lower rank) wins;
    B_j, L_j and resident tokens are updated after every assignment; if no candidate has capacity,
    any capacity-feasible GPU with best s; else PlanningError.
    capacity (tokens) defaults to max(ceil(1.5 * sum(len) / P), max len) (reading R16: S:74's 1.5x
    headroom, never below the longest sequence).  Returns (seq_dest, combine_bytes[P][P])."""
    seq_len = [int(x) for x in seq_len]
    rows_at = np.asarray(rows_at, np.int64)
    S, P = rows_at.shape
    if capacity is None or capacity <= 0:
        capacity = max(-(-3 * sum(seq_len) // (2 * P)), max(seq_len, default=0))
    f = [combine_traffic(rows_at[i], row_bytes) for i in range(S)]
    H = [candidate_set(f[i], q) for i in range(S)]
    B = [0] * P
    L = [0] * P
    resident = [0] * P
    dest = [-1] * S
    sign = 1 if objective == "min" else -1
    for i in sorted(range(S), key=lambda i: (-seq_len[i], i)):
        li = seq_len[i]

        def key(j):
            return (sign * cost_growth(B[j], L[j], li, d), int(f[i][j]), j)

        feas = [j for j in H[i] if resident[j] + li <= capacity]
        if not feas:
            feas = [j for j in range(P) if resident[j] + li <= capacity]
        if not feas:
            raise PlanningError(f"sequence {i} (len {li}) fits on no GPU (capacity {capacity})")
        j = min(feas, key=key)
        dest[i] = j
        B[j] += 1
        L[j] = max(L[j], li)
        resident[j] += li
    comb = np.zeros((P, P), np.int64)
    for i in range(S):
        for r in range(P):
            if r != dest[i]:
                comb[r, dest[i]] += rows_at[i, r] * row_bytes
    return np.array(dest, np.int64), comb
