"""Seeded synthetic inputs for the token-condensed MoE layer (shared by oracle tests, GPU tests, bench).

This module holds NONE of the method's arithmetic (no routing, similarity, condensation, packing or
expert math): it only draws random arrays with the shapes and structure of the paper's workloads.
Both the oracle (`oracle/`) and the CUDA path consume exactly the arrays produced here.

Recipe:
  * sequence bias: each sequence draws pi_s ~ Dirichlet(0.3 * 1_E) and each token its primary expert
    e ~ pi_s  -- "more than half of sequences use no more than 3 experts" (Fig. 3);
  * embeddings: every expert owns `centres` unit centres mu_{e,c}; a token is
    x = sqrt(d) * (mu_{e,c} + tau * eps), eps ~ N(0, I/d).  With probability `phi` the token is
    "tight" (tau ~ U[0.2, 0.6]) otherwise "loose" (tau = 1.5).  Tight tokens of one centre have
    normalized cosine ~0.87-0.98 so a threshold h=0.9 cuts through that band -- the "significant
    prevalence of similar tokens" of P:224-228 / "62% very similar" of P:91;
  * `dup` of tokens are bit-exact copies of an earlier token of the same sequence and expert;
  * gate: W_g[e,:] = beta * sum_c mu_{e,c}, so top-1 follows the drawn expert and top-2 is noise;
  * expert weights W1, W2 (W3) ~ N(0, 0.02^2) in nn.Linear layout ([f,d], [d,f], [f,d]); dY ~ N(0,1);
  * bf16 configs round X, W1, W2, W3, dY to bf16 (round-to-nearest-even) so both sides see identical
    values; W_g stays fp32.
Seeds: rank r of a batch uses seed + r; centres use a fixed seed shared by all ranks.
"""
from __future__ import annotations

import dataclasses
import numpy as np


@dataclasses.dataclass(frozen=True)
class LayerConfig:
    name: str
    num_experts: int
    top_k: int
    d_model: int
    d_ffn: int
    seqs_per_rank: int
    seq_len: int
    dtype: str = "bf16"          # "bf16" or "fp32"
    act: str = "gelu"            # "gelu" or "swiglu"
    h: float = 0.9               # condensation threshold on the normalized-cosine scale
    world: int = 1               # simulated / real ranks

    @property
    def tokens_per_rank(self) -> int:
        return self.seqs_per_rank * self.seq_len

    @property
    def renormalize(self) -> bool:
        return self.top_k > 1


# BASELINE.json configs.  T per rank fixed at 8192 for C2-C5.
CONFIGS = {
    "C1": LayerConfig("C1-tiny-fp32", 4, 2, 256, 1024, 2, 128, "fp32", "gelu", 0.9, 4),
    "C2": LayerConfig("C2-gpt-moe", 8, 2, 1024, 4096, 16, 512, "bf16", "gelu", 0.9, 1),
    "C3": LayerConfig("C3-bert-moe", 16, 1, 768, 3072, 16, 512, "bf16", "gelu", 0.9, 1),
    "C4": LayerConfig("C4-gpt-moe-stack-layer", 32, 2, 2048, 8192, 8, 1024, "bf16", "gelu", 0.9, 1),
    "C5": LayerConfig("C5-mixtral", 8, 2, 4096, 14336, 2, 4096, "bf16", "swiglu", 0.9, 1),
}


def bf16_round(a: np.ndarray) -> np.ndarray:
    """Round fp32 values to the nearest bf16 (RNE); returns float32 holding bf16-representable values."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    u = a.view(np.uint32).astype(np.uint64)
    lsb = (u >> 16) & 1
    u = (u + 0x7FFF + lsb) & 0xFFFF0000
    out = u.astype(np.uint32).view(np.float32)
    nan = np.isnan(a)
    if nan.any():
        out = out.copy()
        out[nan] = np.nan
    return out


def bf16_bits(a: np.ndarray) -> np.ndarray:
    """uint16 bit patterns of bf16-representable float32 values (exact truncation)."""
    a = np.ascontiguousarray(a, dtype=np.float32)
    return (a.view(np.uint32) >> 16).astype(np.uint16)


def _cast(a: np.ndarray, dtype: str) -> np.ndarray:
    a = a.astype(np.float32)
    return bf16_round(a) if dtype == "bf16" else a


def expert_centres(E: int, d: int, centres: int = 4, seed: int = 999) -> np.ndarray:
    rng = np.random.default_rng(seed)
    mu = rng.standard_normal((E, centres, d))
    mu /= np.linalg.norm(mu, axis=-1, keepdims=True)
    return mu


def make_tokens(cfg: LayerConfig, rank: int = 0, seed: int = 1234, phi: float = 0.5,
                dup: float = 0.05, centres: int = 4, num_seqs: int | None = None,
                seq_len: int | None = None):
    """Token embeddings X [S*L, d] (float32 holding dtype-representable values) for one rank,
    plus the per-token drawn expert and sequence id (for diagnostics only)."""
    E, d = cfg.num_experts, cfg.d_model
    S = cfg.seqs_per_rank if num_seqs is None else num_seqs
    L = cfg.seq_len if seq_len is None else seq_len
    mu = expert_centres(E, d, centres)
    rng = np.random.default_rng(seed + rank)
    T = S * L
    X = np.empty((T, d), dtype=np.float64)
    drawn = np.empty(T, dtype=np.int64)
    seq_of = np.repeat(np.arange(S), L)
    for s in range(S):
        pi = rng.dirichlet(np.full(E, 0.3))
        e = rng.choice(E, size=L, p=pi)
        c = rng.integers(0, centres, size=L)
        tight = rng.random(L) < phi
        tau = np.where(tight, rng.uniform(0.2, 0.6, size=L), 1.5)
        eps = rng.standard_normal((L, d)) / np.sqrt(d)
        xs = np.sqrt(d) * (mu[e, c] + tau[:, None] * eps)
        # exact duplicates of an earlier token of the same sequence and drawn expert
        isdup = rng.random(L) < dup
        for i in np.nonzero(isdup)[0]:
            prev = np.nonzero(e[:i] == e[i])[0]
            if prev.size:
                xs[i] = xs[prev[rng.integers(0, prev.size)]]
        X[s * L:(s + 1) * L] = xs
        drawn[s * L:(s + 1) * L] = e
    return _cast(X, cfg.dtype), drawn, seq_of


def make_gate(cfg: LayerConfig, beta: float | None = None, centres: int = 4) -> np.ndarray:
    """Gate weights W_g [E, d] fp32 (nn.Linear layout: logits = X @ W_g^T)."""
    E, d = cfg.num_experts, cfg.d_model
    mu = expert_centres(E, d, centres)
    beta = (2.0 / np.sqrt(d)) if beta is None else beta
    return (beta * mu.sum(axis=1)).astype(np.float32)


def make_expert_weights(cfg: LayerConfig, experts: range | None = None, seed: int = 4321):
    """Expert weights in nn.Linear layout: W1 [E, f, d], W2 [E, d, f], W3 [E, f, d] (SwiGLU only).
    Each expert draws from its own seed so a rank can build only its local experts."""
    E, d, f = cfg.num_experts, cfg.d_model, cfg.d_ffn
    experts = range(E) if experts is None else experts
    W1 = np.empty((len(experts), f, d), np.float32)
    W2 = np.empty((len(experts), d, f), np.float32)
    W3 = np.empty((len(experts), f, d), np.float32) if cfg.act == "swiglu" else None
    for i, e in enumerate(experts):
        rng = np.random.default_rng(seed + 7919 * e)
        W1[i] = rng.standard_normal((f, d), dtype=np.float32) * 0.02
        W2[i] = rng.standard_normal((d, f), dtype=np.float32) * 0.02
        if W3 is not None:
            W3[i] = rng.standard_normal((f, d), dtype=np.float32) * 0.02
    W1, W2 = _cast(W1, cfg.dtype), _cast(W2, cfg.dtype)
    if W3 is not None:
        W3 = _cast(W3, cfg.dtype)
    return W1, W2, W3


def make_grad_out(cfg: LayerConfig, T: int, rank: int = 0, seed: int = 2718) -> np.ndarray:
    rng = np.random.default_rng(seed + rank)
    return _cast(rng.standard_normal((T, cfg.d_model), dtype=np.float32), cfg.dtype)


def make_layer_inputs(cfg: LayerConfig, rank: int = 0, **kw):
    """Everything one rank needs for a fwd+bwd step."""
    X, drawn, seq_of = make_tokens(cfg, rank=rank, **kw)
    Wg = make_gate(cfg)
    W1, W2, W3 = make_expert_weights(cfg)
    dY = make_grad_out(cfg, X.shape[0], rank=rank)
    return dict(X=X, Wg=Wg, W1=W1, W2=W2, W3=W3, dY=dY, drawn=drawn, seq_of=seq_of)


def make_migration_problem(num_seqs: int, num_ranks: int, seed: int = 77, lens=(256, 1024, 64)):
    """Sequence lengths l ~ U{256..1024 step 64} and rows_at[S][P] (rows of each sequence's expert
    outputs located on each rank) drawn with the biased expert activation of Fig. 3."""
    rng = np.random.default_rng(seed)
    lo, hi, step = lens
    seq_len = rng.choice(np.arange(lo, hi + 1, step), size=num_seqs).astype(np.int32)
    home = (np.arange(num_seqs) % num_ranks).astype(np.int32)
    rows_at = np.zeros((num_seqs, num_ranks), np.int64)
    for i in range(num_seqs):
        pi = rng.dirichlet(np.full(num_ranks, 0.3))
        rows_at[i] = rng.multinomial(int(seq_len[i]) * 2, pi)
    return seq_len, home, rows_at
