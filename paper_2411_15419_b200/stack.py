"""Multi-block driver: a stack of transformer blocks, each an attention sub-layer followed by the
token-condensed MoE sub-layer, both with residuals, forward and backward.  BASELINE config 4 ("GPT-MoE
12-layer stack, 32 experts top-2, seq 1024, d_model 2048, with sequence-migration placement enabled vs
disabled"); SURVEY §8(f) rows 1 and 3.

* MoE sub-layer: libluffy through the C ABI (CondensedMoELayer), the residual added in the uncondense pass
  (luffy_uncondense_residual).  With sequence migration every block runs K9 -> Alg. 1 on every
  rank (luffy_plan_migration) and its combine delivers each sequence's expert outputs -- and its residual
  rows -- to the rank chosen to host the sequence's NEXT attention; that rank then also dispatches the
  sequence's tokens to the next MoE layer.
* Attention sub-layer: the sequences a rank hosts, padded to the longest of them (B sequences x L), i.e.
  exactly the work Eq. (1) prices, T_att(B, L) = 3 B L d^2 + 2 B L^2 d.  This sub-layer is NOT part
  of the north star's hot path (it is the step after it, §8(f) row 3) and is plain PyTorch: one cuBLAS GEMM
  for the QKV projection and torch's SDPA (flash) kernel, causal, d/128 heads.
* Fast similarity measurement: with `history`, block b's condensation takes its S1/S2 shortcuts
  from block b-1 (luffy_layer_set_history) -- only without migration, where consecutive blocks see the same
  tokens in the same order on a rank.

Weights are random-initialised on the device, GPT-2 style: N(0, 0.02^2), with the two projections that write
into the residual stream (the attention's value projection -- Eq. (1) has no separate output projection --
and the experts' W2) scaled by 1/sqrt(2 n_blocks), so every block perturbs the residual stream by a small
step as in a trained-from-init transformer; gates follow workload.make_gate with a per-block perturbation
so that routing changes from block to block.
"""
from __future__ import annotations

import numpy as np
import torch
import torch.nn.functional as F

from . import layer as LY
from . import luffy as L


class _MoEFn(torch.autograd.Function):
    """Autograd node of one MoE sub-layer; its backward is libluffy's (weight gradients stay in the layer's
    fp32 buffers, as an optimizer would read them)."""

    @staticmethod
    def forward(ctx, x, blk):
        y = blk.moe_forward(x)
        ctx.blk = blk
        ctx.save_for_backward(x)
        return y

    @staticmethod
    def backward(ctx, dy):
        (x,) = ctx.saved_tensors
        return ctx.blk.moe_backward(dy.contiguous(), x), None


class Block:
    def __init__(self, index: int, E: int, k: int, d: int, f: int, max_tokens: int, world: int, rank: int,
                 device, h: float, migrate_q: int, fast_measure: bool, max_seqs: int, gate: np.ndarray, seed: int,
                 n_blocks: int = 1):
        self.i, self.E, self.k, self.d, self.f, self.h = index, E, k, d, f, h
        self.world, self.rank, self.q = world, rank, migrate_q
        self.dev = device
        El = E // world
        self.layer = LY.CondensedMoELayer(E, k, d, f, max_tokens=max_tokens, world=world, rank=rank, device=device,
                                          fast_measure=fast_measure, max_seqs=max_seqs)
        g = torch.Generator(device=device)
        g.manual_seed(seed + 7919 * index)
        rnd = lambda *shape: (torch.randn(*shape, generator=g, device=device) * 0.02).to(torch.bfloat16)
        res_scale = 1.0 / np.sqrt(2.0 * n_blocks)  # residual-branch projections (GPT-2 init)
        self.w1 = rnd(El, f, d)
        self.w2 = (rnd(El, d, f).float() * res_scale).to(torch.bfloat16)
        wqkv = rnd(d, 3 * d)
        wqkv[:, 2 * d:] = (wqkv[:, 2 * d:].float() * res_scale).to(torch.bfloat16)
        self.wqkv = wqkv.requires_grad_(True)
        rng = np.random.default_rng(seed + index)
        self.wg = torch.from_numpy((gate * (1.0 + 0.1 * rng.standard_normal(gate.shape))).astype(np.float32)).to(device)
        self.heads = d // 128
        self.lens_in = None     # sequence lengths of the tokens entering the block (this rank, in row order)
        self.lens_out = None    # ... and leaving it (the hosted sequences, with migration)
        self.lens_all = None    # every rank's lens_in (migration planning)
        self.mig_info = {}
        self.want_stats = False  # diagnostic passes: synchronous condensation stats (layer.stats)

    # ---- attention over the hosted sequences, padded to the longest (the Eq. (1) work)
    def attention(self, x: torch.Tensor) -> torch.Tensor:
        lens = self.lens_in
        B, Lm, d = len(lens), max(lens), self.d
        pos = np.concatenate([b * Lm + np.arange(l_) for b, l_ in enumerate(lens)])
        idx = torch.from_numpy(pos).to(self.dev)
        xp = torch.zeros(B * Lm, d, dtype=x.dtype, device=x.device).index_put((idx,), x)
        qkv = (xp @ self.wqkv).view(B, Lm, 3, self.heads, d // self.heads).permute(2, 0, 3, 1, 4)
        o = F.scaled_dot_product_attention(qkv[0], qkv[1], qkv[2], is_causal=True)
        o = o.transpose(1, 2).reshape(B * Lm, d)
        return x + o.index_select(0, idx)

    # ---- MoE sub-layer (libluffy)
    def moe_forward(self, x: torch.Tensor) -> torch.Tensor:
        lay = self.layer
        if self.q <= 0 or self.world == 1:
            self.lens_out = list(self.lens_in)
            return lay.forward(x, self.wg, self.w1, self.w2, None, h=self.h, residual=True, stats=self.want_stats)
        y, _, _, dest, _ = lay.forward_migrated(x, self.wg, self.w1, self.w2, None, h=self.h, seq_len=self.lens_in,
                                                q=self.q, residual=True, lens_all=self.lens_all, want_tokens=False,
                                                stats=self.want_stats)
        # the sequences every rank hosts next, in (home rank, sequence) order (luffy_set_migration's order):
        # every rank derives the next block's lens_all from the same plan, so no collective is needed
        flat = [(q, l_) for q, ls in enumerate(self.lens_all) for l_ in ls]
        self.lens_all_out = [[l_ for (q, l_), g in zip(flat, dest) if int(g) == r] for r in range(self.world)]
        self.lens_out = self.lens_all_out[self.rank]
        home = np.repeat(np.arange(self.world), [len(v) for v in self.lens_all])
        self.mig_info = {"migrated_seqs": int(np.sum(np.asarray(dest) != home)), "hosted_seqs": len(self.lens_out)}
        return y

    def moe_backward(self, dy: torch.Tensor, x: torch.Tensor) -> torch.Tensor:
        return self.layer.backward(dy, x, self.wg, self.w1, self.w2, None, residual=True)["dx"]

    def close(self):
        self.layer.close()


class MoEStack:
    """n_blocks transformer blocks on this rank (world ranks in lockstep); see the module docstring."""

    def __init__(self, n_blocks: int, E: int, k: int, d: int, f: int, tokens_per_rank: int, world: int = 1,
                 rank: int = 0, device="cuda", h: float = 0.9, migrate_q: int = 0, history=None, seed: int = 1234,
                 gate: np.ndarray | None = None, total_seqs: int = 256):
        self.world, self.rank, self.d = world, rank, d
        self.migrate = migrate_q > 0 and world > 1
        # with migration a rank may host up to 1.5x its share (Alg. 1's capacity, reading R16)
        cap = int(np.ceil(1.5 * tokens_per_rank)) + 1024 if self.migrate else tokens_per_rank
        self.cap = cap
        if gate is None:
            rng = np.random.default_rng(seed)
            gate = (rng.standard_normal((E, d)) * 0.02).astype(np.float32)
        fm = history is not None and not self.migrate
        self.blocks = [Block(i, E, k, d, f, cap, world, rank, device, h, migrate_q if self.migrate else 0, fm,
                             total_seqs, gate, seed, n_blocks) for i in range(n_blocks)]
        if fm:
            S1, S2 = history
            for i, b in enumerate(self.blocks):
                b.layer.set_history(self.blocks[i - 1].layer if i > 0 else None, S1, S2)

    def forward(self, x: torch.Tensor, lens: list[int]):
        """x [T, d] (this rank's sequences, lengths `lens`); returns (y [T', d], lens') for the sequences this
        rank hosts after the last block."""
        import torch.distributed as dist
        lens_all = None
        if self.migrate:  # once per step; later blocks derive every rank's sequences from the plan
            lens_all = [None] * self.world
            dist.all_gather_object(lens_all, [int(v) for v in lens])
        for b in self.blocks:
            b.lens_in = list(lens)
            b.lens_all = lens_all
            x = b.attention(x)
            x = _MoEFn.apply(x, b)
            lens = b.lens_out
            lens_all = getattr(b, "lens_all_out", None)
        return x, lens

    def step(self, x: torch.Tensor, lens: list[int], dy_pool: torch.Tensor):
        """One training step: forward through every block, backward with dY = dy_pool[:T'] (synthetic)."""
        x = x.detach()
        y, lens_out = self.forward(x, lens)
        torch.autograd.backward(y, dy_pool[: y.shape[0]])
        return y, lens_out

    def close(self):
        for b in self.blocks:
            b.close()


def attention_flops(B: int, Lm: int, d: int) -> int:
    """Eq. (1), P:307 (P := 1): 3 B L d^2 + 2 B L^2 d (the C ABI's luffy_attention_cost)."""
    return L.luffy_attention_cost(B, Lm, d)
