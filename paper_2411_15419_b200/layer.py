"""Token-condensed expert-parallel MoE layer driven through the libluffy C ABI.

This class is plumbing: it allocates device buffers with PyTorch and calls the C-ABI entry points in the
paper's order: route -> condense -> dispatch -> expert FFN -> combine -> uncondense, and the
backward in reverse.  Every arithmetic step runs in libluffy's CUDA kernels.
"""
from __future__ import annotations

import torch

from . import luffy as L

_TORCH_DT = {L.BF16: torch.bfloat16, L.FP32: torch.float32}


class CondensedMoELayer:
    def __init__(self, num_experts: int, top_k: int, d_model: int, d_ffn: int, max_tokens: int,
                 dtype: str = "bf16", act: str = "gelu", world: int = 1, rank: int = 0,
                 renormalize: int = -1, max_recv_rows: int = 0, device: torch.device | str = "cuda",
                 group=None, fast_measure: bool = False, max_seqs: int = 0):
        self.device = torch.device(device)
        self.dt = L.BF16 if dtype == "bf16" else L.FP32
        self.tdt = _TORCH_DT[self.dt]
        self.act = L.SWIGLU if act == "swiglu" else L.GELU
        self.E, self.k, self.d, self.f, self.Tmax = num_experts, top_k, d_model, d_ffn, max_tokens
        self.world, self.rank = world, rank
        self.El = num_experts // world
        self.cfg = L.make_config(world, rank, num_experts, top_k, d_model, d_ffn, self.dt, self.act, renormalize,
                                 max_tokens, max_recv_rows, max_seqs, 1 if fast_measure else 0)
        self.ctx = L.luffy_create(self.cfg)
        nbytes = L.luffy_layer_workspace_bytes(self.cfg)
        self.ws = torch.empty(nbytes, dtype=torch.uint8, device=self.device)
        self.layer = L.luffy_layer_create(self.ctx, self.ws, nbytes)
        if world > 1:
            # map every rank's exchange region (CUDA IPC over NVLink); torch.distributed only carries
            # the handle blobs (plumbing)
            import torch.distributed as dist
            mine = L.luffy_layer_ipc_handle(self.layer)
            handles = [None] * world
            dist.all_gather_object(handles, mine, group=group)
            L.luffy_layer_ipc_open(self.layer, handles)
        C = max_tokens * top_k
        self.send_rows = C + num_experts * L.ROW_ALIGN
        self.recv_rows = max_recv_rows if max_recv_rows > 0 else world * C + self.El * L.ROW_ALIGN
        if world == 1:
            self.recv_rows = max(self.recv_rows, self.send_rows)
        pre_cols = 2 * d_ffn if self.act == L.SWIGLU else d_ffn
        dev, tdt = self.device, self.tdt
        self.idx = torch.empty(max_tokens, top_k, dtype=torch.int32, device=dev)
        self.w = torch.empty(max_tokens, top_k, dtype=torch.float32, device=dev)
        self.rep = torch.empty(max_tokens, top_k, dtype=torch.int32, device=dev)
        one = world == 1  # world > 1: recv / gathered / d_expert_out / d_send live in the layer's exchange region
        self.recv = torch.empty(self.recv_rows, d_model, dtype=tdt, device=dev) if one else None
        self.pre = torch.empty(self.recv_rows, pre_cols, dtype=tdt, device=dev)
        self.act_buf = torch.empty(self.recv_rows, d_ffn, dtype=tdt, device=dev)
        self.out = torch.empty(self.recv_rows, d_model, dtype=tdt, device=dev) if one else None
        self.gathered = self.out
        self.y = torch.empty(max_tokens, d_model, dtype=tdt, device=dev)
        # backward buffers
        self.d_gathered = torch.empty(self.recv_rows, d_model, dtype=tdt, device=dev) if one else None
        self.d_out = self.d_gathered
        self.dpre = torch.empty(self.recv_rows, pre_cols, dtype=tdt, device=dev)
        self.d_recv = torch.empty(self.recv_rows, d_model, dtype=tdt, device=dev) if one else None
        self.dx = torch.empty(max_tokens, d_model, dtype=tdt, device=dev)
        self.dw = torch.empty(max_tokens, top_k, dtype=torch.float32, device=dev)
        self.dw1 = torch.empty(self.El, d_ffn, d_model, dtype=torch.float32, device=dev)
        self.dw2 = torch.empty(self.El, d_model, d_ffn, dtype=torch.float32, device=dev)
        self.dw3 = torch.empty(self.El, d_ffn, d_model, dtype=torch.float32, device=dev) if self.act == L.SWIGLU else None
        self.dwg = torch.empty(num_experts, d_model, dtype=torch.float32, device=dev)
        self.T = 0
        self.stats = None

    def set_history(self, prev: "CondensedMoELayer | None", S1: float = 0.8, S2: float = 0.2):
        """Fast similarity measurement with history shortcuts from the previous block."""
        L.luffy_layer_set_history(self.layer, prev.layer if prev is not None else None, S1, S2)

    def close(self):
        if getattr(self, "layer", None):
            L.luffy_layer_destroy(self.layer)
            self.layer = None
        if getattr(self, "ctx", None):
            L.luffy_destroy(self.ctx)
            self.ctx = None

    def __del__(self):
        try:
            self.close()
        except Exception:
            pass

    @staticmethod
    def _stream():
        return torch.cuda.current_stream().cuda_stream

    def forward(self, x: torch.Tensor, w_gate: torch.Tensor, w1, w2, w3=None, h: float = 0.9,
                stats: bool = False, want_rows: bool = False, out: torch.Tensor | None = None,
                residual: bool = False) -> torch.Tensor:
        """y = MoE(x), or x + MoE(x) with residual=True (luffy_uncondense_residual)."""
        T = x.shape[0]
        s = self._stream()
        self.T = T
        self.mig = False
        y = self.y if out is None else out
        L.luffy_route(self.layer, x, w_gate, T, self.idx, self.w, s)
        self.stats = L.luffy_condense(self.layer, x, h, self.rep, s, stats=stats)
        self.rows = L.luffy_dispatch(self.layer, x, self.recv, s, want_rows=want_rows)
        L.luffy_expert_ffn(self.layer, self.recv, w1, w2, w3, self.out, self.pre, self.act_buf, s)
        L.luffy_combine(self.layer, self.out, self.gathered, s)
        if residual:
            L.luffy_uncondense_residual(self.layer, self.gathered, x, y, s)
        else:
            L.luffy_uncondense(self.layer, self.gathered, y, s)
        return y[:T]

    def forward_migrated(self, x: torch.Tensor, w_gate: torch.Tensor, w1, w2, w3=None, h: float = 0.9,
                         seq_len=None, q: int = 1, seq_dest=None, capacity: int = 0, objective: int = 0, group=None,
                         residual: bool = False, stats: bool = False, lens_all=None, want_tokens: bool = True):
        """Forward with sequence migration (world > 1): K9 rows -> Alg. 1 on every rank (the
        C-ABI planner, or a given `seq_dest`) -> the combine delivers each sequence's expert outputs to
        the rank hosting it.  Returns (y [n_out, d] for the hosted tokens, home_rank, home_token,
        seq_dest, rows_at)."""
        import numpy as np
        import torch.distributed as dist
        assert self.world > 1
        T = x.shape[0]
        s = self._stream()
        self.T = T
        L.luffy_route(self.layer, x, w_gate, T, self.idx, self.w, s)
        self.stats = L.luffy_condense(self.layer, x, h, self.rep, s, stats=stats)
        self.mig = True
        lens = lens_all
        if lens is None:
            lens = [None] * self.world
            dist.all_gather_object(lens, [int(v) for v in seq_len], group=group)
        seq_len_all = np.array([v for ls in lens for v in ls], np.int32)
        rows_at = L.luffy_sequence_rows(self.layer, seq_len, self.world, s, counts=[len(v) for v in lens])
        if seq_dest is None:
            esize = 2 if self.dt == L.BF16 else 4
            seq_dest, _ = L.luffy_plan_migration(seq_len_all, rows_at, q, self.d * esize, self.d,
                                                 capacity_tokens=capacity, objective=objective)
        n_out = L.luffy_set_migration(self.layer, seq_len_all, seq_dest, s)
        L.luffy_dispatch(self.layer, x, None, s)
        L.luffy_expert_ffn(self.layer, None, w1, w2, w3, None, self.pre, self.act_buf, s)
        L.luffy_combine(self.layer, None, None, s)
        self.y_out = torch.empty(max(n_out, 1), self.d, dtype=self.tdt, device=self.device)
        if residual:
            L.luffy_uncondense_residual(self.layer, None, x, self.y_out, s)
        else:
            L.luffy_uncondense(self.layer, None, self.y_out, s)
        if not want_tokens:
            return self.y_out[:n_out], None, None, np.asarray(seq_dest), rows_at
        torch.cuda.current_stream().synchronize()
        home_rank, home_tok = L.luffy_migration_out_tokens(self.layer, n_out)
        return self.y_out[:n_out], home_rank, home_tok, np.asarray(seq_dest), rows_at

    def backward(self, dy: torch.Tensor, x: torch.Tensor, w_gate: torch.Tensor, w1, w2, w3=None,
                 residual: bool = False):
        """Backward of forward / forward_migrated; residual=True adds the residual branch's dY to dx."""
        s = self._stream()
        L.luffy_uncondense_bwd(self.layer, dy, self.gathered, self.d_gathered, self.dw, s)
        L.luffy_combine_bwd(self.layer, self.d_gathered, self.d_out, s)
        L.luffy_expert_ffn_bwd(self.layer, self.d_out, self.recv, w1, w2, w3, self.pre, self.act_buf, self.dpre,
                               self.d_recv, self.dw1, self.dw2, self.dw3, s)
        if residual:
            L.luffy_dispatch_bwd_residual(self.layer, self.d_recv, None if getattr(self, "mig", False) else dy, self.dx, s)
        else:
            L.luffy_dispatch_bwd(self.layer, self.d_recv, self.dx, s)
        L.luffy_route_bwd(self.layer, x, w_gate, self.dw, self.dx, self.dwg, s)
        T = self.T
        return dict(dx=self.dx[:T], dwg=self.dwg, dw1=self.dw1, dw2=self.dw2, dw3=self.dw3, dw=self.dw[:T])


class HostStepper:
    """Training steps of a layer fed from HOST (pinned) buffers, pipelined over three streams: the inputs
    of step i+1 (X, dY) are uploaded on a copy stream while step i computes, and the output Y of step i is
    downloaded on a second copy stream while its backward runs.  Every step copies its own inputs and its
    result; device buffers are double-buffered and ordered with events (an upload waits for the backward
    that last read its buffer, a forward waits for the download that last read its output buffer)."""

    def __init__(self, layer: CondensedMoELayer, tokens: int, graphs: bool = True):
        dev, tdt, d = layer.device, layer.tdt, layer.d
        self.layer, self.T, self.dev = layer, tokens, dev
        # one GPU: the forward and the backward of each buffer parity are captured once as CUDA graphs and
        # replayed (no per-step host launch cost); the copies and their events stay on the copy streams
        self.graphs = graphs and layer.world == 1
        self._g, self._gkey = None, None
        self.x = [torch.empty(tokens, d, dtype=tdt, device=dev) for _ in range(2)]
        self.dy = [torch.empty(tokens, d, dtype=tdt, device=dev) for _ in range(2)]
        self.y = [torch.empty(tokens, d, dtype=tdt, device=dev) for _ in range(2)]
        self.h2d = torch.cuda.Stream(device=dev)
        self.d2h = torch.cuda.Stream(device=dev)
        ev = lambda: [torch.cuda.Event() for _ in range(2)]
        self.ev_in, self.ev_used, self.ev_y, self.ev_out = ev(), ev(), ev(), ev()

    def run(self, batches, w_gate, w1, w2, w3=None, h: float = 0.9):
        """batches: sequence of (host X, host dY, host Y out).  Returns when the last Y is on the host
        side of the compute stream's order (callers time it with events on the current stream)."""
        cs = torch.cuda.current_stream(self.dev)
        batches = list(batches)
        n, T = len(batches), self.T
        start = torch.cuda.Event()
        start.record(cs)

        def upload(i):
            b = i % 2
            self.h2d.wait_event(start if i < 2 else self.ev_used[b])
            with torch.cuda.stream(self.h2d):
                self.x[b].copy_(batches[i][0], non_blocking=True)
                self.dy[b].copy_(batches[i][1], non_blocking=True)
            self.ev_in[b].record(self.h2d)

        key = (w_gate.data_ptr(), w1.data_ptr(), w2.data_ptr(), None if w3 is None else w3.data_ptr(), float(h))
        if self.graphs and self._gkey != key:
            cap = torch.cuda.Stream(device=self.dev)
            cap.wait_stream(cs)
            self._g = []
            for b in range(2):
                gf, gb = torch.cuda.CUDAGraph(), torch.cuda.CUDAGraph()
                with torch.cuda.graph(gf, stream=cap):
                    self.layer.forward(self.x[b][:T], w_gate, w1, w2, w3, h=h, out=self.y[b])
                with torch.cuda.graph(gb, stream=cap):
                    self.layer.backward(self.dy[b][:T], self.x[b][:T], w_gate, w1, w2, w3)
                self._g.append((gf, gb))
            cs.wait_stream(cap)
            self._gkey = key

        upload(0)
        for i in range(n):
            b = i % 2
            if i + 1 < n:
                upload(i + 1)
            cs.wait_event(self.ev_in[b])
            if i >= 2:
                cs.wait_event(self.ev_out[b])
            if self.graphs:
                self._g[b][0].replay()
                y = self.y[b][:T]
            else:
                y = self.layer.forward(self.x[b][:T], w_gate, w1, w2, w3, h=h, out=self.y[b])
            self.ev_y[b].record(cs)
            self.d2h.wait_event(self.ev_y[b])
            with torch.cuda.stream(self.d2h):
                batches[i][2].copy_(y, non_blocking=True)
            self.ev_out[b].record(self.d2h)
            if self.graphs:
                self._g[b][1].replay()
            else:
                self.layer.backward(self.dy[b][:T], self.x[b][:T], w_gate, w1, w2, w3)
            self.ev_used[b].record(cs)
        cs.wait_event(self.ev_out[(n - 1) % 2])
