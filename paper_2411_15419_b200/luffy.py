"""Thin ctypes binding of libluffy (include/luffy.h): same names, argument marshalling only.

Every function takes device pointers as ints (e.g. ``tensor.data_ptr()``) and a CUDA stream handle
(``torch.cuda.current_stream().cuda_stream``), exactly like the C ABI.  A non-OK status raises
LuffyError with luffy_last_error().  There is no fallback: if libluffy.so is missing, importing this
module raises.
"""
from __future__ import annotations

import ctypes
import os

import numpy as np

_LIB_PATH = os.path.join(os.path.dirname(os.path.abspath(__file__)), "libluffy.so")

OK, E_INVALID, E_CUDA, E_NCCL, E_CAPACITY, E_UNSUPPORTED, E_STATE = range(7)
FP32, BF16 = 0, 1
GELU, SWIGLU = 0, 1
ROW_ALIGN = 128
MAX_EXPERTS = 256

EXPORTED = [
    "luffy_create", "luffy_destroy", "luffy_layer_workspace_bytes",
    "luffy_layer_create", "luffy_layer_destroy", "luffy_last_error", "luffy_launch_count",
    "luffy_layer_rows", "luffy_route", "luffy_condense", "luffy_dispatch", "luffy_expert_ffn",
    "luffy_combine", "luffy_uncondense", "luffy_uncondense_bwd", "luffy_combine_bwd",
    "luffy_expert_ffn_bwd", "luffy_dispatch_bwd", "luffy_route_bwd", "luffy_plan_migration",
    "luffy_attention_cost", "luffy_adaptive_threshold", "luffy_debug_copy", "luffy_debug_gemm", "luffy_exchange_plan", "luffy_layer_set_exchange_timeout",
    "luffy_debug_gram_dump", "luffy_debug_set_pdl", "luffy_layer_set_history", "luffy_uncondense_residual",
    "luffy_dispatch_bwd_residual",
    "luffy_ipc_handle_bytes", "luffy_layer_ipc_handle", "luffy_layer_ipc_open", "luffy_layer_exchange_buffers",
    "luffy_sequence_rows", "luffy_set_migration", "luffy_migration_out_tokens",
]


class LuffyError(RuntimeError):
    def __init__(self, status: int, msg: str):
        super().__init__(f"luffy status {status}: {msg}")
        self.status = status


class Config(ctypes.Structure):
    _fields_ = [(n, ctypes.c_int32) for n in (
        "world", "rank", "num_experts", "top_k", "d_model", "d_ffn", "dtype", "act", "renormalize",
        "max_tokens", "max_recv_rows", "max_seqs", "fast_measure")]


class CondenseStats(ctypes.Structure):
    _fields_ = [("copies", ctypes.c_int64), ("reps", ctypes.c_int64), ("ambiguous_pairs", ctypes.c_int64),
                ("near_tie_tokens", ctypes.c_int64), ("decided_pairs", ctypes.c_int64),
                ("skipped_tiles", ctypes.c_int64), ("rounds", ctypes.c_int32),
                ("reps_per_expert", ctypes.c_int32 * MAX_EXPERTS),
                ("copies_per_expert", ctypes.c_int32 * MAX_EXPERTS)]


class MigrationProblem(ctypes.Structure):
    _fields_ = [("num_seqs", ctypes.c_int32), ("num_ranks", ctypes.c_int32), ("q", ctypes.c_int32),
                ("objective", ctypes.c_int32), ("seq_len", ctypes.POINTER(ctypes.c_int32)),
                ("rows_at", ctypes.POINTER(ctypes.c_int64)), ("row_bytes", ctypes.c_int64),
                ("capacity_tokens", ctypes.c_int64), ("d_model", ctypes.c_int64)]


def _load():
    if not os.path.exists(_LIB_PATH):
        raise ImportError(f"{_LIB_PATH} is not built; run `python -m paper_2411_15419_b200.build` "
                          "(there is no CPU fallback)")
    lib = ctypes.CDLL(_LIB_PATH, mode=ctypes.RTLD_GLOBAL)
    P, I32, I64, F32, SZ = ctypes.c_void_p, ctypes.c_int32, ctypes.c_int64, ctypes.c_float, ctypes.c_size_t
    sig = {
        "luffy_create": (I32, [ctypes.POINTER(Config), ctypes.POINTER(P)]),
        "luffy_ipc_handle_bytes": (SZ, []),
        "luffy_layer_ipc_handle": (I32, [P, P]),
        "luffy_layer_ipc_open": (I32, [P, P]),
        "luffy_sequence_rows": (I32, [P, P, I32, P, P, P]),
        "luffy_set_migration": (I32, [P, P, P, ctypes.POINTER(I64), P]),
        "luffy_migration_out_tokens": (I32, [P, P, P]),
        "luffy_layer_exchange_buffers": (I32, [P, ctypes.POINTER(P), ctypes.POINTER(P), ctypes.POINTER(P),
                                                ctypes.POINTER(P)]),
        "luffy_destroy": (None, [P]),
        "luffy_layer_workspace_bytes": (SZ, [ctypes.POINTER(Config)]),
        "luffy_layer_create": (I32, [P, P, SZ, ctypes.POINTER(P)]),
        "luffy_layer_destroy": (None, [P]),
        "luffy_last_error": (ctypes.c_char_p, []),
        "luffy_launch_count": (I64, []),
        "luffy_layer_rows": (I32, [P, ctypes.POINTER(I64), ctypes.POINTER(I64)]),
        "luffy_route": (I32, [P, P, P, I32, P, P, P]),
        "luffy_condense": (I32, [P, P, F32, P, ctypes.POINTER(CondenseStats), P]),
        "luffy_dispatch": (I32, [P, P, P, ctypes.POINTER(I64), P]),
        "luffy_expert_ffn": (I32, [P, P, P, P, P, P, P, P, P]),
        "luffy_combine": (I32, [P, P, P, P]),
        "luffy_uncondense": (I32, [P, P, P, P]),
        "luffy_uncondense_bwd": (I32, [P, P, P, P, P, P]),
        "luffy_combine_bwd": (I32, [P, P, P, P]),
        "luffy_expert_ffn_bwd": (I32, [P, P, P, P, P, P, P, P, P, P, P, P, P, P]),
        "luffy_dispatch_bwd": (I32, [P, P, P, P]),
        "luffy_route_bwd": (I32, [P, P, P, P, P, P, P]),
        "luffy_plan_migration": (I32, [ctypes.POINTER(MigrationProblem), P, P]),
        "luffy_attention_cost": (I64, [I64, I64, I64]),
        "luffy_adaptive_threshold": (I32, [ctypes.c_double, ctypes.c_double, I32, P]),
        "luffy_debug_copy": (I32, [P, I32, P, ctypes.POINTER(SZ), P]),
        "luffy_exchange_plan": (I32, [I32, I32, I32, P, P, P, P, P, P, I64, P, P]),
        "luffy_layer_set_exchange_timeout": (I32, [P, I64]),
        "luffy_debug_gram_dump": (I32, [P, P, ctypes.c_size_t]),
        "luffy_debug_set_pdl": (None, [I32]),
        "luffy_layer_set_history": (I32, [P, P, F32, F32]),
        "luffy_uncondense_residual": (I32, [P, P, P, P, P]),
        "luffy_dispatch_bwd_residual": (I32, [P, P, P, P, P]),
        "luffy_debug_gemm": (I32, [I32, I32, I32, P, P, P, P, P, P, I32, P, I32, I64, I32, I32, I32, I32, P]),
    }
    for name, (res, args) in sig.items():
        fn = getattr(lib, name)
        fn.restype = res
        fn.argtypes = args
    return lib


LIB = _load()


def _check(st: int):
    if st != OK:
        raise LuffyError(st, LIB.luffy_last_error().decode(errors="replace"))


def _p(x):
    """int / None / tensor -> pointer value."""
    if x is None:
        return None
    if isinstance(x, int):
        return x
    return x.data_ptr()


# ---------------------------------------------------------------- lifetime

def make_config(world=1, rank=0, num_experts=8, top_k=2, d_model=1024, d_ffn=4096, dtype=BF16, act=GELU,
                renormalize=-1, max_tokens=8192, max_recv_rows=0, max_seqs=0, fast_measure=0) -> Config:
    return Config(world, rank, num_experts, top_k, d_model, d_ffn, dtype, act, renormalize, max_tokens,
                  max_recv_rows, max_seqs, fast_measure)


def luffy_create(cfg: Config) -> int:
    out = ctypes.c_void_p()
    _check(LIB.luffy_create(ctypes.byref(cfg), ctypes.byref(out)))
    return out.value


def luffy_ipc_handle_bytes() -> int:
    return LIB.luffy_ipc_handle_bytes()


def luffy_layer_ipc_handle(layer: int) -> bytes:
    buf = (ctypes.c_uint8 * luffy_ipc_handle_bytes())()
    _check(LIB.luffy_layer_ipc_handle(layer, ctypes.cast(buf, ctypes.c_void_p)))
    return bytes(buf)


def luffy_layer_ipc_open(layer: int, all_handles: list):
    blob = b"".join(all_handles)
    arr = (ctypes.c_uint8 * len(blob)).from_buffer_copy(blob)
    _check(LIB.luffy_layer_ipc_open(layer, ctypes.cast(arr, ctypes.c_void_p)))


def luffy_layer_exchange_buffers(layer: int):
    ptrs = [ctypes.c_void_p() for _ in range(4)]
    _check(LIB.luffy_layer_exchange_buffers(layer, *[ctypes.byref(p) for p in ptrs]))
    return tuple(p.value for p in ptrs)


def luffy_destroy(ctx: int):
    LIB.luffy_destroy(ctx)


def luffy_layer_workspace_bytes(cfg: Config) -> int:
    n = LIB.luffy_layer_workspace_bytes(ctypes.byref(cfg))
    if n == 0:
        raise LuffyError(E_INVALID, "invalid config")
    return n


def luffy_layer_create(ctx: int, workspace, nbytes: int) -> int:
    out = ctypes.c_void_p()
    _check(LIB.luffy_layer_create(ctx, _p(workspace), nbytes, ctypes.byref(out)))
    return out.value


def luffy_layer_destroy(layer: int):
    LIB.luffy_layer_destroy(layer)


def luffy_launch_count() -> int:
    return LIB.luffy_launch_count()


def luffy_layer_rows(layer: int):
    s, r = ctypes.c_int64(), ctypes.c_int64()
    _check(LIB.luffy_layer_rows(layer, ctypes.byref(s), ctypes.byref(r)))
    return s.value, r.value


# ---------------------------------------------------------------- forward

def luffy_route(layer, x, w_gate, T, topk_idx, topk_w, stream):
    _check(LIB.luffy_route(layer, _p(x), _p(w_gate), T, _p(topk_idx), _p(topk_w), stream))


def luffy_condense(layer, x, h, rep, stream, stats: bool = False):
    st = CondenseStats() if stats else None
    _check(LIB.luffy_condense(layer, _p(x), float(h), _p(rep), ctypes.byref(st) if st is not None else None, stream))
    return st


def luffy_dispatch(layer, x, recv, stream, want_rows: bool = False):
    rows = ctypes.c_int64(-1)
    _check(LIB.luffy_dispatch(layer, _p(x), _p(recv), ctypes.byref(rows) if want_rows else None, stream))
    return rows.value if want_rows else None


def luffy_expert_ffn(layer, recv, w1, w2, w3, out, saved_pre, saved_act, stream):
    _check(LIB.luffy_expert_ffn(layer, _p(recv), _p(w1), _p(w2), _p(w3), _p(out), _p(saved_pre), _p(saved_act), stream))


def luffy_combine(layer, expert_out, gathered, stream):
    _check(LIB.luffy_combine(layer, _p(expert_out), _p(gathered), stream))


def luffy_uncondense(layer, gathered, y, stream):
    _check(LIB.luffy_uncondense(layer, _p(gathered), _p(y), stream))


# ---------------------------------------------------------------- backward

def luffy_uncondense_bwd(layer, dy, gathered, d_gathered, d_topk_w, stream):
    _check(LIB.luffy_uncondense_bwd(layer, _p(dy), _p(gathered), _p(d_gathered), _p(d_topk_w), stream))


def luffy_combine_bwd(layer, d_gathered, d_expert_out, stream):
    _check(LIB.luffy_combine_bwd(layer, _p(d_gathered), _p(d_expert_out), stream))


def luffy_expert_ffn_bwd(layer, d_out, recv, w1, w2, w3, saved_pre, saved_act, scratch_dpre, d_recv, dw1, dw2, dw3, stream):
    _check(LIB.luffy_expert_ffn_bwd(layer, _p(d_out), _p(recv), _p(w1), _p(w2), _p(w3), _p(saved_pre), _p(saved_act),
                                    _p(scratch_dpre), _p(d_recv), _p(dw1), _p(dw2), _p(dw3), stream))


def luffy_dispatch_bwd(layer, d_recv, dx, stream):
    _check(LIB.luffy_dispatch_bwd(layer, _p(d_recv), _p(dx), stream))


def luffy_route_bwd(layer, x, w_gate, d_topk_w, dx, dw_gate, stream):
    _check(LIB.luffy_route_bwd(layer, _p(x), _p(w_gate), _p(d_topk_w), _p(dx), _p(dw_gate), stream))


# ---------------------------------------------------------------- sequence migration (host)

def luffy_plan_migration(seq_len, rows_at, q, row_bytes, d_model, capacity_tokens=0, objective=0):
    seq_len = np.ascontiguousarray(seq_len, dtype=np.int32)
    rows_at = np.ascontiguousarray(rows_at, dtype=np.int64)
    S, P = rows_at.shape
    prob = MigrationProblem(S, P, int(q), int(objective),
                            seq_len.ctypes.data_as(ctypes.POINTER(ctypes.c_int32)),
                            rows_at.ctypes.data_as(ctypes.POINTER(ctypes.c_int64)),
                            int(row_bytes), int(capacity_tokens), int(d_model))
    dest = np.empty(S, np.int32)
    comb = np.empty((P, P), np.int64)
    _check(LIB.luffy_plan_migration(ctypes.byref(prob), dest.ctypes.data, comb.ctypes.data))
    return dest, comb


def luffy_attention_cost(B, L, d) -> int:
    return LIB.luffy_attention_cost(int(B), int(L), int(d))


def luffy_adaptive_threshold(l_ini: float, l_prev: float, scale2: bool = False) -> float:
    """Eq. (2): the condensation threshold of the next iteration from the first and the previous
    loss; scale2 selects the factor-2 reading R17b."""
    h = ctypes.c_float(0.0)
    _check(LIB.luffy_adaptive_threshold(float(l_ini), float(l_prev), int(bool(scale2)), ctypes.byref(h)))
    return h.value


DBG = dict(gcnt=(0, np.int32), goff=(1, np.int32), gtok=(2, np.int32), adjoff=(3, np.int64), adj=(4, np.uint32),
           rep_local=(5, np.int32), soff=(6, np.int32), perm=(7, np.int32), pos=(8, np.int32), nrep=(9, np.int32),
           rounds=(10, np.uint32), greedy_times=(11, np.uint32), hone=(12, np.uint32), hzero=(13, np.uint32),
           dec1=(14, np.uint32), dec0=(15, np.uint32), tskip=(16, np.uint8))


def luffy_debug_copy(layer, item: str, stream) -> np.ndarray:
    code, dt = DBG[item]
    n = ctypes.c_size_t(0)
    _check(LIB.luffy_debug_copy(layer, code, None, ctypes.byref(n), stream))
    out = np.empty(n.value // np.dtype(dt).itemsize, dt)
    if n.value:
        _check(LIB.luffy_debug_copy(layer, code, out.ctypes.data, ctypes.byref(n), stream))
    return out


def luffy_debug_gemm(kind, dtype, epi, A, B, B3, D, aux, D3, Msplit, off, G, max_rows, M, N, K, b_kmajor, stream):
    _check(LIB.luffy_debug_gemm(kind, dtype, epi, _p(A), _p(B), _p(B3), _p(D), _p(aux), _p(D3), Msplit, _p(off), G,
                                max_rows, M, N, K, b_kmajor, stream))


def luffy_exchange_plan(world: int, rank: int, num_experts: int, counts_all):
    """Dispatch/combine plan (the same code the device count exchange runs, csrc/xplan.h): dict with
    send_off [E+1], recv_off [E_l+1], dst_base [E], rank_of / slot_of [recv_off[-1]], send_rows_to [P],
    recv_rows_from [P]."""
    counts_all = np.ascontiguousarray(counts_all, dtype=np.int32)
    El = num_experts // world
    so = np.empty(num_experts + 1, np.int32)
    ro = np.empty(El + 1, np.int32)
    db = np.empty(num_experts, np.int32)
    cap = int(counts_all.astype(np.int64).sum()) + El * ROW_ALIGN
    rk = np.empty(max(cap, 1), np.int32)
    sl = np.empty(max(cap, 1), np.int32)
    st = np.empty(world, np.int64)
    rf = np.empty(world, np.int64)
    _check(LIB.luffy_exchange_plan(world, rank, num_experts, counts_all.ctypes.data, so.ctypes.data, ro.ctypes.data,
                                   db.ctypes.data, rk.ctypes.data, sl.ctypes.data, cap, st.ctypes.data, rf.ctypes.data))
    n = int(ro[-1])
    return dict(send_off=so, recv_off=ro, dst_base=db, rank_of=rk[:n], slot_of=sl[:n], send_rows_to=st,
                recv_rows_from=rf)


def luffy_uncondense_residual(layer, gathered, x, y, stream):
    _check(LIB.luffy_uncondense_residual(layer, _p(gathered), _p(x), _p(y), stream))


def luffy_dispatch_bwd_residual(layer, d_recv, dy, dx, stream):
    _check(LIB.luffy_dispatch_bwd_residual(layer, _p(d_recv), _p(dy), _p(dx), stream))


def luffy_layer_set_history(layer, prev, S1: float = 0.8, S2: float = 0.2):
    """Fast similarity measurement: take history shortcuts from `prev` (a luffy layer or None)."""
    _check(LIB.luffy_layer_set_history(layer, prev, float(S1), float(S2)))


def luffy_debug_set_pdl(on: bool):
    LIB.luffy_debug_set_pdl(1 if on else 0)


def luffy_debug_gram_dump(layer, buf):
    """Register a device fp32 tensor (or None) that the following luffy_condense calls fill with the Gram."""
    if buf is None:
        _check(LIB.luffy_debug_gram_dump(layer, None, 0))
    else:
        _check(LIB.luffy_debug_gram_dump(layer, ctypes.c_void_p(buf.data_ptr()), buf.numel()))


def luffy_layer_set_exchange_timeout(layer, ms: int):
    _check(LIB.luffy_layer_set_exchange_timeout(layer, int(ms)))


def luffy_sequence_rows(layer, seq_len, world, stream, counts=None):
    """K9: distinct representative rows of every rank's sequences on every rank -> [sum(counts), world] int64.
    counts: sequences per rank (None: every rank has len(seq_len))."""
    seq_len = np.ascontiguousarray(seq_len, dtype=np.int32)
    S = seq_len.size
    cnt = np.full(world, S, np.int32) if counts is None else np.ascontiguousarray(counts, dtype=np.int32)
    out = np.empty((int(cnt.sum()), world), np.int64)
    _check(LIB.luffy_sequence_rows(layer, seq_len.ctypes.data, S, cnt.ctypes.data, out.ctypes.data, stream))
    return out


def luffy_set_migration(layer, seq_len_all, seq_dest, stream) -> int:
    seq_len_all = np.ascontiguousarray(seq_len_all, dtype=np.int32)
    seq_dest = np.ascontiguousarray(seq_dest, dtype=np.int32)
    n = ctypes.c_int64()
    _check(LIB.luffy_set_migration(layer, seq_len_all.ctypes.data, seq_dest.ctypes.data, ctypes.byref(n), stream))
    return n.value


def luffy_migration_out_tokens(layer, n_out: int):
    hr = np.empty(n_out, np.int32)
    ht = np.empty(n_out, np.int32)
    _check(LIB.luffy_migration_out_tokens(layer, hr.ctypes.data, ht.ctypes.data))
    return hr, ht
