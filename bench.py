"""Benchmark: token-condensed MoE layer fwd+bwd tokens/s on B200 (BASELINE.json metric).

    python bench.py [--gpus N] [--steps K] [--warmup W] [--config C2] [--h 0.9] [--impl luffy|reference]

N > 1 is launched by torchrun (one process per GPU); each rank holds T tokens (weak scaling) and E/N
experts; the dispatch/combine are device-initiated NVLink transfers inside libluffy's kernels (CUDA IPC;
torch.distributed only carries the IPC handles).  --migrate Q adds sequence migration (K9 + Alg. 1 with
candidate-set size Q on every rank) to every step.  A step = route -> condense -> dispatch -> expert FFN -> combine ->
uncondense -> and the whole backward, all through the libluffy C ABI.  Inputs are synthetic
(workload.py), generated on the host and resident in HBM before timing; the per-step working set
(~1 GB of activations) exceeds the 126 MB L2.

Prints ONE JSON line on rank 0.
"""
from __future__ import annotations

import argparse
import json
import os
import statistics
import subprocess
import sys
import threading
import time

ROOT = os.path.dirname(os.path.abspath(__file__))
sys.path.insert(0, ROOT)

import numpy as np  # noqa: E402

import workload  # noqa: E402

METRIC = "MoE-layer fwd+bwd tokens/s"
UNIT = "tokens/s"
PEAKS_FALLBACK = {"hbm_gbs": 6650.0, "bf16_tflops": 1590.0, "bf16_tflops_sustained": 1400.0}


def _peaks():
    try:
        with open(os.path.join(ROOT, "MEASURED_PEAKS.json")) as fh:
            p = json.load(fh)
        return p, "measured"
    except Exception:
        return PEAKS_FALLBACK, "fallback"


def _kname(raw: str) -> str:
    nm = raw.replace("(anonymous namespace)::", "").replace("void ", "").replace("luffy::", "")
    return nm.split("(")[0].split("<")[0].strip()


def kernel_table(step, steps: int = 10):
    """Warm per-kernel device durations (CUPTI via torch.profiler), PDL off so a kernel's duration excludes
    its dependency wait (luffy_debug_set_pdl; results are bitwise the same).  {kernel: (launches/step,
    us/step)} -- measured live in this process, never under ncu."""
    import torch
    from torch.profiler import ProfilerActivity, profile

    from paper_2411_15419_b200 import luffy as L
    L.luffy_debug_set_pdl(False)
    try:
        for _ in range(2):
            step()
        torch.cuda.synchronize()
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(steps):
                step()
            torch.cuda.synchronize()
    finally:
        L.luffy_debug_set_pdl(True)
    agg = {}
    for e in prof.events():
        if e.device_type.name == "CUDA" and "Memcpy" not in e.name and "Memset" not in e.name:
            a = agg.setdefault(_kname(e.name), [0, 0.0])
            a[0] += 1
            a[1] += e.device_time
    return {k: (c / steps, us / steps) for k, (c, us) in agg.items()}


def ffn_work(cfg, R: int, El: int):
    """Algorithmic work of the six expert-FFN GEMMs of one fwd+bwd: flops 12 R d f (GeLU) /
    18 R d f (SwiGLU); compulsory HBM bytes: activation rows (bf16) written and read by the GEMMs that
    need them (recv, act, GeLU'/pre, out, dO, dPre, d_recv), expert weights read twice (fwd, dgrad) and
    the fp32 weight gradients written once."""
    d, f, B = cfg.d_model, cfg.d_ffn, 2 if cfg.dtype == "bf16" else 4
    if cfg.act == "swiglu":
        flops = 18 * R * d * f
        rows = R * B * (6 * d + 13 * f)   # pre [2f] 2x, act [f] 3x, dpre [2f] 3x
        wts = El * d * f * (3 * 2 * B + 3 * 4)
    else:
        flops = 12 * R * d * f
        rows = R * B * (6 * d + 8 * f)
        wts = El * d * f * (2 * 2 * B + 2 * 4)
    return flops, rows + wts


def mem_kernel_bytes(name: str, cfg, T: int, R: int, Rpad: int, parts: int) -> float | None:
    """Compulsory HBM bytes of one launch of each memory-side kernel (None: not a memory-side kernel).
    B = element bytes; C = T k copies; R = representatives (expert rows), Rpad = padded slots."""
    d, E, k = cfg.d_model, cfg.num_experts, cfg.top_k
    B = 2 if cfg.dtype == "bf16" else 4
    C = T * k
    table = {
        "route_e8_kernel": T * d * B + E * d * 4 + T * E * 4 + C * 8,
        "route_fast_kernel": T * d * B + E * d * 4 + T * E * 4 + C * 8,
        "route_kernel": T * d * B + E * d * 4 + T * E * 4 + C * 8,
        "gather_norm_kernel": T * d * B + C * d * B + C * 8,             # x once, group rows + norms written
        "pack_rows_kernel": R * d * B + Rpad * d * B,
        "uncondense_kernel": R * d * B + T * d * B + C * 8,              # each slot's row once, y written
        "uncondense_bwd_window_kernel": T * d * B + R * d * B + Rpad * d * B + C * 4,
        "unpack_bwd_kernel": R * d * B + T * d * B,
        "route_bwd_fused8_kernel": 3 * T * d * B + T * E * 4 + parts * E * d * 4,
        "route_bwd_fast_kernel": 2 * T * d * B + T * E * 4,
        "wg_partial_fast_kernel": T * d * B + parts * E * d * 4,
        "wg_reduce_kernel": parts * E * d * 4 + E * d * 4,
    }
    return table.get(name)


def ncu_traffic(config: str, world: int):
    """DRAM read+write bytes per step of the FFN GEMMs and of the Gram from the per-config ncu --set full
    capture committed under profiles/ (tools/ncu_capture.sh), or None."""
    import glob
    paths = sorted(glob.glob(os.path.join(ROOT, "profiles", f"r*_ncu_full_{config}_n{world}.json")))
    if not paths:
        return None, None, None
    with open(paths[-1]) as fh:
        ks = json.load(fh)
    dram = lambda k: k.get("dram_read", 0) + k.get("dram_write", 0)
    gem = [k for k in ks if k["kernel"].startswith("gemm_tc_kernel")][:6]   # the first step's six GEMMs
    gr = [k for k in ks if k["kernel"].startswith("gram_tc_kernel")][-1:]
    return (sum(dram(k) for k in gem) if len(gem) == 6 else None, dram(gr[0]) if gr else None,
            os.path.relpath(paths[-1], ROOT))


class ClockSampler:
    """nvidia-smi clocks and throttle reasons sampled during the timed region."""

    def __init__(self, dev: int):
        self.dev = dev
        self.proc = None
        self.lines = []          # (host time, csv line)
        self.window = (0.0, float("inf"))

    def start(self):
        q = ("clocks.sm,clocks.max.sm,power.draw,clocks_event_reasons.hw_slowdown,"
             "clocks_event_reasons.hw_thermal_slowdown,clocks_event_reasons.sw_thermal_slowdown,"
             "clocks_event_reasons.sw_power_cap")
        try:
            self.proc = subprocess.Popen(["nvidia-smi", f"--query-gpu={q}", "--format=csv,noheader,nounits",
                                          "-lms", "50", "-i", str(self.dev)], stdout=subprocess.PIPE,
                                         stderr=subprocess.DEVNULL, text=True)
            self.t = threading.Thread(target=self._read, daemon=True)
            self.t.start()
            t0 = time.time()
            while not self.lines and time.time() - t0 < 20:   # wait for the first sample
                time.sleep(0.05)
        except Exception:
            self.proc = None
        return self

    def _read(self):
        for line in self.proc.stdout:
            self.lines.append((time.time(), line.strip()))

    def stop(self):
        if self.proc:
            self.proc.terminate()
            try:
                self.proc.wait(timeout=5)
            except Exception:
                self.proc.kill()

    def summary(self):
        sm, mx, reasons = [], None, set()
        names = ["hw_slowdown", "hw_thermal_slowdown", "sw_thermal_slowdown", "sw_power_cap"]
        lo, hi = self.window
        for ts, ln in self.lines:
            if ts < lo or ts > hi:
                continue
            parts = [p.strip() for p in ln.split(",")]
            if len(parts) < 7:
                continue
            try:
                sm.append(float(parts[0]))
                mx = float(parts[1])
            except ValueError:
                continue
            for n, v in zip(names, parts[3:7]):
                if v.lower().startswith("active"):
                    reasons.add(n)
        return {"sm_mhz": statistics.median(sm) if sm else None, "sm_max_mhz": mx, "reasons": sorted(reasons),
                "samples": len(sm)}


class NvlinkCounter:
    """NVML NVLink data throughput counters of one GPU (KiB, summed over its links): bytes that really
    crossed NVLink during a window -- the evidence for the fused device-initiated exchanges."""

    def __init__(self, dev: int):
        self.h = None
        try:
            import pynvml
            pynvml.nvmlInit()
            self.p = pynvml
            self.h = pynvml.nvmlDeviceGetHandleByIndex(dev)
            self.read()
        except Exception:
            self.h = None

    def read(self):
        if self.h is None:
            return None
        try:
            v = self.p.nvmlDeviceGetFieldValues(self.h, [(self.p.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_TX, 0xFFFFFFFF),
                                                         (self.p.NVML_FI_DEV_NVLINK_THROUGHPUT_DATA_RX, 0xFFFFFFFF)])
            if any(x.nvmlReturn != 0 for x in v):
                return None
            return (v[0].value.ullVal * 1024, v[1].value.ullVal * 1024)
        except Exception:
            return None


def _bind_local_cpus(dev: int):
    """Pin this process to the CPUs NVML reports as local to the GPU (first-touch placement of the pinned
    host buffers on the GPU's NUMA node); no-op when NVML or the affinity call is unavailable."""
    if os.environ.get("LUFFY_NO_CPU_BIND"):
        return
    try:
        import pynvml
        pynvml.nvmlInit()
        h = pynvml.nvmlDeviceGetHandleByIndex(dev)
        words = pynvml.nvmlDeviceGetCpuAffinity(h, (os.cpu_count() + 63) // 64)
        cpus = {64 * i + b for i, wd in enumerate(words) for b in range(64) if (wd >> b) & 1}
        cpus &= set(range(os.cpu_count()))
        if cpus:
            os.sched_setaffinity(0, cpus)
    except Exception:
        pass


def cpu_oracle_step(cfg, inp, ntok: int):
    """The oracle (as it stands) on a bounded sample: fwd+bwd of the first `ntok` tokens."""
    from oracle import luffy_oracle as O
    X = inp["X"][:ntok]
    st = O.layer_forward(X, inp["Wg"], inp["W1"], inp["W2"], inp["W3"], cfg.top_k, cfg.h, act=cfg.act)
    O.layer_backward(st, X, inp["Wg"], inp["W1"], inp["W2"], inp["W3"], inp["dY"][:ntok], act=cfg.act)


def _threads():
    try:
        from threadpoolctl import threadpool_info
        return max((i.get("num_threads", 1) for i in threadpool_info()), default=1)
    except Exception:
        return os.cpu_count() or 1


def _host_info():
    model = None
    try:
        out = subprocess.run(["lscpu"], capture_output=True, text=True, timeout=10).stdout
        model = next((ln.split(":", 1)[1].strip() for ln in out.splitlines() if ln.startswith("Model name")), None)
    except Exception:
        pass
    return {"cpu_count": os.cpu_count(), "lscpu_model": model, "blas_threads": _threads()}


def cpu_baseline(cfg, inp, ntok: int = 0, budget_s: float = 30.0):
    """The oracle as it stands (numpy fp64, all host cores through BLAS) on the full rank-0 batch when it
    fits the budget (C1-C3), else on the largest whole-sequence prefix that does (estimated from a
    256-token probe)."""
    T = inp["X"].shape[0]
    if ntok <= 0:
        probe = min(T, 256)
        t0 = time.perf_counter()
        cpu_oracle_step(cfg, inp, probe)
        per_tok = (time.perf_counter() - t0) / probe
        ntok = T if per_tok * T <= 2 * budget_s else max(cfg.seq_len, int(budget_s / per_tok) // cfg.seq_len * cfg.seq_len)
        ntok = min(ntok, T)
    t0 = time.perf_counter()
    cpu_oracle_step(cfg, inp, ntok)
    dt = time.perf_counter() - t0
    what = "the full" if ntok == T else f"the first {ntok} tokens (whole sequences) of the"
    out = {"value": ntok / dt, "unit": UNIT, "cores": _threads(), "kind": "oracle",
           "sample": f"fwd+bwd of {what} {cfg.name} rank-0 batch ({T} tokens), numpy fp64, {dt:.1f} s",
           "host": _host_info()}
    if ntok == T and dt < 5.0:  # small configs (C1): also on one core
        try:
            from threadpoolctl import threadpool_limits
            with threadpool_limits(limits=1):
                t0 = time.perf_counter()
                cpu_oracle_step(cfg, inp, ntok)
                out["one_core_value"] = ntok / (time.perf_counter() - t0)
        except Exception:
            pass
    return out


def run_reference(args, cfg):
    rank = int(os.environ.get("RANK", "0"))
    if rank != 0:
        return
    inp = workload.make_layer_inputs(cfg, rank=0)
    # bounded sample: the largest whole-sequence prefix of the rank-0 batch (up to the full batch) such
    # that the timed steps fit in ~180 s of host time (warm-up steps run a 64-token sample)
    T = inp["X"].shape[0]
    probe = min(T, 256)
    t0 = time.perf_counter()
    cpu_oracle_step(cfg, inp, probe)
    per_tok = (time.perf_counter() - t0) / probe
    budget = 180.0 / max(1, args.steps)
    ntok = min(T, args.ref_tokens) if args.ref_tokens > 0 else T
    if ntok * per_tok > budget:
        ntok = max(min(64, T), int(budget / per_tok) // cfg.seq_len * cfg.seq_len or int(budget / per_tok))
    for _ in range(args.warmup):
        cpu_oracle_step(cfg, inp, min(ntok, 64))
    times = []
    for _ in range(args.steps):
        t0 = time.perf_counter()
        cpu_oracle_step(cfg, inp, ntok)
        times.append(time.perf_counter() - t0)
    dt = statistics.mean(times)
    val = ntok / dt
    out = {"metric": METRIC, "value": val, "unit": UNIT, "impl": "reference", "n_gpus": args.gpus,
           "steps": args.steps, "warmup": args.warmup, "ms_per_step": dt * 1e3, "higher_is_better": True,
           "scaling": "weak", "vs_baseline": None, "dtype": "f64", "data": "synthetic",
           "config": {"workload": cfg.name, "tokens_per_step": ntok, "E": cfg.num_experts, "k": cfg.top_k,
                      "d_model": cfg.d_model, "d_ffn": cfg.d_ffn, "h": cfg.h},
           "cpu_baseline": {"value": val, "unit": UNIT, "cores": _threads(), "kind": "oracle",
                            "sample": f"each step: fwd+bwd of the first {ntok} tokens (of {T}) of the {cfg.name} "
                                      f"rank-0 batch, numpy fp64", "host": _host_info()},
           "e2e": {"value": val, "unit": UNIT, "h2d_bytes_per_step": 0, "d2h_bytes_per_step": 0}}
    print(json.dumps(out), flush=True)


def stack_lengths(T: int, rng) -> list[int]:
    """Variable sequence lengths l ~ U{256, ..., 1024 step 64} summing to T (the padding premise of
    sequence migration, P:88 / P:296; SURVEY §8(d) C4 lengths)."""
    lens = []
    while sum(lens) < T:
        lens.append(int(min(rng.choice(np.arange(256, 1025, 64)), T - sum(lens))))
    return lens


def run_stack(args, cfg):
    """BASELINE config 4: the C4 block stack (attention at the hosting rank + condensed MoE, residuals),
    fwd+bwd per step, migration on (--migrate q) or off, history shortcuts (--history S1,S2)."""
    import torch
    import torch.distributed as dist

    from paper_2411_15419_b200 import stack as SK
    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    T = cfg.tokens_per_rank
    X, _, _ = workload.make_tokens(cfg, rank=rank)
    x0 = torch.from_numpy(X).to(dev, torch.bfloat16)
    lens0 = stack_lengths(T, np.random.default_rng(4242 + rank))
    hist = tuple(float(v) for v in args.history.split(",")) if args.history else None
    st = SK.MoEStack(args.stack, cfg.num_experts, cfg.top_k, cfg.d_model, cfg.d_ffn, T, world=world, rank=rank,
                     device=dev, h=cfg.h, migrate_q=args.migrate, history=hist, gate=workload.make_gate(cfg),
                     total_seqs=max(256, 4 * len(lens0) * world))
    g = torch.Generator(device=dev)
    g.manual_seed(99 + rank)
    dy_pool = torch.randn(st.cap, cfg.d_model, generator=g, device=dev).to(torch.bfloat16)
    stream = torch.cuda.current_stream()
    clk = ClockSampler(local).start()
    for _ in range(args.warmup):
        st.step(x0, lens0, dy_pool)
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    a, b = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
    t_host0 = time.time()
    a.record(stream)
    for _ in range(args.steps):
        st.step(x0, lens0, dy_pool)
    b.record(stream)
    torch.cuda.synchronize()
    clk.window = (t_host0, time.time())
    time.sleep(0.06)
    clk.stop()
    ms = a.elapsed_time(b)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    # ---- diagnostic pass: attention forward per block (CUDA events) against Eq. (1); condensation stats
    samples, mig, hstats = [], [], []
    for blk in st.blocks:
        blk.want_stats = True
    x, lens = x0, lens0
    lens_all = None
    if st.migrate:
        lens_all = [None] * world
        dist.all_gather_object(lens_all, [int(v) for v in lens])
    for blk in st.blocks:
        blk.lens_in = list(lens)
        blk.lens_all = lens_all
        e0, e1 = torch.cuda.Event(enable_timing=True), torch.cuda.Event(enable_timing=True)
        with torch.no_grad():
            for _ in range(2):
                blk.attention(x)          # warm
            e0.record(stream)
            for _ in range(5):
                xa = blk.attention(x)
            e1.record(stream)
            torch.cuda.synchronize()
            Bq, Lm = len(lens), max(lens)
            samples.append((Bq, Lm, sum(lens), e0.elapsed_time(e1) / 5))
            x = blk.moe_forward(xa)
        lens = blk.lens_out
        lens_all = getattr(blk, "lens_all_out", None)
        s_ = blk.layer.stats
        if s_ is not None:
            hstats.append({"reps": int(s_.reps), "copies": int(s_.copies), "decided_pairs": int(s_.decided_pairs),
                           "skipped_tiles": int(s_.skipped_tiles)})
        mig.append(dict(blk.mig_info))
        blk.want_stats = False
    allsamples = [samples]
    if world > 1:
        allsamples = [None] * world
        dist.all_gather_object(allsamples, samples)
    flat = [s_ for r_ in allsamples for s_ in r_]
    ops = np.array([SK.attention_flops(B_, L_, cfg.d_model) for B_, L_, _, _ in flat], np.float64)
    tms = np.array([t_ for _, _, _, t_ in flat], np.float64)
    c = float((ops * tms).sum() / (ops * ops).sum())         # t = ops / P_eff, least squares
    rel = np.abs(tms - c * ops) / tms
    pad_eff = float(sum(n_ for _, _, n_, _ in flat) / sum(B_ * L_ for B_, L_, _, _ in flat))
    att_ms = float(np.mean([sum(t_ for _, _, _, t_ in r_) for r_ in allsamples]))
    if rank == 0:
        out = {"metric": "MoE stack fwd+bwd tokens/s", "value": world * T * args.steps / (ms / 1e3), "unit": UNIT,
               "n_gpus": world, "steps": args.steps, "warmup": args.warmup, "ms_per_step": ms_step,
               "higher_is_better": True, "scaling": "weak", "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
               "config": {"workload": f"{cfg.name} x {args.stack} blocks (attention + condensed MoE, residual)",
                          "tokens_per_rank": T, "E": cfg.num_experts, "k": cfg.top_k, "d_model": cfg.d_model,
                          "d_ffn": cfg.d_ffn, "h": cfg.h, "seq_len": "U{256..1024 step 64}",
                          "migration_q": args.migrate if st.migrate else 0, "history_S1_S2": hist,
                          "parallelism": f"ep{world}"},
               "attention": {"fwd_ms_per_step_mean_rank": att_ms, "padding_efficiency": pad_eff,
                             "eq1_ops_total": float(ops.sum()),
                             "max_rank_fwd_ms": float(max(sum(t_ for _, _, _, t_ in r_) for r_ in allsamples)),
                             "eq1_fit": {"P_eff_ops_per_s": 1.0 / c * 1e3, "mean_rel_err": float(rel.mean()),
                                         "max_rel_err": float(rel.max()), "samples": len(flat),
                                         "model": "t = (3 B L d^2 + 2 B L^2 d) / P (Eq. 1, P:307), least squares"}},
               "migration_per_block_rank0": mig if st.migrate else None, "condense_per_block_rank0": hstats,
               "clocks": clk.summary()}
        print(json.dumps(out), flush=True)
    st.close()
    if world > 1:
        dist.destroy_process_group()


def main():
    ap = argparse.ArgumentParser()
    ap.add_argument("--gpus", type=int, default=1)
    ap.add_argument("--steps", type=int, default=300)
    ap.add_argument("--warmup", type=int, default=5)
    ap.add_argument("--config", default="C2")
    ap.add_argument("--h", type=float, default=None)
    ap.add_argument("--impl", default="luffy", choices=["luffy", "reference"])
    ap.add_argument("--ref-tokens", type=int, default=0, help="reference-arm sample per step (0: auto, up to the full batch)")
    ap.add_argument("--cpu-tokens", type=int, default=0, help="oracle sample (0: full batch if it fits ~30 s)")
    ap.add_argument("--no-cpu-baseline", action="store_true")
    ap.add_argument("--no-e2e", action="store_true")
    ap.add_argument("--no-ktab", action="store_true", help="skip the CUPTI per-kernel pass (e.g. under ncu)")
    ap.add_argument("--no-graph", action="store_true", help="one GPU: time eager steps instead of CUDA-graph replays")
    ap.add_argument("--migrate", type=int, default=0,
                    help="world > 1: sequence migration with Alg. 1 candidate-set size q (0 = off)")
    ap.add_argument("--stack", type=int, default=0, help="run the N-block stack (attention + MoE) instead of one layer")
    ap.add_argument("--history", default=None, help="S1,S2: fast similarity measurement across blocks (stack)")
    ap.add_argument("--kprof", type=int, default=0, help="also write a warm per-kernel table over this many steps")
    ap.add_argument("--kprof-dir", default=os.path.join(ROOT, "gpurun_out"))
    args = ap.parse_args()
    cfg = workload.CONFIGS[args.config]
    if args.h is not None:
        import dataclasses
        cfg = dataclasses.replace(cfg, h=args.h)
    args.warmup = max(args.warmup, 3)
    if args.impl == "reference":
        return run_reference(args, cfg)
    if args.stack > 0:
        return run_stack(args, cfg)

    import torch
    import torch.distributed as dist

    from paper_2411_15419_b200 import layer as LY
    from paper_2411_15419_b200 import luffy as L

    world = int(os.environ.get("WORLD_SIZE", "1"))
    rank = int(os.environ.get("RANK", "0"))
    local = int(os.environ.get("LOCAL_RANK", "0"))
    torch.cuda.set_device(local)
    dev = torch.device("cuda", local)
    _bind_local_cpus(local)  # host buffers of the e2e path land on the GPU's NUMA node
    if world > 1:
        dist.init_process_group("nccl", device_id=dev)
    E, El = cfg.num_experts, cfg.num_experts // world
    inp = workload.make_layer_inputs(cfg, rank=rank)
    T = inp["X"].shape[0]
    W1, W2, W3 = workload.make_expert_weights(cfg, experts=range(rank * El, (rank + 1) * El))
    tdt = torch.bfloat16 if cfg.dtype == "bf16" else torch.float32

    def dev_t(a, dt=tdt):
        return torch.from_numpy(np.ascontiguousarray(a, np.float32)).to(dev, dt)

    x, dy = dev_t(inp["X"]), dev_t(inp["dY"])
    wg = torch.from_numpy(inp["Wg"]).to(dev)
    w1, w2 = dev_t(W1), dev_t(W2)
    w3 = dev_t(W3) if W3 is not None else None
    lay = LY.CondensedMoELayer(E, cfg.top_k, cfg.d_model, cfg.d_ffn, max_tokens=T, dtype=cfg.dtype, act=cfg.act,
                               world=world, rank=rank, device=dev)
    stream = torch.cuda.current_stream()
    s = stream.cuda_stream
    ev = lambda: torch.cuda.Event(enable_timing=True)
    marks = ["route", "condense", "dispatch", "ffn", "combine", "uncondense", "uncondense_bwd", "combine_bwd",
             "ffn_bwd", "dispatch_bwd", "route_bwd"]

    mig = args.migrate > 0 and world > 1
    if mig:
        # sequences of variable length l ~ U{256..1024 step 64} (padding premise), sum = T
        rng = np.random.default_rng(4242 + rank)
        seq_len = []
        while sum(seq_len) < T:
            seq_len.append(int(min(rng.choice(np.arange(256, 1025, 64)), T - sum(seq_len))))
        lens = [None] * world
        dist.all_gather_object(lens, seq_len)
        seq_len_all = np.array([v for ls in lens for v in ls], np.int32)
        seq_counts = [len(v) for v in lens]
        y_out = torch.empty(world * T, cfg.d_model, dtype=tdt, device=dev)
        dy_out = torch.randn(world * T, cfg.d_model, device=dev).to(tdt)
        mig_stats = {"migrated_seqs": 0, "hosted_tokens": 0}

    SH = [s]  # stream handle the step's calls go to (the capture stream while a CUDA graph records it)

    def step(evs=None):
        s = SH[0]

        def m(i):
            if evs is not None:
                evs[i].record(stream)
        m(0)
        L.luffy_route(lay.layer, x, wg, T, lay.idx, lay.w, s); m(1)
        L.luffy_condense(lay.layer, x, cfg.h, lay.rep, s)
        if mig:  # K9 -> Alg. 1 on every rank (host) -> destinations; the only host sync of the step
            rows_at = L.luffy_sequence_rows(lay.layer, seq_len, world, s, counts=seq_counts)
            dest, _ = L.luffy_plan_migration(seq_len_all, rows_at, args.migrate, cfg.d_model * tdt.itemsize, cfg.d_model)
            n_out = L.luffy_set_migration(lay.layer, seq_len_all, dest, s)
            mig_stats["migrated_seqs"] = int(np.sum(dest != np.repeat(np.arange(world), seq_counts)))
            mig_stats["hosted_tokens"] = int(n_out)
        m(2)
        L.luffy_dispatch(lay.layer, x, lay.recv, s); m(3)
        L.luffy_expert_ffn(lay.layer, lay.recv, w1, w2, w3, lay.out, lay.pre, lay.act_buf, s); m(4)
        L.luffy_combine(lay.layer, lay.out, lay.gathered, s); m(5)
        L.luffy_uncondense(lay.layer, lay.gathered, y_out if mig else lay.y, s); m(6)
        L.luffy_uncondense_bwd(lay.layer, dy_out if mig else dy, lay.gathered, lay.d_gathered, lay.dw, s); m(7)
        L.luffy_combine_bwd(lay.layer, lay.d_gathered, lay.d_out, s); m(8)
        L.luffy_expert_ffn_bwd(lay.layer, lay.d_out, lay.recv, w1, w2, w3, lay.pre, lay.act_buf, lay.dpre, lay.d_recv,
                               lay.dw1, lay.dw2, lay.dw3, s); m(9)
        L.luffy_dispatch_bwd(lay.layer, lay.d_recv, lay.dx, s); m(10)
        L.luffy_route_bwd(lay.layer, x, wg, lay.dw, lay.dx, lay.dwg, s); m(11)

    # stats (one synchronous condense) for the roofline's algorithmic work and the condensed fraction
    L.luffy_route(lay.layer, x, wg, T, lay.idx, lay.w, s)
    st = L.luffy_condense(lay.layer, x, cfg.h, lay.rep, s, stats=True)
    copies_e = np.array(st.copies_per_expert[:E], np.int64)
    reps_e = np.array(st.reps_per_expert[:E], np.int64)
    R = int(st.reps)
    rounds = int(st.rounds)
    clk = ClockSampler(local).start()
    for _ in range(args.warmup):
        step()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    n_ev = len(marks) + 1
    start, stop = ev(), ev()

    # The step is captured into CUDA graphs once and replayed (the whole fwd+bwd is device-side with no host
    # sync; PDL edges are kept by the capture), so host enqueue jitter and launch gaps never reach the GPU.
    # World > 1: two consecutive steps are captured (the receive buffers alternate by step parity) and
    # replayed alternately; every exchange flag carries the device step number (luffy_layer::dseq) that each
    # replay bumps.  Sequence migration (a host planner per step) runs eagerly.
    graph = None
    if not mig and not args.no_graph:
        try:
            cap = torch.cuda.Stream(device=dev)
            cap.wait_stream(stream)
            gs = []
            n0 = L.luffy_launch_count()
            SH[0] = cap.cuda_stream
            for _ in range(1 if world == 1 else 2):
                g = torch.cuda.CUDAGraph()
                with torch.cuda.graph(g, stream=cap):
                    step()
                gs.append(g)
            graph_launches = (L.luffy_launch_count() - n0) // len(gs)
            SH[0] = s
            stream.wait_stream(cap)
            if world > 1:
                dist.barrier()
            for i in range(2 * len(gs)):
                gs[i % len(gs)].replay()
            torch.cuda.synchronize()
            graph = gs
        except Exception as exc:  # capture unsupported here: eager steps
            SH[0] = s
            print(f"[bench] CUDA graph capture failed ({exc}); eager steps", file=sys.stderr)
            torch.cuda.synchronize()
    launches0 = L.luffy_launch_count()
    torch.cuda.synchronize()
    if world > 1:
        dist.barrier()
    t_host0 = time.time()
    start.record(stream)
    for i in range(args.steps):
        if graph is not None:
            graph[i % len(graph)].replay()
        else:
            step()  # no events inside the timed steps: a stream event between kernels would block their PDL overlap
    stop.record(stream)
    host_ms = (time.time() - t_host0) * 1e3 / args.steps  # enqueue time per step (no host sync in the step)
    torch.cuda.synchronize()
    launches = graph_launches if graph is not None else (L.luffy_launch_count() - launches0) // args.steps
    clk.window = (t_host0, time.time())
    time.sleep(0.06)
    clk_window = "timed region"
    need = clk.summary()["samples"] == 0
    if world > 1:  # the step exchanges between ranks: all or none run the continuation
        fl = torch.tensor([int(need)], device=dev)
        dist.all_reduce(fl, op=dist.ReduceOp.MAX)
        need = bool(fl.item())
    if need:
        # the timed region was shorter than the 50 ms sampling period: keep the same step running (untimed)
        # for ~0.3 s and report the clocks seen under that load instead
        t1 = time.time()
        while time.time() - t1 < 0.3:
            for _ in range(20):
                graph[_ % len(graph)].replay() if graph is not None else step()
            torch.cuda.synchronize()
        clk.window = (t1, time.time())
        time.sleep(0.06)
        clk_window = "untimed continuation of the step (timed region shorter than the sampling period)"
    clk.stop()
    if world > 1:
        dist.barrier()
    ms = start.elapsed_time(stop)
    if world > 1:
        t = torch.tensor([ms], device=dev)
        dist.all_reduce(t, op=dist.ReduceOp.MAX)
        ms = float(t.item())
    ms_step = ms / args.steps
    value = world * T * args.steps / (ms / 1e3)
    # per-phase breakdown from a separate pass with events between the API calls (diagnostic only)
    nb_steps = min(args.steps, 50)
    evs = [[ev() for _ in range(n_ev)] for _ in range(nb_steps)]
    for i in range(nb_steps):
        step(evs[i])
    torch.cuda.synchronize()
    breakdown = {m: statistics.mean(evs[i][j].elapsed_time(evs[i][j + 1]) for i in range(nb_steps))
                 for j, m in enumerate(marks)}

    # ---- optional per-kernel table (CUPTI activity via torch.profiler, warm, every rank; never under ncu)
    if args.kprof > 0:
        from torch.profiler import ProfilerActivity, profile
        with profile(activities=[ProfilerActivity.CUDA]) as prof:
            for _ in range(args.kprof):
                step()
            torch.cuda.synchronize()
        agg, spans = {}, []
        for e in prof.events():
            if e.device_type.name == "CUDA":
                nm = e.name.replace("(anonymous namespace)::", "").replace("void ", "").replace("luffy::", "")
                nm = nm.split("(")[0][:70]
                a = agg.setdefault(nm, [0, 0.0, 0.0])
                a[0] += 1
                a[1] += e.device_time
                spans.append((e.time_range.start, e.time_range.end, nm))
        spans.sort()
        for (_, b0, _), (a1, _, nm) in zip(spans, spans[1:]):
            agg[nm][2] += max(0.0, a1 - b0)  # idle gap before this kernel
        busy = sum(b - a for a, b, _ in spans)
        wall = spans[-1][1] - spans[0][0] if spans else 0
        path = os.path.join(args.kprof_dir, f"kprof_{cfg.name}_n{world}_r{rank}.txt")
        os.makedirs(args.kprof_dir, exist_ok=True)
        with open(path, "w") as fh:
            fh.write(f"# {cfg.name} world {world} rank {rank}: per-step us (warm, {args.kprof} steps); "
                     f"kernels busy {busy / args.kprof:.1f} us of {wall / args.kprof:.1f} us wall per step\n")
            for k, (c, us, gap) in sorted(agg.items(), key=lambda kv: -kv[1][1]):
                fh.write(f"{us / args.kprof:9.1f} us  {c / args.kprof:5.1f}x  gap-before {gap / args.kprof:6.1f} us  {k}\n")

    # ---- e2e: the same steps through the public API fed from pinned HOST memory: every step uploads its
    # X and dY and downloads its Y (LY.HostStepper pipelines the copies of step i+1 / i with the compute
    # of step i on two copy streams); timed on the compute stream, max over ranks
    e2e = None
    if not args.no_e2e and not mig:
        hx = torch.empty(x.shape, dtype=tdt, pin_memory=True).copy_(x)
        hdy = torch.empty(dy.shape, dtype=tdt, pin_memory=True).copy_(dy)
        hy = torch.empty(x.shape, dtype=tdt, pin_memory=True)
        stepper = LY.HostStepper(lay, T, graphs=os.environ.get("LUFFY_STEPPER_GRAPHS", "1") != "0")
        stepper.run([(hx, hdy, hy)] * 3, wg, w1, w2, w3, h=cfg.h)
        torch.cuda.synchronize()
        if world > 1:
            dist.barrier()
        a, b = ev(), ev()
        a.record(stream)
        stepper.run([(hx, hdy, hy)] * args.steps, wg, w1, w2, w3, h=cfg.h)
        b.record(stream)
        torch.cuda.synchronize()
        ems = a.elapsed_time(b)
        if world > 1:
            t = torch.tensor([ems], device=dev)
            dist.all_reduce(t, op=dist.ReduceOp.MAX)
            ems = float(t.item())
        # the downloaded result equals the device path's output (deterministic kernels: bitwise)
        y_dev = lay.forward(x, wg, w1, w2, w3, h=cfg.h)
        torch.cuda.synchronize()
        same = bool(torch.equal(hy.to(dev), y_dev))
        nb = x.numel() * x.element_size()
        e2e = {"value": world * T * args.steps / (ems / 1e3), "unit": UNIT, "h2d_bytes_per_step": 2 * nb,
               "d2h_bytes_per_step": nb, "host_result_matches_device": same,
               "pipeline": "H2D of step i+1 and D2H of step i overlap step i's compute (two copy streams)"}

    # ---- condensed fraction of the all-to-all rows (remote = experts on other ranks)
    remote = np.array([e // El != rank for e in range(E)])
    rc, rr = int(copies_e[remote].sum()), int(reps_e[remote].sum())
    frac_all = 1.0 - R / max(1, int(copies_e.sum()))
    frac_remote = (1.0 - rr / rc) if rc else None
    if world > 1:
        t = torch.tensor([rc, rr, int(copies_e.sum()), R], device=dev, dtype=torch.float64)
        dist.all_reduce(t)
        rc, rr, ctot, rtot = (float(v) for v in t.tolist())
        frac_remote = 1.0 - rr / rc if rc else None
        frac_all = 1.0 - rtot / ctot

    # ---- rooflines.  Peaks: MEASURED_PEAKS.json burst figures (every timing here is a
    # sub-second evented / CUPTI window, not a long sustained run).
    peaks, src = _peaks()
    hbm_peak = float(peaks.get("hbm_gbs", 6550.0))
    tc_peak = float(peaks.get("bf16_tflops", 1672.3)) if cfg.dtype == "bf16" else 80.0
    tc_src = f"{src} bf16_tflops (burst)" if cfg.dtype == "bf16" else "fp32 SIMT nominal (148 SMs x 128 FFMA x 2 x 2.1 GHz)"
    # (1) dominant group: the six grouped expert GEMMs (tcgen05), timed with CUDA events around the
    # luffy_expert_ffn / luffy_expert_ffn_bwd calls (their only launches at world == 1)
    R_avg = float(R)
    if world > 1:
        t = torch.tensor([float(R)], device=dev, dtype=torch.float64)
        dist.all_reduce(t)
        R_avg = float(t.item()) / world  # each rank runs the rows its experts receive: R on average
    flops, fbytes = ffn_work(cfg, R_avg, El)
    ffn_ms = breakdown["ffn"] + breakdown["ffn_bwd"]
    t_tc, t_hbm = flops / (tc_peak * 1e12), fbytes / (hbm_peak * 1e9)
    traffic, gram_traffic, tsrc = ncu_traffic(args.config, world)
    if t_tc >= t_hbm:
        roof = {"bound": "tensor", "achieved": flops / (ffn_ms / 1e3) / 1e12, "peak": tc_peak, "unit": "TFLOP/s",
                "peak_source": tc_src}
    else:
        roof = {"bound": "hbm", "achieved": fbytes / (ffn_ms / 1e3) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                "peak_source": f"{src} hbm_gbs (copy)"}
    roof.update({"frac": roof["achieved"] / roof["peak"], "traffic": traffic, "traffic_source": tsrc,
                 "kernel": "expert FFN grouped GEMMs (fwd 2 + bwd 4 tcgen05 launches per step)",
                 "per": "one step (6 launches)", "algorithmic_flops": flops, "algorithmic_bytes": fbytes,
                 "intensity_flop_per_byte": flops / fbytes, "ridge_flop_per_byte": tc_peak * 1e3 / hbm_peak,
                 "roofline_time_us": max(t_tc, t_hbm) * 1e6, "measured_us": ffn_ms * 1e3,
                 "timing": "CUDA events around the two FFN calls, evented pass after the timed region"})
    # (2) per-kernel table (CUPTI, PDL off): the Gram and the memory-side kernels against their rooflines
    ktab = kernel_table(step, steps=10) if not (mig or args.no_ktab) else {}
    gram_roof, mem_roof, shares = None, None, None
    if ktab:
        tot = sum(us for _, us in ktab.values())
        shares = {k: {"us_per_step": round(us, 2), "launches": c, "share": round(us / tot, 4)}
                  for k, (c, us) in sorted(ktab.items(), key=lambda kv: -kv[1][1])}
        gk = ktab.get("gram_tc_kernel") or ktab.get("gram_simt_kernel")
        if gk and cfg.h <= 1.0:
            n_g = copies_e.astype(np.float64)
            gflops = float((n_g * (n_g + 1)).sum()) * cfg.d_model  # upper triangle incl. diagonal, 2 flop per MAC
            gram_roof = {"bound": "tensor", "achieved": gflops / (gk[1] * 1e-6) / 1e12, "peak": tc_peak,
                         "unit": "TFLOP/s", "frac": gflops / (gk[1] * 1e-6) / 1e12 / tc_peak,
                         "traffic": gram_traffic, "kernel": "similarity Gram + threshold (gram_tc_kernel)",
                         "algorithmic_flops": gflops, "measured_us": gk[1], "timing": "CUPTI, warm, PDL off"}
        parts = (T + 31) // 32
        mb, mus, used = 0.0, 0.0, []
        for k_, (c, us) in ktab.items():
            b_ = mem_kernel_bytes(k_, cfg, T, int(R_avg), int(R_avg) + E * 128, parts)
            if b_ is not None:
                mb += b_ * c
                mus += us
                used.append(k_)
        if mus > 0:
            mem_roof = {"bound": "hbm", "achieved": mb / (mus * 1e-6) / 1e9, "peak": hbm_peak, "unit": "GB/s",
                        "frac": mb / (mus * 1e-6) / 1e9 / hbm_peak, "traffic": None,
                        "kernel": "memory-side kernels (sum): " + ", ".join(sorted(used)),
                        "algorithmic_bytes": mb, "measured_us": mus, "timing": "CUPTI, warm, PDL off"}

    # ---- NVLink (world > 1): bytes that crossed NVLink per step (NVML counters over the timed region) against
    # the algorithmic 4 R_remote d B (dispatch, combine and both backward exchanges), and the push bandwidth of
    # the dispatch kernel alone (its remote bytes / its CUPTI duration) against 900 GB/s nominal and the
    # 770 GB/s measured peer copy (B200_PROFILING.md)
    nvlink = None
    if world > 1:
        B_ = 2 if cfg.dtype == "bf16" else 4
        remote_rows = int(reps_e[[e // El != rank for e in range(E)]].sum())
        alg = 4 * remote_rows * cfg.d_model * B_
        # NVML's NVLink counters perturb the exchange while they are polled (measured: C2 N=2 0.64 -> 1.3 ms
        # per step), so they are read over a separate window of 10 steps after every timed measurement
        nv = None
        if not os.environ.get("LUFFY_NO_NVML"):
            nvl = NvlinkCounter(local)
            torch.cuda.synchronize()
            dist.barrier()
            c0 = nvl.read()
            for _ in range(10):
                step()
            torch.cuda.synchronize()
            c1 = nvl.read()
            if c0 and c1:
                nv = {"tx_bytes_per_step": (c1[0] - c0[0]) / 10, "rx_bytes_per_step": (c1[1] - c0[1]) / 10,
                      "window": "10 steps after the timed region (the counters perturb the exchange)"}
        push = None
        pk, pkn = None, None
        for kn in ("xpack_push_tma_kernel", "xpack_push_kernel"):
            if ktab and kn in ktab:
                pk, pkn = ktab[kn], kn
                break
        if pk:
            gbs = remote_rows * cfg.d_model * B_ / (pk[1] * 1e-6) / 1e9
            push = {"kernel": f"{pkn} (fused pack + dispatch push)", "remote_bytes": remote_rows * cfg.d_model * B_,
                    "us": pk[1], "GBps": gbs, "frac_of_900_nominal": gbs / 900.0, "frac_of_770_measured_peer_copy": gbs / 770.0}
        nvlink = {"algorithmic_bytes_per_step_rank": alg, "nvml_counters_rank": nv, "dispatch_push": push,
                  "step_avg_GBps_rank": alg / (ms_step * 1e-3) / 1e9}
        allnv = [None] * world
        dist.all_gather_object(allnv, nvlink)
        nvlink = {"per_rank": allnv}
    if rank == 0:
        cpu = None
        if not args.no_cpu_baseline:
            cpu = cpu_baseline(cfg, inp, args.cpu_tokens)
        clocks = clk.summary()
        clocks["window"] = clk_window
        out = {"metric": METRIC, "value": value, "unit": UNIT, "n_gpus": world, "steps": args.steps,
               "warmup": args.warmup, "ms_per_step": ms_step, "higher_is_better": True, "scaling": "weak",
               "vs_baseline": None, "dtype": cfg.dtype, "data": "synthetic",
               "config": {"workload": cfg.name, "tokens_per_rank": T, "global_tokens": world * T,
                          "E": E, "k": cfg.top_k, "d_model": cfg.d_model, "d_ffn": cfg.d_ffn, "act": cfg.act,
                          "h": cfg.h, "parallelism": f"ep{world}",
                          "l2": "per-step working set (~1 GB activations) exceeds the 126 MB L2; no explicit flush"},
               "condensed_frac_rows": frac_all, "a2a_bytes_condensed_frac": frac_remote,
               "greedy_rounds": rounds, "reps_rank0": R,
               "migration": ({"q": args.migrate, **mig_stats} if mig else None),
               "breakdown_ms": breakdown, "roofline": roof, "roofline_gram": gram_roof, "roofline_memory": mem_roof,
               "kernel_shares": shares, "nvlink": nvlink, "cpu_baseline": cpu, "e2e": e2e,
               "gpu_launches": int(launches), "host_enqueue_ms_per_step": host_ms, "clocks": clocks,
               "step_exec": "cuda_graph_replay" if graph is not None else "eager"}
        print(json.dumps(out), flush=True)
    lay.close()
    if world > 1:
        dist.destroy_process_group()


if __name__ == "__main__":
    main()
