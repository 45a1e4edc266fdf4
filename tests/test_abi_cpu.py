"""CPU checks of the C-ABI library: it loads without a GPU, exports every symbol include/luffy.h
declares, validates configs on the host, and its host-side planner (Alg. 1) matches the oracle."""
import os
import re

import numpy as np
import pytest

import workload
from oracle import luffy_oracle as O

ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


@pytest.fixture(scope="module")
def L():
    from paper_2411_15419_b200 import build
    build.build()
    from paper_2411_15419_b200 import luffy
    return luffy


def test_exports_every_declared_symbol(L):
    hdr = open(os.path.join(ROOT, "include", "luffy.h")).read()
    declared = set(re.findall(r"LUFFY_API\s+[\w\s\*]+?\b(luffy_\w+)\s*\(", hdr))
    assert declared == set(L.EXPORTED)
    out = os.popen(f"nm -D --defined-only {L._LIB_PATH}").read()
    exported = set(re.findall(r" T (luffy_\w+)", out))
    assert declared <= exported


def test_workspace_validation(L):
    good = L.make_config(num_experts=8, top_k=2, d_model=1024, d_ffn=4096, max_tokens=8192)
    assert L.luffy_layer_workspace_bytes(good) > 0
    for bad in [dict(num_experts=7, world=2), dict(top_k=9), dict(d_model=1000), dict(max_tokens=0),
                dict(dtype=5), dict(world=2, rank=2)]:
        kw = dict(num_experts=8, top_k=2, d_model=1024, d_ffn=4096, max_tokens=8192)
        kw.update(bad)
        with pytest.raises(L.LuffyError):
            L.luffy_layer_workspace_bytes(L.make_config(**kw))


def test_attention_cost_matches_eq1(L):
    for line in open(os.path.join(ROOT, "tests", "golden", "eq1_attention_cost.txt")):
        if line.strip() and not line.startswith("#"):
            B, Ln, d, P, exp = map(int, line.split())
            assert L.luffy_attention_cost(B, Ln, d) == exp
    rng = np.random.default_rng(0)
    for _ in range(100):
        B, Ln, d = (int(x) for x in rng.integers(0, 5000, 3))
        assert L.luffy_attention_cost(B, Ln, d) == O.attention_cost(B, Ln, d)


@pytest.mark.parametrize("objective", ["min", "max"])
def test_planner_matches_oracle(L, objective):
    rng = np.random.default_rng(1)
    for trial in range(300):
        S, P = int(rng.integers(1, 40)), int(rng.integers(1, 9))
        seq_len = rng.integers(1, 1025, S)
        rows_at = rng.integers(0, 600, (S, P))
        q = int(rng.integers(1, P + 1))
        d = int(rng.choice([8, 768, 1024, 4096]))
        cap = int(rng.choice([0, 0, int(seq_len.max())]))
        try:
            od, oc = O.plan_migration(seq_len, rows_at, q, 2048, d, capacity=cap, objective=objective)
        except O.PlanningError:
            with pytest.raises(L.LuffyError):
                L.luffy_plan_migration(seq_len, rows_at, q, 2048, d, capacity_tokens=cap,
                                       objective=0 if objective == "min" else 1)
            continue
        gd, gc = L.luffy_plan_migration(seq_len, rows_at, q, 2048, d, capacity_tokens=cap,
                                        objective=0 if objective == "min" else 1)
        assert np.array_equal(gd, od), trial
        assert np.array_equal(gc, oc), trial


def test_planner_paper_workload_and_worked_values(L):
    seq_len, home, rows_at = workload.make_migration_problem(128, 8)
    for q in (1, 2, 4, 8):
        od, oc = O.plan_migration(seq_len, rows_at, q, 2 * 2048, 2048)
        gd, gc = L.luffy_plan_migration(seq_len, rows_at, q, 2 * 2048, 2048)
        assert np.array_equal(od, gd) and np.array_equal(oc, gc)
    # 3 copies on device 0, 1 on device 1, 64-byte rows; one sequence, q=1 -> device 0
    d, c = L.luffy_plan_migration([4], [[3, 1]], 1, 64, 8)
    assert d[0] == 0 and c[1, 0] == 64


def test_planner_rejects_bad_arguments(L):
    with pytest.raises(L.LuffyError):
        L.luffy_plan_migration([3], [[1, 1]], 0, 8, 8)          # q < 1
    with pytest.raises(L.LuffyError):
        L.luffy_plan_migration([10, 10], [[1, 1], [1, 1]], 2, 8, 8, capacity_tokens=5)


def test_every_kernel_enters_through_pdl():
    """Kernels are launched with programmatic stream serialization; correctness along the stream needs
    every kernel to execute griddepcontrol.wait (pdl_enter) before its first global access, and no launch
    may bypass launch_pdl (a <<<>>> launch would not carry the attribute; harmless, but unmeasured)."""
    csrc = os.path.join(ROOT, "paper_2411_15419_b200", "csrc")
    kernels = 0
    for fn in sorted(os.listdir(csrc)):
        if not fn.endswith((".cu", ".cuh")):
            continue
        src = open(os.path.join(csrc, fn)).read()
        code = re.sub(r"//[^\n]*", "", src)
        assert "<<<" not in code, f"{fn}: raw <<<>>> launch"
        for m in re.finditer(r"__global__[^;{]*?\)\s*\{", code, re.S):
            body = code[m.end():m.end() + 200].lstrip()
            if body.startswith("pdl_defer();"):
                # deferred wait (tensor-core kernels): pdl_enter() follows the prologue and comes before the
                # first read of a kernel-argument pointer (a.*[...]) in the kernel
                full = code[m.end():]
                end = full.find("\n}\n")
                k = full[:end]
                i_enter = k.find("pdl_enter();")
                assert i_enter > 0, f"{fn}: pdl_defer() without pdl_enter()"
                first_read = re.search(r"\ba\.\w+\[", k)
                assert first_read is None or first_read.start() > i_enter, f"{fn}: global read before pdl_enter()"
            else:
                assert body.startswith("pdl_enter();"), f"{fn}: kernel at offset {m.start()} does not start with pdl_enter()"
            kernels += 1
    assert kernels >= 30


def test_adaptive_threshold_eq2(L):
    """Eq. (2) in the library: as printed it equals the oracle and the worked values; the factor-2
    reading R17b doubles it (range [2/(1+e), 1]); h decreases as the loss falls; invalid inputs raise."""
    rows = [ln.split() for ln in open(os.path.join(ROOT, "tests", "golden", "eq2_adaptive_threshold.txt"))
            if ln.strip() and not ln.startswith("#")]
    for l_ini, l_prev, want in rows:
        h = L.luffy_adaptive_threshold(float(l_ini), float(l_prev))
        assert abs(h - float(want)) < 5e-6
    rng = np.random.default_rng(7)
    prev_h = None
    for l_prev in np.linspace(12.0, 0.0, 25):
        h1 = L.luffy_adaptive_threshold(10.0, l_prev)
        h2 = L.luffy_adaptive_threshold(10.0, l_prev, scale2=True)
        assert abs(h1 - O.adaptive_threshold(10.0, l_prev)) < 1e-6
        assert abs(h2 - 2 * h1) < 1e-6 and 2 / (1 + np.e) - 1e-6 <= h2 <= 1.0
        if prev_h is not None:
            assert h1 <= prev_h + 1e-7
        prev_h = h1
    for l_ini, l_prev in rng.uniform(0.1, 20.0, size=(50, 2)):
        assert abs(L.luffy_adaptive_threshold(l_ini, l_prev) - O.adaptive_threshold(l_ini, l_prev)) < 1e-6
    with pytest.raises(L.LuffyError):
        L.luffy_adaptive_threshold(0.0, 1.0)
    with pytest.raises(L.LuffyError):
        L.luffy_adaptive_threshold(1.0, float("nan"))
