"""Multi-GPU parity (NCCL dispatch/combine over NVLink): torchrun with 2 (and 4 when available) ranks,
each checked against the fp64 oracle by tests/mp_gpu_worker.py."""
import os
import socket
import subprocess
import sys

import pytest
import torch

pytestmark = pytest.mark.gpu
ROOT = os.path.dirname(os.path.dirname(os.path.abspath(__file__)))


def _port():
    s = socket.socket()
    s.bind(("127.0.0.1", 0))
    p = s.getsockname()[1]
    s.close()
    return p


def _run(n, config, h=0.9, extra=(), env=None):
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", "mp_gpu_worker.py"),
           "--config", config, "--h", str(h), *extra]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT,
                       env=dict(os.environ, **(env or {})))
    print(r.stdout[-4000:], r.stderr[-4000:])
    return r


@pytest.mark.parametrize("n,config,h", [(2, "C2S", 0.9), (2, "C2S", 1.01), (2, "C1", 0.9), (4, "C2S", 0.9),
                                        (2, "C2", 0.9)])
def test_expert_parallel_parity(n, config, h):
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    r = _run(n, config, h)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count('"ok": true') == n


def test_expert_parallel_parity_warp_push():
    """The warp-store dispatch push (LUFFY_PUSH_TMA=0) against the same oracle as the default TMA push."""
    if torch.cuda.device_count() < 2:
        pytest.skip("needs 2 GPUs")
    r = _run(2, "C2S", 0.9, env={"LUFFY_PUSH_TMA": "0"})
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count('"ok": true') == 2


@pytest.mark.parametrize("n,extra", [(2, ("--residual",)), (4, ("--residual",))])
def test_residual_block_parity(n, extra):
    """Residual block y = x + MoE(x) (luffy_uncondense_residual / luffy_dispatch_bwd_residual) at world > 1."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    r = _run(n, "C2S", 0.9, extra=extra)
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count('"ok": true') == n


@pytest.mark.parametrize("n,mode,extra", [(2, "rotate", ()), (2, "plan", ()), (4, "plan", ()), (4, "rotate", ()),
                                          (2, "plan", ("--residual", "--uneven")),
                                          (4, "rotate", ("--residual", "--uneven"))])
def test_sequence_migration_parity(n, mode, extra):
    """Alg. 1 in the layer: K9 rows_at exact vs the oracle, the planner's seq_dest equal to the oracle's
    Alg. 1, outputs at the hosting rank and all gradients at home / expert ranks within tolerance."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    r = _run(n, "C2S", 0.9, extra=("--migrate", mode, "--q", "2") + tuple(extra))
    assert r.returncode == 0, r.stdout[-3000:] + r.stderr[-3000:]
    assert r.stdout.count('"ok": true') == n


@pytest.mark.parametrize("n", [2, 4])
def test_graph_replay_world_gt1(n):
    """Two captured world > 1 steps replayed alternately give the eager step's outputs bitwise
    (tests/mp_graph_worker.py): the exchange flags carry the device step number."""
    if torch.cuda.device_count() < n:
        pytest.skip(f"needs {n} GPUs")
    cmd = [sys.executable, "-m", "torch.distributed.run", "--nnodes=1", f"--nproc-per-node={n}",
           "--master-addr", "127.0.0.1", f"--master-port={_port()}", os.path.join(ROOT, "tests", "mp_graph_worker.py")]
    r = subprocess.run(cmd, capture_output=True, text=True, timeout=900, cwd=ROOT)
    print(r.stdout[-3000:], r.stderr[-3000:])
    assert r.returncode == 0, r.stdout[-2000:] + r.stderr[-2000:]
    assert r.stdout.count('"ok": true') == n
