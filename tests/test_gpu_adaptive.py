"""Eq. (2) driving the condensation threshold from the training loss (§8(f) row 2): a student
condensed MoE layer regresses a teacher through libluffy's forward/backward with SGD on the experts; each
iteration's h equals the oracle's Eq. (2) (reading R17, c = 2) of the logged losses, starts at 1 (only
exact duplicates condensed) and the condensed fraction grows as the loss falls."""
import dataclasses

import numpy as np
import pytest

import workload
from oracle import luffy_oracle as O

pytestmark = pytest.mark.gpu


def test_adaptive_threshold_training_loop():
    from paper_2411_15419_b200 import adaptive as AD
    cfg = dataclasses.replace(workload.CONFIGS["C2"], seqs_per_rank=2, d_ffn=1024)
    inp = workload.make_layer_inputs(cfg)
    log = AD.train_adaptive(cfg, inp, iters=30)
    losses = [r["loss"] for r in log]
    print("\n" + "\n".join(f"it {r['iter']:2d} h {r['h']:.4f} loss {r['loss']:.5f} condensed {r['condensed_frac']:.3f}"
                           for r in log))
    assert log[0]["h"] == 1.0
    for t in range(1, len(log)):        # h_t from l_ini = loss_0 and l_{t-1} (Eq. 2, c = 2)
        assert abs(log[t]["h"] - O.adaptive_threshold(losses[0], losses[t - 1], c=2.0)) < 1e-6
    assert losses[-1] < 0.8 * losses[0], "the loss must fall for the threshold to adapt"
    assert log[-1]["h"] < log[1]["h"] - 0.02
    assert log[-1]["condensed_frac"] > log[0]["condensed_frac"]
