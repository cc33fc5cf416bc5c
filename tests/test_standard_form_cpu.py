"""CPU checks of the standard-form golden traces (tests/golden/standard_golden.npz,
made by the reference's standard_form.hpp) and of the host-side mirror: the
trace bookkeeping the GPU harness reproduces (epoch lengths add up to the
iteration count, restart decay by beta per epoch, the restart chain of an
already-optimal start), and option validation. GPU runs: test_gpu_standard_form.py."""
from __future__ import annotations

from pathlib import Path

import numpy as np
import pytest

from paper_2311_12180_b200.lp import CsrMatrix
from paper_2311_12180_b200.standard_form import StandardFormLp, StandardPdhgOptions

G = np.load(Path(__file__).resolve().parent / "golden" / "standard_golden.npz")
NAMES = ["f0", "f1", "f2", "f3", "f4", "r30x60", "r200x500"]


@pytest.mark.parametrize("name", NAMES)
def test_golden_trace_bookkeeping(name):
    kkt, lens, cnt = G[f"{name}/kkt"], G[f"{name}/lens"], G[f"{name}/counters"]
    s, beta, tol, limit = G[f"{name}/params"]
    assert len(kkt) == len(lens) == cnt[0]
    assert lens.sum() == cnt[1]  # every inner iteration belongs to one epoch
    assert np.all(kkt[1:] <= beta * kkt[:-1] * (1 + 1e-12))  # restart fires at KKT(avg) <= beta KKT(start)
    if cnt[2]:
        assert kkt[-1] <= tol and lens[-1] == 0
    else:
        assert cnt[1] == limit
    # step within the theorem's range: s = 0.9 / (2 ||A||)
    assert s == pytest.approx(0.9 / (2.0 * G[f"{name}/norm"][0]), rel=1e-15)
    n, m = len(G[f"{name}/c"]), len(G[f"{name}/b"])
    assert G[f"{name}/iter_x"].shape == (min(200, cnt[1]), n) and G[f"{name}/iter_y"].shape[1] == m


def test_golden_restart_chain():
    assert G["chain/counters"][1] == 10 and np.all(G["chain/kkt"] == 0.0) and np.all(G["chain/lens"] <= 1)


def test_options_and_lp_validation():
    with pytest.raises(ValueError, match="step_size must be positive"):
        StandardPdhgOptions(step_size=0.0).validate()
    with pytest.raises(ValueError, match="restart_decay must lie"):
        StandardPdhgOptions(step_size=0.1, restart_decay=1.0).validate()
    StandardPdhgOptions(step_size=0.1).validate()
    a = CsrMatrix(1, 2, np.array([0, 1]), np.array([0]), np.array([1.0]))
    with pytest.raises(ValueError, match="dimension mismatch"):
        StandardFormLp(a, np.ones(2), np.ones(2)).validate()
