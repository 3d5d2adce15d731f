"""Candidate-move scorer against golden objectives made by the unmodified
reference's apply_shift (tests/golden/make_golden_scoring.py): the oracle's
restatement on CPU, the CUDA path (``amvm_score_moves``) on the GPU, both
bitwise, both modes."""

import numpy as np
import pytest

from oracle import oracle as O
from tests.golden_io import load

REC = load("scoring")


def _adjacent(rec):
    t = rec["t_all"]
    n, nlev = t.shape
    out = np.full((n, 2), np.inf)
    for j in range(n):
        k = int(rec["idx"][j])
        if k > 0:
            out[j, 0] = t[j, k - 1]
        if k + 1 < nlev:
            out[j, 1] = t[j, k + 1]
    return out


@pytest.mark.parametrize("k", range(len(REC)))
def test_oracle_scores_equal_reference_apply_shift(k):
    rec = REC[k]
    t, best, best_t = O.score_moves(rec["A"], rec["residual"], rec["levels"], rec["idx"], "all")
    np.testing.assert_array_equal(t, rec["t_all"])
    ta, _, _ = O.score_moves(rec["A"], rec["residual"], rec["levels"], rec["idx"], "adjacent")
    np.testing.assert_array_equal(ta, _adjacent(rec))


@pytest.mark.gpu
@pytest.mark.parametrize("k", range(len(REC)))
def test_device_scores_equal_reference_apply_shift(k):
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    import paper_2508_13437_b200 as P

    rec = REC[k]
    inst = P.Instance(rec["A"], rec["b"], P.ValueSet(rec["levels"]))
    sol = P.Solution(np.asarray(rec["idx"]), rec["residual"], float(rec["objective"]), 0)
    sc = P.score_moves(inst, sol, "all")
    np.testing.assert_array_equal(sc.t, rec["t_all"])
    np.testing.assert_array_equal(P.score_moves(inst, sol, "adjacent").t, _adjacent(rec))
