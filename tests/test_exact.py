"""Exact oracle (dmmv.oracle.brute_force, oracle.py:38-111): the numpy
restatement and the GPU enumeration (amvm_brute_force) against the
reference's own results (tests/golden/brute_force.npz, made by
make_golden_exact.py) — bit-exact best_t and best_idx for both arithmetic
orders (prune=False / prune=True) — and the GPU against the restatement on
instances too large for the reference's pruned DFS to be quick."""

import numpy as np
import pytest

from tests.golden_io import load


def test_oracle_brute_force_matches_reference_goldens():
    from oracle import oracle as O

    recs = load("brute_force")
    assert len(recs) >= 19
    for r in recs:
        for prune, key in ((False, ""), (True, "pruned_")):
            idx, t, enum = O.brute_force(r["A"], r["b"], r["levels"], prune=prune)
            np.testing.assert_array_equal(idx, r[f"{key}best_idx"])
            assert t == r[f"{key}best_t"]
        assert enum == r["enumerated"]


def test_budget_check_precedes_any_device_work(monkeypatch):
    """BudgetExceededError (oracle.py:19-28,53-55) is raised on the host, with
    the reference's message, before the device is touched."""
    import torch

    import paper_2508_13437_b200 as P

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    inst = P.Instance(np.ones((2, 30)), np.ones(2), P.ValueSet([0.0, 1.0]))
    with pytest.raises(P.BudgetExceededError, match=r"needs 1073741824 assignments but the budget is 10000000"):
        P.brute_force(inst)
    with pytest.raises(ValueError):
        P.brute_force(inst, budget=5)
    from paper_2508_13437_b200 import _native
    with pytest.raises(_native.NativeUnavailable):
        P.brute_force(P.Instance(np.ones((2, 3)), np.ones(2), P.ValueSet([0.0, 1.0])))


@pytest.fixture(scope="module")
def amvm():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    import paper_2508_13437_b200 as P

    return P


@pytest.mark.gpu
def test_gpu_brute_force_matches_reference_goldens(amvm):
    P = amvm
    for r in load("brute_force"):
        inst = P.Instance(r["A"], r["b"], P.ValueSet(r["levels"]))
        for prune, key in ((False, ""), (True, "pruned_")):
            res = P.brute_force(inst, prune=prune)
            np.testing.assert_array_equal(res.best_idx, r[f"{key}best_idx"])
            assert res.best_t == r[f"{key}best_t"], (key, res.best_t, r[f"{key}best_t"])
            assert res.enumerated == r["enumerated"]


@pytest.mark.gpu
@pytest.mark.parametrize("m,n,nlev,kind", [(48, 14, 3, "float"), (200, 8, 7, "float"), (12, 20, 2, "int"),
                                           (3000, 9, 3, "float"), (30, 11, 4, "int"),
                                           (1, 9, 4, "float"), (1, 11, 3, "float")])
def test_gpu_brute_force_matches_oracle_large(amvm, m, n, nlev, kind):
    """Up to 4.8M codes; m = 3000 exceeds the shared-memory staging of A
    (the global-memory path).  Integer data: many exact ties, so the
    lexicographic tie-break is exercised."""
    from oracle import oracle as O

    P = amvm
    rng = np.random.default_rng(m * 1000 + n)
    if kind == "float":
        A = rng.uniform(-1, 1, (m, n))
        lv = np.sort(rng.uniform(-2, 2, nlev))
        b = A @ rng.uniform(lv[0], lv[-1], n)
    else:
        A = rng.integers(-2, 3, (m, n)).astype(float)
        lv = np.arange(nlev, dtype=float) - nlev // 2
        b = rng.integers(-3, 4, m).astype(float)
    inst = P.Instance(A, b, P.ValueSet(lv))
    for prune in (False, True):
        idx, t, enum = O.brute_force(A, b, lv, prune=prune)
        res = P.brute_force(inst, prune=prune)
        np.testing.assert_array_equal(res.best_idx, idx)
        assert res.best_t == t
        assert res.enumerated == enum
