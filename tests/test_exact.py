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


def test_swap_check_host_validation(monkeypatch):
    """n > 64 and delta <= 0 are rejected before any device work, with the
    reference's messages (oracle.py:142-143, localsearch.py:110-111)."""
    import torch

    import paper_2508_13437_b200 as P

    monkeypatch.setattr(torch.cuda, "is_available", lambda: False)
    inst = P.Instance(np.ones((2, 65)), np.ones(2), P.ValueSet([0.0, 1.0]))
    sol = P.Solution.from_indices(inst, np.zeros(65, dtype=np.intp))
    with pytest.raises(ValueError, match="restricted to n <= 64"):
        P.exhaustive_swap_check(inst, sol)
    with pytest.raises(ValueError, match="delta = x_i - x_j > 0"):
        P.is_improving(inst, sol, P.SwapCandidate(0, 1, 0.0))


@pytest.mark.gpu
def test_gpu_swap_check_matches_reference(amvm):
    """Every pair's recomputed objective bitwise (numpy's compute_residual
    order, incl. the m = 1 ddot path), every verdict, and the report."""
    from paper_2508_13437_b200.exact import is_improving_batch

    P = amvm
    recs = load("swap_check")
    assert len(recs) >= 7
    for r in recs:
        inst = P.Instance(r["A"], r["b"], P.ValueSet(r["levels"]))
        sol = P.Solution.from_indices(inst, r["idx"].astype(np.intp))
        assert sol.objective == r["objective"]
        rep = P.exhaustive_swap_check(inst, sol)
        assert rep.pairs_checked == r["pairs_checked"]
        assert len(rep.discrepancies) == r["n_discrepancies"] and len(rep.boundary) == r["n_boundary"]
        x = sol.values(inst)
        pairs = [(i, j) for i in range(inst.n) for j in range(inst.n) if i != j and x[i] > x[j]]
        cands = [P.SwapCandidate(i, j, float(x[i] - x[j])) for i, j in pairs]
        v = is_improving_batch(inst, sol, cands)
        np.testing.assert_array_equal(v, [bool(r["V"][i, j]) for i, j in pairs])
        assert P.is_improving(inst, sol, cands[0]) == bool(r["V"][pairs[0]])
        # the per-pair objectives behind the report, bit for bit
        from paper_2508_13437_b200 import _native as N
        import torch
        dev = torch.device("cuda")
        At, b, lv = inst.device_arrays(dev)
        prob = N.Problem(inst.m, inst.n, len(inst.values), 1, At.data_ptr(), b.data_ptr(), lv.data_ptr())
        idx = torch.from_numpy(r["idx"]).to(dev)
        s = torch.from_numpy(sol.residual).to(dev)
        T = torch.zeros(inst.n * inst.n, dtype=torch.float64, device=dev)
        V = torch.zeros(inst.n * inst.n, dtype=torch.int32, device=dev)
        N.check(N.load_library().amvm_swap_check(N.C.byref(prob), N.ptr(idx), N.ptr(s), float(sol.objective),
                                                 N.ptr(T), N.ptr(V), N.stream_handle()), "amvm_swap_check")
        T = T.cpu().numpy().reshape(inst.n, inst.n)
        for i, j in pairs:
            assert T[i, j] == r["T"][i, j], (i, j, T[i, j], r["T"][i, j])
