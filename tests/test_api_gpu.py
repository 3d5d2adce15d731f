"""GPU parity of the reference's remaining public path API against goldens
made by the unmodified reference (tests/golden/make_golden_api.py):
apply_shift / apply_swap sequences (incl. REFRESH_PERIOD crossings),
accept verdicts, the operator bank's select/update trajectory and
best_swap with the l2 tie-break over several worker counts.  Bitwise."""

import numpy as np
import pytest

from tests.golden_io import load

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def P():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    import paper_2508_13437_b200 as P
    from paper_2508_13437_b200 import _native

    _native.load_library()
    return P


def _inst_sol(P, rec):
    inst = P.Instance(rec["A"], rec["b"], P.ValueSet(rec["levels"]))
    sol = P.Solution(rec["idx0"], rec["r0"], rec["obj0"], int(rec["cnt0"]))
    return inst, sol


@pytest.mark.parametrize("k", range(24))
def test_apply_shift_sequence(P, k):
    rec = load("api_shift")[k]
    inst, sol = _inst_sol(P, rec)
    for q, (j, lvl) in enumerate(zip(rec["js"], rec["ls"])):
        P.apply_shift(inst, sol, int(j), int(lvl))
        assert sol.objective == rec["objs"][q], q
        assert sol.updates_since_refresh == rec["cnts"][q], q
    np.testing.assert_array_equal(sol.idx, rec["idx1"])
    np.testing.assert_array_equal(sol.residual, rec["r1"])
    assert sol.objective == rec["obj1"] and sol.updates_since_refresh == rec["cnt1"]


@pytest.mark.parametrize("k", range(24))
def test_apply_swap_sequence(P, k):
    rec = load("api_swap")[k]
    inst, sol = _inst_sol(P, rec)
    for q, (i, j) in enumerate(zip(rec["is"], rec["js"])):
        P.apply_swap(inst, sol, int(i), int(j))
        assert sol.objective == rec["objs"][q], q
        assert sol.updates_since_refresh == rec["cnts"][q], q
    np.testing.assert_array_equal(sol.idx, rec["idx1"])
    np.testing.assert_array_equal(sol.residual, rec["r1"])


def test_refresh_crossed_in_goldens():
    """The sequences above do cross REFRESH_PERIOD (counter reset to 0)."""
    for name in ("api_shift", "api_swap"):
        assert any((np.diff(r["cnts"]) < 0).any() for r in load(name)), name


def test_accept_verdicts(P):
    for rec in load("api_accept"):
        cur = P.Solution(np.zeros(1, np.intp), rec["cur_r"], rec["cur_obj"])
        cand = P.Solution(np.zeros(1, np.intp), rec["cand_r"], rec["cand_obj"])
        for l2 in (0, 1):
            got = P.accept(cur, cand, P.SolverConfig(l2_tiebreak=bool(l2)))
            assert int(got) == rec[f"verdict_l2_{l2}"], (rec["cur_r"].size, l2)


@pytest.mark.parametrize("k", range(12))
def test_operator_bank_trajectory(P, k):
    rec = load("api_bank")[k]
    s1, s2, s3 = rec["sigma"]
    cfg = P.SolverConfig(decay=float(rec["decay"]), sigma1=s1, sigma2=s2, sigma3=s3)
    bank = P.OperatorBank(float(rec["decay"]))
    rng = np.random.default_rng(int(rec["seed"]))
    outs = (P.OUTCOME_NEW_BEST, P.OUTCOME_IMPROVED, P.OUTCOME_ACCEPTED, P.OUTCOME_REJECTED)
    for it, o in enumerate(rec["outcomes"]):
        p = P.select_operators(bank, rng)
        assert p == rec["picks"][it], it
        P.update_weights(bank, p, outs[int(o)], cfg)
    np.testing.assert_array_equal(bank.weights, rec["weights"])
    np.testing.assert_array_equal(bank.scores, rec["scores"])
    np.testing.assert_array_equal(bank.segment_uses, rec["segment_uses"])
    np.testing.assert_array_equal(bank.lifetime_uses, rec["lifetime_uses"])
    assert bank.iteration == rec["iteration"]
    st = rng.bit_generator.state
    want = [int(x) for x in rec["state_after"]]
    assert [st["state"]["state"] >> 64, st["state"]["state"] & (2**64 - 1), st["state"]["inc"] >> 64,
            st["state"]["inc"] & (2**64 - 1), st["has_uint32"], st["uinteger"]] == want


@pytest.mark.parametrize("k", range(41))
def test_best_swap_l2_tiebreak(P, k):
    rec = load("api_swap_l2")[k]
    inst, sol = _inst_sol(P, rec)
    for workers, k_eps, mc, i, j, d, t in rec["runs"]:
        fc = P.FilterConfig(k_eps=int(k_eps), max_candidates=None if mc < 0 else int(mc), workers=int(workers),
                            l2_tiebreak=True)
        got = P.best_swap(inst, sol, fc)
        if i < 0:
            assert got is None
        else:
            assert got is not None, (workers, k_eps, mc)
            assert (got.i, got.j, got.delta, got.predicted_t) == (int(i), int(j), d, t), (workers, k_eps, mc)


def test_reference_tie_instance(P):
    """tests/test_localsearch.py:320-332: lexicographic (0, 1) without the
    tie-break, the smaller-residual (2, 3) with it."""
    inst = P.Instance(np.column_stack([[0.4, 0.0, 0.0, 0.5], [-0.4, 0.0, 0.0, 0.5], [0.4, 0.0, -0.45, -0.5],
                                       [-0.4, 0.0, 0.45, -0.5]]), np.array([-0.1, -0.5, 0.05, 0.0]),
                      P.ValueSet(np.array([0.0, 1.0])))
    sol = P.Solution.from_indices(inst, np.array([1, 0, 1, 0]))
    got = P.best_swap(inst, sol, P.FilterConfig(l2_tiebreak=False))
    assert (got.i, got.j, got.predicted_t) == (0, 1, 0.5)
    got = P.best_swap(inst, sol, P.FilterConfig(l2_tiebreak=True))
    assert (got.i, got.j, got.predicted_t) == (2, 3, 0.5)
