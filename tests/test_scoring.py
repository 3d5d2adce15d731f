"""Batched candidate-move scoring (``amvm_score_moves``) against the oracle's
numpy restatement of the one_opt candidate objective
(localsearch.py:76-78): every score bitwise, the best move identical.
Edge cases: m below / not a multiple of the warp, one column, one level (no
move), more levels than one register pass (C2-like 1024-level grid), levels
at both ends of the grid, shared-A batches."""

import numpy as np
import pytest

from oracle import oracle as O

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


CASES = [(64, 16, 5), (1, 7, 4), (31, 9, 3), (33, 1, 6), (100, 40, 16), (257, 33, 17), (5, 6, 1),
         (2048, 96, 16), (300, 20, 1024), (128, 64, 2),
         # k_score_adj (adjacent set, even m <= 8192): 1..4 columns per stage,
         # up to 16 rows per thread, more slabs than SMs, fewer columns than SMs
         (8192, 37, 16), (4096, 300, 16), (1500, 600, 16), (1000, 1000, 8), (6000, 5, 3), (2, 3, 4)]


def _instance(P, m, n, nlev, seed, integer=False):
    rng = np.random.default_rng(seed)
    if integer:
        A = rng.integers(-3, 4, (m, n)).astype(float)
        lv = np.arange(nlev, dtype=float) - nlev // 2
    else:
        A = rng.normal(0, 1, (m, n))
        lv = np.sort(rng.choice(np.linspace(-4, 4, max(4 * nlev, 8) + 1), nlev, replace=False))
    idx = rng.integers(0, nlev, n)
    idx[: min(2, n)] = [0, nlev - 1][: min(2, n)]  # both ends of the grid
    b = A @ lv[rng.integers(0, nlev, n)] + rng.normal(0, 0.3, m)
    inst = P.Instance(A, b, P.ValueSet(lv))
    return inst, P.Solution.from_indices(inst, idx)


@pytest.mark.parametrize("mode", ["adjacent", "all"])
@pytest.mark.parametrize("case", range(len(CASES)))
@pytest.mark.parametrize("integer", [False, True])
def test_scores_bitwise_vs_oracle(P, case, mode, integer):
    m, n, nlev = CASES[case]
    inst, sol = _instance(P, m, n, nlev, 100 + case, integer)
    got = P.score_moves(inst, sol, mode)
    t, best, best_t = O.score_moves(inst.A, sol.residual, inst.values.levels, sol.idx, mode)
    np.testing.assert_array_equal(got.t, t)
    assert got.best == best
    if best is not None:
        assert got.best_t == best_t
        assert got.improving == (best_t < sol.objective)
    if mode == "all":
        np.testing.assert_array_equal(got.t[np.arange(n), sol.idx], np.full(n, sol.objective))


def test_adjacent_move_agrees_with_engine_one_opt_first_step(P):
    """The reference's one_opt takes, in its first sweep, the first column
    whose best adjacent score beats the objective: the scores say which."""
    inst, sol = _instance(P, 512, 64, 16, 7)
    sc = P.score_moves(inst, sol, "adjacent")
    t, _, _ = O.score_moves(inst.A, sol.residual, inst.values.levels, sol.idx, "adjacent")
    first = next((j for j in range(inst.n) if t[j].min() < sol.objective), None)
    got = next((j for j in range(inst.n) if sc.t[j].min() < sol.objective), None)
    assert got == first


def test_shared_A_batch_matches_single_instances(P):
    import torch

    from paper_2508_13437_b200 import _native as N
    from paper_2508_13437_b200.scoring import score_moves_device

    rng = np.random.default_rng(5)
    m, n, nlev, count = 200, 48, 16, 6
    A = rng.normal(0, 1, (m, n))
    LV = np.sort(rng.normal(0, 1, (count, nlev)), axis=1)
    IDX = rng.integers(0, nlev, (count, n))
    S = rng.normal(0, 0.5, (count, m))
    dev = torch.device("cuda", 0)
    At = torch.from_numpy(np.ascontiguousarray(A.T)).to(dev)
    lv = torch.from_numpy(LV).to(dev)
    B = torch.zeros((count, m), dtype=torch.float64, device=dev)
    prob = N.Problem(m, n, nlev, count, At.data_ptr(), B.data_ptr(), lv.data_ptr())
    for mode in ("adjacent", "all"):
        t, best, best_t = score_moves_device(prob, torch.from_numpy(IDX.astype(np.int32)).to(dev),
                                             torch.from_numpy(S).to(dev), mode)
        t = t.cpu().numpy()
        for c in range(count):
            tr, br, btr = O.score_moves(A, S[c], LV[c], IDX[c], mode)
            np.testing.assert_array_equal(t[c], tr)
            nv = t.shape[2]
            j, v = divmod(int(best[c]), nv)
            lvl = IDX[c, j] + (-1 if v == 0 else 1) if mode == "adjacent" else v
            assert (j, lvl) == br and float(best_t[c]) == btr


def test_bad_mode_is_a_value_error(P):
    inst, sol = _instance(P, 8, 4, 3, 1)
    with pytest.raises(ValueError, match="mode must be one of"):
        P.score_moves(inst, sol, "every")


def test_adjacent_batch_and_workspace_reuse(P):
    """Several instances per k_score_adj launch (every slab CTA walks all of
    them; per-instance tickets) and back-to-back calls on one workspace (the
    kernel leaves its ticket counters at zero)."""
    import torch

    from paper_2508_13437_b200 import _native as N
    from paper_2508_13437_b200.scoring import score_moves_device

    rng = np.random.default_rng(9)
    m, n, nlev, count = 2048, 700, 16, 3
    A = rng.normal(0, 1, (m, n))
    LV = np.sort(rng.normal(0, 1, (count, nlev)), axis=1)
    dev = torch.device("cuda", 0)
    At = torch.from_numpy(np.ascontiguousarray(A.T)).to(dev)
    lv = torch.from_numpy(LV).to(dev)
    B = torch.zeros((count, m), dtype=torch.float64, device=dev)
    prob = N.Problem(m, n, nlev, count, At.data_ptr(), B.data_ptr(), lv.data_ptr())
    ws = torch.zeros(int(N.load_library().amvm_score_workspace_bytes(N.C.byref(prob))), dtype=torch.uint8,
                     device=dev)
    for rep in range(3):
        IDX = rng.integers(0, nlev, (count, n))
        S = rng.normal(0, 0.5, (count, m))
        t, best, best_t = score_moves_device(prob, torch.from_numpy(IDX.astype(np.int32)).to(dev),
                                             torch.from_numpy(S).to(dev), "adjacent", ws)
        t = t.cpu().numpy()
        for c in range(count):
            tr, br, btr = O.score_moves(A, S[c], LV[c], IDX[c], "adjacent")
            np.testing.assert_array_equal(t[c], tr)
            j, v = divmod(int(best[c]), 2)
            assert (j, IDX[c, j] + (-1 if v == 0 else 1)) == br and float(best_t[c]) == btr, (rep, c)


def test_device_api_rejects_bad_inputs(P):
    import torch

    from paper_2508_13437_b200 import _native as N
    from paper_2508_13437_b200.scoring import score_moves_device

    dev = torch.device("cuda", 0)
    m, n, nlev = 16, 8, 4
    At = torch.zeros((n, m), dtype=torch.float64, device=dev)
    lv = torch.arange(nlev, dtype=torch.float64, device=dev)[None]
    B = torch.zeros((1, m), dtype=torch.float64, device=dev)
    prob = N.Problem(m, n, nlev, 1, At.data_ptr(), B.data_ptr(), lv.data_ptr())
    s = torch.zeros((1, m), dtype=torch.float64, device=dev)
    idx = torch.zeros((1, n), dtype=torch.int32, device=dev)
    with pytest.raises(ValueError, match="int32"):
        score_moves_device(prob, idx.long(), s)
    with pytest.raises(ValueError, match="float64"):
        score_moves_device(prob, idx, s.float())
    with pytest.raises(ValueError, match="lie in"):
        score_moves_device(prob, idx + nlev, s)
    with pytest.raises(ValueError, match="finite"):
        score_moves_device(prob, idx, s * float("nan"))
