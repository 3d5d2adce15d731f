"""Device warm start (amvm_ls_start): initial_solution's regularised
least-squares start (controller.py:134-165) on the GPU, against the
reference's own starts stored in the goldens (idx0, made by numpy/LAPACK).

The target is checked against numpy's at a stated tolerance (Cholesky vs
LAPACK's LU differ at rounding level times the condition number of the
regularised Gram matrix, up to 1e11 here: max-norm relative error
<= TARGET_K * eps * cond(G)); the rounded start must match the reference's exactly on
every golden instance without a continuous warm start (44 of them), and a
solve from it must reproduce the reference trajectory."""

import numpy as np
import pytest

from tests.golden_io import cfg_kwargs, load, named_A

pytestmark = pytest.mark.gpu

TARGET_K = 100.0


def _atol(G, ref_t):
    return max(1e-13, TARGET_K * np.finfo(float).eps * np.linalg.cond(G)) * np.max(np.abs(ref_t))


@pytest.fixture(scope="module")
def amvm():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    import paper_2508_13437_b200 as P

    return P


def _cases():
    out = []
    for nm in ("small_solves", "refresh_solves"):
        out += [(f"{nm}[{k}]", r, r["A"]) for k, r in enumerate(load(nm)) if "continuous_init" not in r]
    for nm in ("c1", "c1x"):
        r = load(f"solve_{nm}")[0]
        A = named_A(nm, r)
        if A is not None:
            out.append((nm, r, A))
    return out


def test_device_start_matches_reference_starts(amvm):
    from paper_2508_13437_b200.controller import _initial_solution_device

    P = amvm
    cases = _cases()
    assert len(cases) >= 40
    for name, rec, A in cases:
        inst = P.Instance(A, rec["b"], P.ValueSet(rec["levels"]))
        sol, target, flag = _initial_solution_device(inst, return_target=True)
        G = A.T @ A + 1e-8 * np.eye(A.shape[1])
        ref_t = np.linalg.solve(G, A.T @ rec["b"])
        assert flag == 0, name
        np.testing.assert_allclose(target, ref_t, rtol=0, atol=_atol(G, ref_t), err_msg=name)
        np.testing.assert_array_equal(sol.idx, rec["idx0"], err_msg=name)
        assert sol.objective == rec["obj0"], name


def test_solve_with_device_start_reproduces_c1(amvm):
    P = amvm
    rec = load("solve_c1")[0]
    A = named_A("c1", rec)
    if A is None:
        pytest.skip("C1 matrix not reproducible on this host")
    inst = P.Instance(A, rec["b"], P.ValueSet(rec["levels"]))
    rep = P.solve(inst, P.SolverConfig(**cfg_kwargs(rec)), device_warm_start=True)
    assert rep.initial_objective == rec["initial_objective"]
    assert rep.iterations == int(rec["iterations"])
    np.testing.assert_array_equal(rep.best.idx, rec["best_idx"])
    assert rep.best.objective == rec["best_objective"]


def test_device_start_falls_back_to_zeros(amvm):
    """An overflowing system (controller.py:146-153): the start is the
    rounded zero vector, with a warning."""
    P = amvm
    A = np.full((6, 3), 1e200)
    inst = P.Instance(A, np.ones(6), P.ValueSet([-1.0, 0.5, 2.0]))
    with pytest.warns(UserWarning, match="least-squares start"):
        sol = P.initial_solution(inst, device=True)
    np.testing.assert_array_equal(sol.idx, [1, 1, 1])


def test_device_start_larger_system(amvm):
    """n = 1200 (more than one substitution sweep per thread, many pivot
    launches) against numpy."""
    from paper_2508_13437_b200.controller import _initial_solution_device

    P = amvm
    rng = np.random.default_rng(11)
    A = rng.standard_normal((1500, 1200))
    lv = np.arange(-8, 8, dtype=float)
    b = A @ rng.uniform(-8, 7, 1200)
    inst = P.Instance(A, b, P.ValueSet(lv))
    sol, target, flag = _initial_solution_device(inst, return_target=True)
    G = A.T @ A + 1e-8 * np.eye(1200)
    ref_t = np.linalg.solve(G, A.T @ b)
    assert flag == 0
    np.testing.assert_allclose(target, ref_t, rtol=0, atol=_atol(G, ref_t))
    ref_idx = np.argmin(np.abs(ref_t[:, None] - lv[None, :]), axis=1)
    assert np.mean(sol.idx == ref_idx) == 1.0
