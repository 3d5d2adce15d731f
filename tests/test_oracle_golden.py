"""Pin the CPU oracle against the reference's own outputs (CPU-only).

The goldens in tests/golden/ were produced by running the unmodified
reference (make_golden.py).  The oracle must reproduce them bit for bit —
trajectories, residuals, candidate lists — except impact scores, whose exp()
may differ by an ulp from numpy's SIMD exp (tolerance stated below).
"""

import numpy as np
import pytest

from tests.golden_io import cfg_kwargs, load, named_A, stored_A

IMPACT_RTOL = 1e-13  # libm exp vs numpy SIMD exp (<= 1 ulp per term)


def _params(O, n, cfg):
    kw = dict(cfg)
    kw.pop("seed")
    return O.make_params(n, **kw)


def _check_solve(O, A, rec):
    cfg = cfg_kwargs(rec)
    prm = _params(O, A.shape[1], cfg)
    out = O.solve(A, rec["b"], rec["levels"], rec["idx0"], rec["r0"], rec["obj0"], 0, prm,
                  O.pcg_from_seed(cfg["seed"]))
    it = int(rec["iterations"])
    assert int(out["iterations"][0]) == it
    np.testing.assert_array_equal(out["trace_pair"][0, :it], rec["trace_pair"])
    np.testing.assert_array_equal(out["trace_accepted"][0, :it], rec["trace_accepted"])
    np.testing.assert_array_equal(out["trace_current_t"][0, :it], rec["trace_current_t"])
    np.testing.assert_array_equal(out["trace_best_t"][0, :it], rec["trace_best_t"])
    np.testing.assert_array_equal(out["best_idx"][0], rec["best_idx"])
    np.testing.assert_array_equal(out["best_residual"][0], rec["best_residual"])
    assert out["best_objective"][0] == rec["best_objective"]
    assert int(out["best_updates"][0]) == int(rec["best_updates"])
    np.testing.assert_array_equal(out["operator_uses"][0], rec["operator_uses"])
    assert out["initial_objective"][0] == rec["initial_objective"]


@pytest.mark.parametrize("k", range(48))
def test_small_solves_bitwise(oracle, k):
    rec = load("small_solves")[k]
    _check_solve(oracle, rec["A"], rec)


@pytest.mark.parametrize("k", range(3))
def test_refresh_solves_bitwise(oracle, k):
    """Lineages crossing REFRESH_PERIOD: pins the dgemv-order refresh."""
    rec = load("refresh_solves")[k]
    _check_solve(oracle, rec["A"], rec)


@pytest.mark.parametrize("name", ["c1", "c1x", "c2", "c4row", "c5row"])
def test_named_solves_bitwise(oracle, name):
    rec = load(f"solve_{name}")[0]
    A = named_A(name, rec)
    if A is None:
        pytest.skip("host numpy does not regenerate the reference matrix bit-exactly")
    _check_solve(oracle, A, rec)


def test_tomography_scaled_bitwise(oracle):
    """C3 family (64^2 phantom, 45 angles, 3 grey levels; A built by the
    reference's own projector): 152K swap-filter survivors at the start."""
    rec = load("solve_c3s")[0]
    _check_solve(oracle, stored_A(rec), rec)


def _sol(rec, prefix):
    return (rec[prefix + "idx"], rec[prefix + "residual"], rec[prefix + "objective"],
            rec[prefix + "updates"])


def _assert_sol(got, rec, prefix):
    idx, r, obj, cnt = got
    np.testing.assert_array_equal(idx, rec[prefix + "idx"])
    np.testing.assert_array_equal(r, rec[prefix + "residual"])
    assert obj == rec[prefix + "objective"]
    assert cnt == rec[prefix + "updates"]


@pytest.fixture(scope="module")
def components():
    return load("components")


def _cprm(O, rec, **kw):
    mc = int(rec["max_candidates"])
    return O.make_params(rec["A"].shape[1], k_eps=int(rec["k_eps"]),
                         max_candidates=None if mc < 0 else mc, alpha=float(rec["alpha"]),
                         r=int(rec["r"]), **kw)


def test_one_opt_and_local_search(oracle, components):
    for rec in components:
        prm = _cprm(oracle, rec)
        got = oracle.one_opt(rec["A"], rec["b"], rec["levels"], *_sol(rec, "in_"), prm)
        _assert_sol(got, rec, "oneopt_")
        got = oracle.local_search(rec["A"], rec["b"], rec["levels"], *_sol(rec, "in_"), prm)
        _assert_sol(got, rec, "ls_")


def test_find_candidates_and_best_swap(oracle, components):
    seen = 0
    for rec in components:
        if "fc_i" not in rec:
            continue
        seen += 1
        prm = _cprm(oracle, rec)
        idx, r, obj, _ = _sol(rec, "in_")
        ci, cj, cd = oracle.find_candidates(rec["A"], rec["b"], rec["levels"], idx, r, obj, prm)
        np.testing.assert_array_equal(ci, rec["fc_i"])
        np.testing.assert_array_equal(cj, rec["fc_j"])
        np.testing.assert_array_equal(cd, rec["fc_delta"])
        bs = oracle.best_swap(rec["A"], rec["b"], rec["levels"], idx, r, obj, prm)
        want = rec["bs"]
        if want[0] < 0:
            assert bs is None
        else:
            assert bs == (int(want[0]), int(want[1]), float(want[2]), float(want[3]))
    assert seen > 40


def test_impact_scores(oracle, components):
    for rec in components:
        if "impact" not in rec:
            continue
        prm = _cprm(oracle, rec)
        idx, r, obj, _ = _sol(rec, "in_")
        d = oracle.impact_scores(rec["A"], rec["b"], rec["levels"], idx, r, obj, prm)
        np.testing.assert_allclose(d, rec["impact"], rtol=IMPACT_RTOL, atol=0)


def test_destroy_and_repair(oracle, components):
    for rec in components:
        prm = _cprm(oracle, rec)
        idx, r, obj, cnt = _sol(rec, "in_")
        seed = int(rec["seed"])
        got, _ = oracle.destroy(0, rec["A"], rec["b"], rec["levels"], idx, r, obj, prm,
                                oracle.pcg_from_seed(seed))
        np.testing.assert_array_equal(got, rec["rd_removed"])
        got, _ = oracle.destroy(1, rec["A"], rec["b"], rec["levels"], idx, r, obj, prm,
                                oracle.pcg_from_seed(seed))
        np.testing.assert_array_equal(got, rec["wd_removed"])
        if "saved" not in rec:
            continue
        sol, _ = oracle.repair(0, rec["A"], rec["b"], rec["levels"], idx, r, obj, cnt, prm,
                               oracle.pcg_from_seed(seed + 1), rec["wd_removed"], rec["saved"])
        _assert_sol(sol, rec, "rr_")
        sol, _ = oracle.repair(1, rec["A"], rec["b"], rec["levels"], idx, r, obj, cnt, prm,
                               oracle.pcg_from_seed(seed + 1), rec["wd_removed"], rec["saved"])
        _assert_sol(sol, rec, "gr_")


def test_rng_primitives_match_numpy(oracle):
    """PCG64 + Generator draws the path consumes (SURVEY.md §8c RNG contract)."""
    import ctypes as C
    lib = oracle.lib()
    for seed in range(12):
        g = np.random.default_rng(seed)
        st = oracle.pcg_from_seed(seed)
        for t in range(60):
            op = (seed + t) % 4
            if op == 0:
                assert lib.orc_random(C.byref(st)) == g.random()
            elif op == 1:
                assert lib.orc_bounded(C.byref(st), 1) == int(g.integers(2))
            elif op == 2:
                n, r = 50 + 37 * t, 1 + t % 9
                out = np.zeros(r, np.int64)
                lib.orc_choice_noreplace(C.byref(st), n, r, out.ctypes.data)
                np.testing.assert_array_equal(out, g.choice(n, size=r, replace=False))
            else:
                p = np.random.default_rng(t).random(1 + t % 7)
                p /= p.sum()
                assert lib.orc_choice_p(C.byref(st), p.ctypes.data, p.size) == int(g.choice(p.size, p=p))


def test_pairwise_sum_matches_numpy(oracle):
    rng = np.random.default_rng(0)
    for n in [0, 1, 5, 7, 8, 9, 127, 128, 129, 300, 1000, 4096, 8193]:
        a = rng.random(n) * 10.0 ** rng.integers(-3, 3, n)
        assert oracle.pairwise_sum(a) == float(a.sum())


def test_norm_matches_host_blas(oracle):
    threadpoolctl = pytest.importorskip("threadpoolctl")
    archs = {i.get("architecture") for i in threadpoolctl.threadpool_info()}
    if not archs & {"SkylakeX", "Cooperlake", "SapphireRapids"}:
        pytest.skip(f"host BLAS kernel {archs} is not the one the goldens were made with")
    rng = np.random.default_rng(1)
    for n in list(range(1, 70)) + [1000, 1024, 2047, 8192]:
        x = rng.standard_normal(n)
        assert oracle.norm(x) == float(np.linalg.norm(x))
