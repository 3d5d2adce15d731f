"""GPU parity: the CUDA path (through the C-ABI) against the reference goldens
and the CPU oracle.  Bit-exact everywhere except impact scores (exp ulp,
tolerance below).  Run on a B200: ``pytest -m gpu``.
"""

import numpy as np
import pytest

from tests.golden_io import cfg_kwargs, load, named_A, stored_A

pytestmark = pytest.mark.gpu

IMPACT_RTOL = 1e-13  # CUDA exp vs numpy SIMD exp, <= 1 ulp per term


@pytest.fixture(scope="module")
def amvm():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    import paper_2508_13437_b200 as P
    from paper_2508_13437_b200 import _native

    _native.load_library()
    return P


def _inst(P, A, rec):
    return P.Instance(A, rec["b"], P.ValueSet(rec["levels"]),
                      continuous_init=rec.get("continuous_init"))


def _check_report(rep, rec):
    it = int(rec["iterations"])
    assert rep.iterations == it
    pairs = np.array([["random+random", "random+greedy", "worst+random", "worst+greedy"].index(e.op_pair)
                      for e in rep.trace], dtype=np.uint8)
    np.testing.assert_array_equal(pairs, rec["trace_pair"])
    np.testing.assert_array_equal(np.array([e.accepted for e in rep.trace], np.uint8), rec["trace_accepted"])
    np.testing.assert_array_equal(np.array([e.current_t for e in rep.trace]), rec["trace_current_t"])
    np.testing.assert_array_equal(np.array([e.best_t for e in rep.trace]), rec["trace_best_t"])
    np.testing.assert_array_equal(rep.best.idx, rec["best_idx"])
    np.testing.assert_array_equal(rep.best.residual, rec["best_residual"])
    assert rep.best.objective == rec["best_objective"]
    assert rep.best.updates_since_refresh == int(rec["best_updates"])
    assert [rep.operator_uses[k] for k in ("random+random", "random+greedy", "worst+random",
                                           "worst+greedy")] == list(rec["operator_uses"])


def _solve_from_golden(P, A, rec):
    inst = _inst(P, A, rec)
    start = P.Solution(rec["idx0"], rec["r0"], rec["obj0"], 0)
    from paper_2508_13437_b200.controller import solve_from
    return solve_from(inst, start, P.SolverConfig(**cfg_kwargs(rec)))


@pytest.mark.parametrize("k", range(48))
def test_small_solves_match_reference(amvm, k):
    rec = load("small_solves")[k]
    _check_report(_solve_from_golden(amvm, rec["A"], rec), rec)


@pytest.mark.parametrize("k", range(3))
def test_refresh_solves_match_reference(amvm, k):
    rec = load("refresh_solves")[k]
    _check_report(_solve_from_golden(amvm, rec["A"], rec), rec)


@pytest.mark.parametrize("name", ["c1", "c1x", "c2", "c4row", "c5row"])
def test_named_solves_match_reference(amvm, name):
    rec = load(f"solve_{name}")[0]
    A = named_A(name, rec)
    if A is None:
        pytest.skip("host numpy does not regenerate the reference matrix bit-exactly")
    _check_report(_solve_from_golden(amvm, A, rec), rec)


def test_tomography_scaled_matches_reference(amvm):
    """C3 family at 64^2 x 45 angles: many filter survivors (adaptive buffer)."""
    rec = load("solve_c3s")[0]
    _check_report(_solve_from_golden(amvm, stored_A(rec), rec), rec)


def test_public_solve_matches_oracle(amvm, oracle):
    """dmmv.solve-equivalent end to end (host initial_solution + device loop)."""
    rng = np.random.default_rng(7)
    for t in range(6):
        m, n = int(rng.integers(8, 90)), int(rng.integers(4, 40))
        A = rng.uniform(-1, 1, (m, n))
        b = rng.uniform(-1, 1, m)
        lv = np.sort(rng.uniform(-1, 1, 6))
        inst = amvm.Instance(A, b, amvm.ValueSet(lv))
        cfg = amvm.SolverConfig(max_iters=120, seed=t, destroy_rate=0.1)
        rep = amvm.solve(inst, cfg)
        s0 = amvm.initial_solution(inst)
        prm = oracle.make_params(n, max_iters=120, destroy_rate=0.1)
        out = oracle.solve(A, b, lv, s0.idx, s0.residual, s0.objective, 0, prm, oracle.pcg_from_seed(t))
        assert rep.iterations == int(out["iterations"][0])
        np.testing.assert_array_equal(rep.best.idx, out["best_idx"][0])
        np.testing.assert_array_equal(rep.best.residual, out["best_residual"][0])
        np.testing.assert_array_equal([e.current_t for e in rep.trace],
                                      out["trace_current_t"][0, :rep.iterations])


def test_time_limit_zero_runs_no_iterations(amvm):
    inst = amvm.Instance(np.eye(3), np.ones(3) * 0.3, amvm.ValueSet([0.0, 1.0]))
    rep = amvm.solve(inst, amvm.SolverConfig(time_limit=0.0))
    assert rep.iterations == 0 and rep.trace == []


# ------------------------------------------------------------- components
@pytest.fixture(scope="module")
def components():
    return load("components")


def _sol(P, rec, prefix):
    return P.Solution(rec[prefix + "idx"], rec[prefix + "residual"], rec[prefix + "objective"],
                      rec[prefix + "updates"])


def _same(sol, rec, prefix):
    np.testing.assert_array_equal(sol.idx, rec[prefix + "idx"])
    np.testing.assert_array_equal(sol.residual, rec[prefix + "residual"])
    assert sol.objective == rec[prefix + "objective"]
    assert sol.updates_since_refresh == rec[prefix + "updates"]


def _fc(P, rec):
    mc = int(rec["max_candidates"])
    return P.FilterConfig(k_eps=int(rec["k_eps"]), max_candidates=None if mc < 0 else mc)


def test_one_opt_local_search_components(amvm, components):
    for rec in components:
        inst = _inst(amvm, rec["A"], rec)
        _same(amvm.one_opt(inst, _sol(amvm, rec, "in_")), rec, "oneopt_")
        _same(amvm.local_search(inst, _sol(amvm, rec, "in_"), _fc(amvm, rec)), rec, "ls_")


def test_find_candidates_best_swap_components(amvm, components):
    for rec in components:
        if "fc_i" not in rec:
            continue
        inst = _inst(amvm, rec["A"], rec)
        sol = _sol(amvm, rec, "in_")
        cands = amvm.find_candidates(inst, sol, _fc(amvm, rec))
        assert [c.i for c in cands] == list(rec["fc_i"])
        assert [c.j for c in cands] == list(rec["fc_j"])
        assert [c.delta for c in cands] == list(rec["fc_delta"])
        bs = amvm.best_swap(inst, sol, _fc(amvm, rec))
        if rec["bs"][0] < 0:
            assert bs is None
        else:
            assert (bs.i, bs.j, bs.delta, bs.predicted_t) == (int(rec["bs"][0]), int(rec["bs"][1]),
                                                              rec["bs"][2], rec["bs"][3])


def test_impact_scores_components(amvm, components):
    for rec in components:
        if "impact" not in rec:
            continue
        inst = _inst(amvm, rec["A"], rec)
        d = amvm.impact_scores(inst, _sol(amvm, rec, "in_"), float(rec["alpha"])).d
        np.testing.assert_allclose(d, rec["impact"], rtol=IMPACT_RTOL, atol=0)


def test_destroy_repair_components(amvm, components):
    for rec in components:
        inst = _inst(amvm, rec["A"], rec)
        sol = _sol(amvm, rec, "in_")
        r = int(rec["r"])
        seed = int(rec["seed"])
        ds = amvm.random_destroy(sol, r, np.random.default_rng(seed))
        np.testing.assert_array_equal(ds.removed, rec["rd_removed"])
        ds = amvm.worst_remove_destroy(inst, sol, r, float(rec["alpha"]), np.random.default_rng(seed))
        np.testing.assert_array_equal(ds.removed, rec["wd_removed"])
        if "saved" not in rec:
            continue
        np.testing.assert_array_equal(ds.saved_idx, rec["saved"])
        rr = amvm.random_repair(inst, _sol(amvm, rec, "in_"), ds, np.random.default_rng(seed + 1))
        _same(rr, rec, "rr_")
        gr = amvm.greedy_repair(inst, _sol(amvm, rec, "in_"), ds)
        _same(gr, rec, "gr_")


def test_rng_stream_advances_like_numpy(amvm):
    """The device consumes exactly the draws numpy would (state written back)."""
    rng_dev = np.random.default_rng(5)
    rng_ref = np.random.default_rng(5)
    sol = amvm.Solution(np.zeros(40, dtype=np.intp), np.zeros(1), 0.0)
    amvm.random_destroy(sol, 7, rng_dev)
    rng_ref.choice(40, size=7, replace=False)
    assert rng_dev.bit_generator.state == rng_ref.bit_generator.state


def test_compute_residual_matches_host_blas_order(amvm, oracle):
    """amvm_compute_residual reproduces numpy's single-threaded A @ x - b."""
    import ctypes as C

    import torch
    from threadpoolctl import threadpool_limits

    from paper_2508_13437_b200 import _native as N

    rng = np.random.default_rng(3)
    for (m, n, count) in [(64, 100, 5), (1024, 256, 9), (2048, 4099, 3), (7, 13, 4), (1, 37, 3), (6, 5, 2)]:
        A = rng.standard_normal((m, n))
        lv = np.sort(rng.uniform(-2, 2, (count, 16)), axis=1)
        idx = rng.integers(0, 16, (count, n)).astype(np.int32)
        B = rng.standard_normal((count, m))
        with threadpool_limits(1):
            want = np.stack([A @ lv[k][idx[k]] - B[k] for k in range(count)])
        dev = torch.device("cuda")
        At = torch.from_numpy(np.ascontiguousarray(A.T)).to(dev)
        Bt, Lt = torch.from_numpy(B).to(dev), torch.from_numpy(lv).to(dev)
        It = torch.from_numpy(idx).to(dev)
        R = torch.empty((count, m), dtype=torch.float64, device=dev)
        O = torch.empty(count, dtype=torch.float64, device=dev)
        Cn = torch.empty(count, dtype=torch.int32, device=dev)
        prob = N.Problem(m, n, 16, count, At.data_ptr(), Bt.data_ptr(), Lt.data_ptr())
        sol = N.SolutionPtrs(It.data_ptr(), R.data_ptr(), O.data_ptr(), Cn.data_ptr())
        N.check(N.load_library().amvm_compute_residual(C.byref(prob), C.byref(sol), N.stream_handle()), "res")
        got = R.cpu().numpy()
        np.testing.assert_array_equal(got, want)
        np.testing.assert_array_equal(O.cpu().numpy(), np.abs(want).max(axis=1))


# ------------------------------------------------------- shared-X batch (PTQ)
def test_ptq_prepare_and_batch_solve_match_host(amvm, oracle):
    """solve_layer == per-row reference semantics (host numpy start + oracle)."""
    from threadpoolctl import threadpool_limits

    from paper_2508_13437_b200 import ptq

    rng = np.random.default_rng(11)
    X = rng.standard_normal((136, 60))
    W = rng.standard_normal((37, 60)) * 0.02
    W[5] = 0.01  # collapsed range -> widened grid (builders.py:367-369)
    cfg = amvm.SolverConfig(max_iters=25, destroy_rate=0.05)
    rep = ptq.solve_layer(X, W, bits=4, cfg=cfg, trace=True)
    prm = oracle.make_params(60, max_iters=25, destroy_rate=0.05)
    for r in range(W.shape[0]):
        w = W[r]
        lo, hi = float(w.min()), float(w.max())
        if hi - lo < 1e-12:
            lo, hi = lo - 0.5, hi + 0.5
        lv = np.linspace(lo, hi, 16)
        np.testing.assert_array_equal(rep.levels[r], lv)
        with threadpool_limits(1):
            b = X @ w
            idx0 = np.argmin(np.abs(w[:, None] - lv[None, :]), axis=1)
            r0 = X @ lv[idx0] - b
        out = oracle.solve(X, b, lv, idx0, r0, float(np.max(np.abs(r0))), 0, prm, oracle.pcg_from_seed(r))
        assert rep.initial_objective[r] == float(np.max(np.abs(r0)))
        assert int(rep.iterations[r]) == int(out["iterations"][0])
        np.testing.assert_array_equal(rep.codes[r], out["best_idx"][0])
        assert rep.objective[r] == out["best_objective"][0]
        it = int(rep.iterations[r])
        np.testing.assert_array_equal(rep.seconds["trace"]["trace_current_t"][r, :it],
                                      out["trace_current_t"][0, :it])


def test_ptq_layer_row_matches_reference_golden(amvm):
    """Row 0 of the C4-shaped layer through the batch pipeline == dmmv.solve."""
    from paper_2508_13437_b200 import ptq
    from tests.golden import recipes
    from tests.golden_io import sha

    rec = load("solve_c4row")[0]
    X, W = recipes.ptq_layer(768, 3072)
    if sha(X) != rec["A_sha"]:
        pytest.skip("host numpy does not regenerate X bit-exactly")
    cfg = amvm.SolverConfig(**cfg_kwargs(rec))
    rep = ptq.solve_layer(X, W[:3], bits=4, cfg=cfg, trace=True)
    assert rep.initial_objective[0] == rec["initial_objective"]
    np.testing.assert_array_equal(rep.codes[0], rec["best_idx"])
    assert rep.objective[0] == rec["best_objective"]
    it = int(rec["iterations"])
    np.testing.assert_array_equal(rep.seconds["trace"]["trace_current_t"][0, :it], rec["trace_current_t"])


def _batch_vs_oracle(amvm, oracle, A, B, lv, idx0, cfg_kw, check=None):
    """One amvm_solve over a batch sharing A (start = idx0), every checked
    instance compared with the oracle's solve from the same start and seed."""
    import torch

    from paper_2508_13437_b200 import _native as N
    from paper_2508_13437_b200.controller import make_params

    count, n = idx0.shape
    m = A.shape[0]
    nlev = lv.size
    R0 = np.stack([A @ lv[idx0[k]] - B[k] for k in range(count)])
    obj0 = np.abs(R0).max(axis=1)
    cfg = amvm.SolverConfig(**cfg_kw)
    prm = make_params(cfg, n)
    dev = torch.device("cuda")
    t = lambda a, dt: torch.from_numpy(np.ascontiguousarray(a, dtype=dt)).to(dev)  # noqa: E731
    At, Bt, Lt = t(A.T, np.float64), t(B, np.float64), t(np.tile(lv, (count, 1)), np.float64)
    I0, R0t, O0, C0 = t(idx0, np.int32), t(R0, np.float64), t(obj0, np.float64), t(np.zeros(count), np.int32)
    rngs = t(N.seed_states(np.arange(count)).view(np.uint8), np.uint8)
    T = cfg.max_iters
    bi, br = torch.empty((count, n), dtype=torch.int32, device=dev), torch.empty((count, m), dtype=torch.float64, device=dev)
    bo, bc = torch.empty(count, dtype=torch.float64, device=dev), torch.empty(count, dtype=torch.int32, device=dev)
    io, it = torch.empty(count, dtype=torch.float64, device=dev), torch.empty(count, dtype=torch.int32, device=dev)
    ou = torch.empty((count, 4), dtype=torch.int64, device=dev)
    tc = torch.empty((count, T), dtype=torch.float64, device=dev)
    tb = torch.empty((count, T), dtype=torch.float64, device=dev)
    tp = torch.empty((count, T), dtype=torch.uint8, device=dev)
    ta = torch.empty((count, T), dtype=torch.uint8, device=dev)
    res = N.ResultPtrs(N.SolutionPtrs(bi.data_ptr(), br.data_ptr(), bo.data_ptr(), bc.data_ptr()),
                       io.data_ptr(), it.data_ptr(), ou.data_ptr(), tc.data_ptr(), tb.data_ptr(), tp.data_ptr(),
                       ta.data_ptr(), None, None)
    prob = N.Problem(m, n, nlev, count, At.data_ptr(), Bt.data_ptr(), Lt.data_ptr())
    start = N.SolutionPtrs(I0.data_ptr(), R0t.data_ptr(), O0.data_ptr(), C0.data_ptr())
    lib = N.load_library()
    nb = lib.amvm_workspace_bytes(N.C.byref(prob), N.C.byref(prm))
    ws = torch.empty(nb, dtype=torch.uint8, device=dev)
    N.check(lib.amvm_solve(N.C.byref(prob), N.C.byref(prm), N.C.byref(start), N.ptr(rngs), N.C.byref(res),
                           N.ptr(ws), N.C.c_size_t(nb), N.stream_handle()), "amvm_solve")
    N.check(lib.amvm_status(N.ptr(ws), N.stream_handle()), "amvm_solve")
    okw = {k: v for k, v in cfg_kw.items() if k != "seed"}
    oprm = oracle.make_params(n, **okw)
    host = {k: v.cpu().numpy() for k, v in dict(it=it, tc=tc, tb=tb, tp=tp, ta=ta, bi=bi, br=br, bo=bo, ou=ou).items()}
    for k in (range(count) if check is None else check):
        out = oracle.solve(A, B[k], lv, idx0[k], R0[k], obj0[k], 0, oprm, oracle.pcg_from_seed(k))
        n_it = int(out["iterations"][0])
        assert int(host["it"][k]) == n_it, k
        np.testing.assert_array_equal(host["tc"][k, :n_it], out["trace_current_t"][0, :n_it])
        np.testing.assert_array_equal(host["tb"][k, :n_it], out["trace_best_t"][0, :n_it])
        np.testing.assert_array_equal(host["tp"][k, :n_it], out["trace_pair"][0, :n_it])
        np.testing.assert_array_equal(host["ta"][k, :n_it], out["trace_accepted"][0, :n_it])
        np.testing.assert_array_equal(host["bi"][k], out["best_idx"][0])
        np.testing.assert_array_equal(host["br"][k], out["best_residual"][0])
        assert host["bo"][k] == out["best_objective"][0]
        np.testing.assert_array_equal(host["ou"][k], out["operator_uses"][0])
    return host


def test_swap_filter_overflow_path_matches_oracle(amvm, oracle):
    """More filter survivors than a batch slot's buffer (17 instances => the
    batch cap 1024; n=80 with k_eps=1 keeps ~1500 pairs): the exact overflow
    path (counting passes + cut) must still return the reference's first
    max_candidates in (-delta, i, j) order — checked via whole trajectories."""
    rng = np.random.default_rng(21)
    count, m, n, nlev = 17, 24, 80, 6
    A = rng.uniform(-1, 1, (m, n))
    lv = np.sort(rng.uniform(-1, 1, nlev))
    B = rng.uniform(-1, 1, (count, m))
    idx0 = rng.integers(0, nlev, (count, n)).astype(np.int32)
    _batch_vs_oracle(amvm, oracle, A, B, lv, idx0,
                     dict(max_iters=6, k_eps=1, max_candidates=3, destroy_rate=0.05))


def test_chunked_batch_migrates_bitwise(amvm, oracle):
    """More instances than resident CTAs: the solve runs one ALNS iteration
    per task and instances migrate between CTAs (parked state in the
    workspace).  Trajectories must equal the oracle's; planted instances
    reach objective 0 mid-run and must stop exactly there."""
    rng = np.random.default_rng(33)
    count, m, n, nlev = 700, 18, 14, 5
    A = rng.integers(-4, 5, (m, n)).astype(float)
    lv = np.arange(nlev, dtype=float) - 2.0
    B = rng.integers(-6, 7, (count, m)).astype(float)
    xs = rng.integers(0, nlev, (count, n))
    planted = np.arange(count) % 5 == 0
    B[planted] = np.stack([A @ lv[xs[k]] for k in np.nonzero(planted)[0]])
    idx0 = rng.integers(0, nlev, (count, n)).astype(np.int32)
    host = _batch_vs_oracle(amvm, oracle, A, B, lv, idx0, dict(max_iters=9, destroy_rate=0.2),
                            check=range(0, count, 3))
    assert (host["it"] < 9).any() and (host["it"] == 9).any()  # both early stops and full runs
