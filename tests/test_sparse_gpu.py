"""The sparse engine (amvm_solve_sparse: A only as CSC + CSR, no dense
copy) against the reference's own tomography runs and against the dense
engine: traces, best assignments and objectives bit for bit."""

import numpy as np
import pytest

from tests.golden_io import cfg_kwargs, load, stored_A

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tomo():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    from paper_2508_13437_b200 import _native, tomo

    _native.load_library()
    return tomo


def _csr(A):
    import torch

    rows, cols = np.nonzero(A)
    indptr = np.zeros(A.shape[0] + 1, dtype=np.int64)
    np.add.at(indptr, rows + 1, 1)
    indptr = np.cumsum(indptr)
    return (torch.from_numpy(indptr).cuda(), torch.from_numpy(cols.astype(np.int64)).cuda(),
            torch.from_numpy(A[rows, cols]).cuda())


def _check(o, rec, k=0):
    it = int(rec["iterations"])
    assert int(o["iterations"][k]) == it
    np.testing.assert_array_equal(o["trace_current_t"][k, :it].cpu().numpy(), rec["trace_current_t"])
    np.testing.assert_array_equal(o["trace_best_t"][k, :it].cpu().numpy(), rec["trace_best_t"])
    np.testing.assert_array_equal(o["trace_pair"][k, :it].cpu().numpy(), rec["trace_pair"])
    np.testing.assert_array_equal(o["trace_accepted"][k, :it].cpu().numpy(), rec["trace_accepted"])
    np.testing.assert_array_equal(o["best_idx"][k].cpu().numpy(), rec["best_idx"])
    assert float(o["best_objective"][k]) == rec["best_objective"]


@pytest.mark.parametrize("name", ["c3s", "c3m"])
def test_sparse_engine_matches_reference_tomography(tomo, name):
    from paper_2508_13437_b200 import SolverConfig

    rec = load(f"solve_{name}")[0]
    if name == "c3s":
        csr = _csr(stored_A(rec))
        m, n = (int(v) for v in rec["A_shape"])
    else:
        side, n_angles = (int(v) for v in rec["A_recipe"])
        csr = tomo.projection_csr_device(side, n_angles)
        m, n = side * n_angles, side * side
    sb = tomo.SparseSliceBatch(csr, m, n, rec["b"][None], rec["levels"], rec["idx0"][None])
    np.testing.assert_array_equal(sb.r0[0].cpu().numpy(), rec["r0"])  # numpy's dgemv order
    cfg = SolverConfig(**cfg_kwargs(rec))
    o = sb.solve(cfg, seeds=[cfg.seed], trace=True)
    sb.check_status()
    _check(o, rec)


def test_sparse_engine_equals_dense_engine_on_a_slice_batch(tomo):
    """Eight 24^2 x 16-angle slices, 12 iterations: sparse == dense, slice by slice."""
    import torch

    from paper_2508_13437_b200 import SolverConfig

    side, n_angles, lv = 24, 16, (0.0, 1.0, 2.0)
    fe = tomo.build_tomo_device(side, lv, n_angles, 0.2, seeds=tuple(range(8)),
                                phantom_kinds=("squares", "disk", "checker"), sirt_iters=30)
    m, n = fe["m"], fe["n"]
    cfg = SolverConfig(max_iters=12, destroy_rate=0.02)
    sp = tomo.SparseSliceBatch(fe["csr"], m, n, fe["B"], fe["levels"], fe["idx0"])
    A = torch.sparse_csr_tensor(*fe["csr"], size=(m, n), dtype=torch.float64).to_dense()
    de = tomo.SliceBatch(A, fe["B"].cpu().numpy(), fe["levels"], fe["idx0"].cpu().numpy())
    os_ = sp.solve(cfg, seeds=np.arange(8), trace=True)
    od = de.solve(cfg, seeds=np.arange(8), trace=True)
    sp.check_status()
    de.check_status()
    np.testing.assert_array_equal(sp.r0.cpu().numpy(), de._lb.r0.cpu().numpy())
    for key in ("iterations", "best_objective", "best_idx", "trace_current_t", "trace_best_t", "trace_pair",
                "trace_accepted"):
        np.testing.assert_array_equal(os_[key].cpu().numpy(), od[key].cpu().numpy(), err_msg=key)
    # reference-equivalent candidate counts: both engines against the CPU oracle
    from oracle import oracle as O

    Ah, Bh, I0 = A.cpu().numpy(), fe["B"].cpu().numpy(), fe["idx0"].cpu().numpy()
    L = np.asarray(lv)
    prm = O.make_params(n, max_iters=12, destroy_rate=0.02)
    R0 = sp.r0.cpu().numpy()
    ref = O.solve(Ah, Bh, np.tile(L, (8, 1)), I0, R0, np.abs(R0).max(axis=1), np.zeros(8), prm,
                  [O.pcg_from_seed(k) for k in range(8)])
    np.testing.assert_array_equal(od["best_objective"].cpu().numpy(), ref["best_objective"])
    np.testing.assert_array_equal(od["moves_scored"][:, 0].cpu().numpy(), ref["moves_scored"][:, 0])
    np.testing.assert_array_equal(os_["moves_scored"][:, 0].cpu().numpy(), ref["moves_scored"][:, 0])


def test_sparse_workspace_is_small(tomo):
    """Full-size C3 geometry: the sparse workspace is O(slots (m + n)), far
    below the dense engine's two m x n copies."""
    from paper_2508_13437_b200 import SolverConfig

    side, n_angles = 256, 180
    csr = tomo.projection_csr_device(side, n_angles)
    m, n = side * n_angles, side * side
    sb = tomo.SparseSliceBatch(csr, m, n, np.zeros((1, m)), (0.0, 1.0, 2.0), np.zeros((1, n), np.int32))
    ws = sb.workspace_bytes(SolverConfig(max_iters=2))
    assert 0 < ws < 2 * 8 * m * n / 8, ws


@pytest.mark.parametrize("side,n_angles,slices,iters", [(24, 16, 8, 12), (64, 45, 6, 4)])
def test_column_indexed_filter_equals_general_filter(tomo, side, n_angles, slices, iters):
    """The sparse engine's column-indexed candidate filter (filter rows'
    nonzeros indexed by column, pairs enumerated from the argmax row) keeps
    exactly the general staged-row filter's survivors: whole trajectories
    and candidate counts bitwise, with and without max_candidates truncation."""
    from paper_2508_13437_b200 import SolverConfig

    lv = (0.0, 1.0, 2.0)
    fe = tomo.build_tomo_device(side, lv, n_angles, 0.2, seeds=tuple(range(slices)),
                                phantom_kinds=("squares", "disk", "checker"), sirt_iters=20)
    m, n = fe["m"], fe["n"]
    for maxc in (5000, 64):
        cfg = SolverConfig(max_iters=iters, destroy_rate=0.02, max_candidates=maxc)
        outs = []
        for col in (True, False):
            sb = tomo.SparseSliceBatch(fe["csr"], m, n, fe["B"], fe["levels"], fe["idx0"], column_filter=col)
            assert (sb.max_row_nnz > 0) == col
            outs.append(sb.solve(cfg, seeds=np.arange(slices), trace=True))
            sb.check_status()
        for key in ("iterations", "best_objective", "best_idx", "trace_current_t", "trace_best_t", "trace_pair",
                    "trace_accepted", "moves_scored", "operator_uses"):
            np.testing.assert_array_equal(outs[0][key].cpu().numpy(), outs[1][key].cpu().numpy(),
                                          err_msg=f"{key} (max_candidates={maxc})")


@pytest.mark.parametrize("side,n_angles", [(16, 48), (32, 32)])
def test_column_indexed_filter_overflow_path(tomo, monkeypatch, side, n_angles):
    """More filter survivors than the candidate buffer (AMVM_SPARSE_CAP
    shrinks it): the column-indexed filter finds the max_candidates cut by
    counting passes and a per-i histogram and keeps exactly the general
    filter's truncated list."""
    from paper_2508_13437_b200 import SolverConfig

    lv = (0.0, 1.0, 2.0)
    fe = tomo.build_tomo_device(side, lv, n_angles, 0.2, seeds=tuple(range(20)),
                                phantom_kinds=("squares", "disk", "checker"), sirt_iters=20)
    m, n = fe["m"], fe["n"]
    cfg = SolverConfig(max_iters=6, destroy_rate=0.02, max_candidates=16)
    monkeypatch.setenv("AMVM_SPARSE_CAP", "1024")
    outs = []
    for col in (True, False):
        sb = tomo.SparseSliceBatch(fe["csr"], m, n, fe["B"], fe["levels"], fe["idx0"], column_filter=col)
        outs.append(sb.solve(cfg, seeds=np.arange(20), trace=True))
        sb.check_status()
    assert int(outs[0]["phase_cycles"][:, 9].sum()) > 0  # candidates were found
    for key in ("iterations", "best_objective", "best_idx", "trace_current_t", "trace_best_t", "trace_pair",
                "trace_accepted", "moves_scored"):
        np.testing.assert_array_equal(outs[0][key].cpu().numpy(), outs[1][key].cpu().numpy(), err_msg=key)


@pytest.mark.parametrize("seed", [0, 1, 2])
def test_solve_routes_general_sparse_A_bitwise(tomo, monkeypatch, seed):
    """solve() on a general sparse A (mixed signs, explicit structure unlike a
    projector, 1.6M entries at ~2 % density) runs the sparse engine; its
    report equals the dense engine's (AMVM_SPARSE_ROUTE=0) bit for bit."""
    import paper_2508_13437_b200 as P

    rng = np.random.default_rng(100 + seed)
    m, n = 1536, 1024
    A = np.where(rng.random((m, n)) < 0.02, rng.standard_normal((m, n)), 0.0)
    x = rng.integers(0, 5, n).astype(float) - 2.0
    b = A @ x + rng.uniform(-0.5, 0.5, m)
    inst = P.Instance(A, b, P.ValueSet(np.array([-2.0, -1.0, 0.0, 1.0, 2.0])))
    cfg = P.SolverConfig(max_iters=25, seed=seed, destroy_rate=0.02)
    reps = []
    for route in ("1", "0"):
        monkeypatch.setenv("AMVM_SPARSE_ROUTE", route)
        reps.append(P.solve(P.Instance(A, b, inst.values), cfg))
    sp, de = reps
    assert sp.best.objective == de.best.objective
    np.testing.assert_array_equal(sp.best.idx, de.best.idx)
    assert [(e.current_t, e.best_t, e.op_pair, e.accepted) for e in sp.trace] == \
        [(e.current_t, e.best_t, e.op_pair, e.accepted) for e in de.trace]
