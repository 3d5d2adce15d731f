"""Device projector (amvm_projector_*): the CSR built on the GPU must equal
the host restatement (tomo.projection_csr, itself sha-pinned to the
reference's parallel_beam_matrix) bit for bit — indptr, pixel order and
every length — including axis-parallel rays (angle 0 and pi/2 with an even
angle count), odd sides, and the full C3 size (256^2 x 180)."""

import numpy as np
import pytest

from tests.golden_io import load, sha, stored_A

pytestmark = pytest.mark.gpu


@pytest.fixture(scope="module")
def tomo():
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    from paper_2508_13437_b200 import tomo as T

    return T


@pytest.mark.parametrize("side,n_angles", [(16, 9), (7, 4), (33, 7), (64, 45), (128, 64), (256, 180)])
def test_device_projector_matches_host(tomo, side, n_angles):
    ip, ix, v = tomo.projection_csr(side, n_angles)
    dp, dx, dv = tomo.projection_csr_device(side, n_angles)
    np.testing.assert_array_equal(dp.cpu().numpy(), ip)
    np.testing.assert_array_equal(dx.cpu().numpy(), ix)
    assert np.array_equal(dv.cpu().numpy().view(np.uint64), v.view(np.uint64))


def test_device_projector_matches_reference_matrices(tomo):
    import torch

    rec = load("solve_c3s")[0]
    dp, dx, dv = tomo.projection_csr_device(64, 45)
    A = torch.sparse_csr_tensor(dp, dx, dv, size=(64 * 45, 64 * 64)).to_dense().cpu().numpy()
    assert np.array_equal(A.view(np.uint64), stored_A(rec).view(np.uint64))
    rec = load("solve_c3m")[0]
    side, n_angles = (int(v) for v in rec["A_recipe"])
    dp, dx, dv = tomo.projection_csr_device(side, n_angles)
    A = torch.sparse_csr_tensor(dp, dx, dv, size=(side * n_angles, side * side)).to_dense().cpu().numpy()
    assert sha(A) == str(rec["A_sha"])


@pytest.mark.parametrize("name", ["c3s", "c3m"])
def test_device_front_end_matches_reference_build_tomo(tomo, name):
    """build_tomo on the GPU vs the reference's own instances
    (make_golden.py: TomoSpec squares, levels 0/1/2, eta = 5% of the max row
    sum, sirt_iters 100, seed 0): projections b bit for bit, the SIRT warm
    start within SIRT_ATOL (sparse vs dense BLAS summation order), and its
    rounded start equal to the reference's initial solution."""
    SIRT_ATOL = 1e-9
    rec = load(f"solve_{name}")[0]
    if name == "c3s":
        side, n_angles = 64, 45
        A = stored_A(rec)
    else:
        side, n_angles = (int(v) for v in rec["A_recipe"])
        A = tomo.projection_matrix(side, n_angles)
    eta = 0.05 * float(A.sum(axis=1).max())
    del A
    out = tomo.build_tomo_device(side, (0.0, 1.0, 2.0), n_angles, eta, seeds=(0,), phantom_kinds=("squares",),
                                 sirt_iters=100)
    b = out["B"][0].cpu().numpy()
    assert np.array_equal(b.view(np.uint64), rec["b"].view(np.uint64))
    if "continuous_init" in rec:
        np.testing.assert_allclose(out["warm"][0].cpu().numpy(), rec["continuous_init"], rtol=0, atol=SIRT_ATOL)
    np.testing.assert_array_equal(out["idx0"][0].cpu().numpy(), rec["idx0"])


def test_sirt_validation(tomo):
    import torch

    csr = (torch.tensor([0, 1], device="cuda"), torch.tensor([0], device="cuda"),
           torch.tensor([-1.0], device="cuda", dtype=torch.float64))
    with pytest.raises(ValueError, match="non-negative"):
        tomo.sirt_device(csr, 1, 1, torch.ones((1, 1), device="cuda", dtype=torch.float64), 3)


def test_solve_slices_matches_oracle_per_slice(tomo):
    """tomo.solve_slices (the per-rank unit of the slice sharding): each
    slice's report equals the oracle's solve of that slice from the same
    device-built inputs (projector, projections, SIRT start; seed = slice id)."""
    import torch

    from oracle import oracle as O
    from paper_2508_13437_b200 import SolverConfig

    side, n_angles, lv = 16, 12, (0.0, 1.0, 2.0)
    slices = np.array([3, 4, 7])
    kinds = ("squares", "disk", "checker")
    cfg = SolverConfig(max_iters=8, destroy_rate=0.05)
    rep = tomo.solve_slices(side, lv, n_angles, 0.1, slices, kinds, cfg=cfg, sirt_iters=20)
    fe = tomo.build_tomo_device(side, lv, n_angles, 0.1, seeds=tuple(int(k) for k in slices),
                                phantom_kinds=tuple(kinds[k % 3] for k in slices), sirt_iters=20)
    m, n = fe["m"], fe["n"]
    A = torch.sparse_csr_tensor(*fe["csr"], size=(m, n), dtype=torch.float64).to_dense().cpu().numpy()
    B, idx0 = fe["B"].cpu().numpy(), fe["idx0"].cpu().numpy()
    L = np.asarray(lv)
    prm = O.make_params(n, max_iters=8, destroy_rate=0.05)
    for q, k in enumerate(slices):
        # the start residual in the device's BLAS order == numpy's on this host
        r0 = A @ L[idx0[q]] - B[q]
        ref = O.solve(A, B[q], L, idx0[q], r0, float(np.max(np.abs(r0))), 0, prm, O.pcg_from_seed(int(k)))
        assert rep.slices[q] == k
        np.testing.assert_array_equal(rep.codes[q].astype(np.int32), ref["best_idx"][0])
        assert rep.objective[q] == ref["best_objective"][0]
        assert rep.iterations[q] == ref["iterations"][0]
        assert rep.moves_scored[q, 0] == ref["moves_scored"][0, 0]  # reference-equivalent count
