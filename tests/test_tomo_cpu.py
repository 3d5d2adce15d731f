"""Tomography front end (C3 family): the package's projector must reproduce
the reference's projection matrix bit for bit (CPU-only)."""

import numpy as np

from paper_2508_13437_b200 import tomo
from tests.golden_io import load, sha, stored_A


def test_projector_matches_stored_reference_matrix():
    rec = load("solve_c3s")[0]  # 64^2 x 45 angles, A from dmmv.parallel_beam_matrix
    A = tomo.projection_matrix(64, 45)
    ref = stored_A(rec)
    assert A.shape == ref.shape
    assert np.array_equal(A.view(np.uint64), ref.view(np.uint64))


def test_projector_matches_medium_reference_sha():
    rec = load("solve_c3m")[0]
    side, n_angles = (int(v) for v in rec["A_recipe"])
    assert sha(tomo.projection_matrix(side, n_angles)) == str(rec["A_sha"])


def test_csr_rows_and_phantoms():
    indptr, idx, val = tomo.projection_csr(16, 9)
    assert indptr.size == 16 * 9 + 1 and indptr[-1] == idx.size == val.size
    assert np.all(val > 0) and np.all((idx >= 0) & (idx < 256))
    for r in range(indptr.size - 1):  # strictly increasing pixels per ray
        assert np.all(np.diff(idx[indptr[r]:indptr[r + 1]]) > 0)
    # every ray through the box has total length <= the box diagonal
    lens = np.add.reduceat(val, indptr[:-1][np.diff(indptr) > 0])
    assert np.all(lens <= 16 * np.sqrt(2) + 1e-9)
    img = tomo.phantom("squares", 16)
    assert set(np.unique(img)) == {0, 1, 2}
