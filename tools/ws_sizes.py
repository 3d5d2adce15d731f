"""Device workspace of the sparse engine for the full 256^2 x 180 slice
(1 and 148 slices) next to the dense engine's copies (diagnostic)."""
import os
import sys

sys.path.insert(0, os.path.dirname(os.path.dirname(os.path.abspath(__file__))))
import numpy as np  # noqa: E402

from paper_2508_13437_b200 import SolverConfig, tomo  # noqa: E402

csr = tomo.projection_csr_device(256, 180)
m, n = 256 * 180, 256 * 256
for count in (1, 148):
    sb = tomo.SparseSliceBatch(csr, m, n, np.zeros((count, m)), (0.0, 1.0, 2.0), np.zeros((count, n), np.int32))
    ws = sb.workspace_bytes(SolverConfig(max_iters=1))
    a_bytes = sum(t.numel() * t.element_size() for t in (sb.cptr, sb.crow, sb.cval, sb.rptr, sb.rcol, sb.rval))
    print(f"slices={count} sparse workspace {ws / 1e9:.2f} GB, A as CSC+CSR {a_bytes / 1e9:.2f} GB, "
          f"max_col_nnz {sb.max_col_nnz}; dense engine copies A/At/Ar {3 * 8 * m * n / 1e9:.1f} GB")
