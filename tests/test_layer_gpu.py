"""The benchmarked workload itself, parity-checked: whole PTQ layers of the
C5 (4096 -> 14336) and C4 (768 -> 3072) shapes pushed through
ptq.solve_layer with more rows than resident CTA slots (the chunked,
migrating persistent path bench.py times), at the full 100 ALNS iterations
per row, against goldens made by the unmodified reference for C5 rows
{0, 1, 14335} and C4 rows {0, 3071} (tests/golden/make_golden_layers.py):
best codes, objectives, iteration counts and the full per-iteration trace,
bit for bit."""

import numpy as np
import pytest

from tests.golden import recipes
from tests.golden_io import load, sha

pytestmark = pytest.mark.gpu

LAYERS = {"c5": (4096, 14336, 640), "c4": (768, 3072, 700)}


@pytest.mark.parametrize("name", ["c4", "c5"])
def test_layer_rows_match_reference(name):
    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    from paper_2508_13437_b200 import SolverConfig, ptq

    d, total, lead = LAYERS[name]
    recs = load(f"layer_{name}")
    X, W = recipes.ptq_layer(d, total)
    if sha(X) != recs[0]["X_sha"] or sha(W) != recs[0]["W_sha"]:
        pytest.skip("this host's numpy does not regenerate the layer bits")
    pinned = [int(r["row"]) for r in recs]
    rows = np.unique(np.concatenate([np.arange(lead), pinned]))
    assert rows.size > 296  # more rows than resident slots: the chunked, migrating path
    rep = ptq.solve_layer(X, W, bits=4, cfg=SolverConfig(max_iters=100), rows=rows, trace=True)
    tr = rep.seconds["trace"]
    for rec in recs:
        k = int(np.searchsorted(rows, int(rec["row"])))
        it = int(rec["iterations"])
        assert rep.iterations[k] == it
        np.testing.assert_array_equal(rep.levels[k], rec["levels"])
        assert rep.initial_objective[k] == rec["initial_objective"]
        np.testing.assert_array_equal(rep.codes[k].astype(np.int32), rec["best_idx"])
        assert rep.objective[k] == rec["best_objective"]
        np.testing.assert_array_equal(tr["trace_current_t"][k, :it], rec["trace_current_t"])
        np.testing.assert_array_equal(tr["trace_best_t"][k, :it], rec["trace_best_t"])
        np.testing.assert_array_equal(tr["trace_pair"][k, :it], rec["trace_pair"])
        np.testing.assert_array_equal(tr["trace_accepted"][k, :it], rec["trace_accepted"])


def test_c5_random_rows_full_depth_match_oracle():
    """64 fixed random rows of the C5 layer at the full 100 iterations (the
    bench's CPU baseline sample, tools/cpu_full_depth.py) against the CPU
    oracle's run of the same rows: every trace, code and objective bitwise."""
    import os

    import torch

    if not torch.cuda.is_available():
        pytest.fail("GPU test run without a visible CUDA device")
    from paper_2508_13437_b200 import SolverConfig, ptq

    path = os.path.join(os.path.dirname(__file__), "golden", "c5_fulldepth64.npz")
    if not os.path.exists(path):
        pytest.skip("tests/golden/c5_fulldepth64.npz not generated (tools/cpu_full_depth.py)")
    g = np.load(path)
    rows = g["rows"]
    X, W = recipes.ptq_layer(4096, 14336)
    rep = ptq.solve_layer(X, W, bits=4, cfg=SolverConfig(max_iters=100), rows=rows, trace=True)
    tr = rep.seconds["trace"]
    np.testing.assert_array_equal(rep.iterations, g["iterations"])
    np.testing.assert_array_equal(rep.objective, g["best_objective"])
    np.testing.assert_array_equal(rep.codes.astype(np.int8), g["best_idx"])
    for f in ("trace_current_t", "trace_best_t", "trace_pair", "trace_accepted"):
        np.testing.assert_array_equal(tr[f][:, :100], g[f][:, :100], err_msg=f)
